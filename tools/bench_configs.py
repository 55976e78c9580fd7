"""Per-config throughput report: every BASELINE.json config
through the product path (sphbi_evaluate / sphbi_evaluate_p3, device-resident
inputs, device-clock stats), plus the reference CPU path (oracle/_ref, all
host cores) on a bounded sample of the same pairs.

    python tools/bench_configs.py [--reps 3] [--cpu] [--out profiles/r01_configs.json]

Rates are pair-evaluations per second (one (particle, triangle) pair within h
evaluated to value + 2-gradient and reduced). "device" = pair finding +
evaluation + reduction on the device clock; "eval" = evaluation + reduction.
cfg1 is latency-bound (2.5k pairs): it is timed as R back-to-back calls.
cfg2 mode B (full cell-list pairing, ~6.3e10 pairs) runs on a seeded particle
subsample and reports the rate.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_21686_b200 import _native as N  # noqa: E402
from paper_2507_21686_b200 import scenes  # noqa: E402
from paper_2507_21686_b200.sphbi import Context, PolyKernel, _raise, table1_terms  # noqa: E402

dev = torch.device("cuda", 0)


def run_device(ctx, sc, kernel, h, reps, pairs=None, repeat=1, pieces=None):
    """Device-resident evaluation; returns dict of best-of-reps timings.
    pieces: list of KernelSpec -> one-pass piecewise evaluation (sphbi_evaluate_piecewise)."""
    desc = table1_terms(PolyKernel(list(kernel.coefficients), kernel.normalization)).desc()
    if pieces is not None:
        descs = (N.KernelDesc * len(pieces))()
        for j, kk in enumerate(pieces):
            descs[j] = table1_terms(PolyKernel(list(kk.coefficients), kk.normalization)).desc()
        scales = np.array([kk.support_scale for kk in pieces], dtype=np.float64)
    p = torch.from_numpy(np.ascontiguousarray(sc.particles)).to(dev)
    t = torch.from_numpy(np.ascontiguousarray(sc.triangles)).to(dev)
    vals = None
    fn = ctx.lib.sphbi_evaluate
    if sc.values is not None and sc.values.ndim == 2 and sc.values.shape[1] == 10:
        vals = torch.from_numpy(np.ascontiguousarray(sc.values)).to(dev)
        fn = ctx.lib.sphbi_evaluate_p3
    n, T = p.shape[0], t.shape[0]
    ov = torch.empty(n, dtype=torch.float64, device=dev)
    og = torch.empty((n, 2), dtype=torch.float64, device=dev)
    ip = it = None
    npairs = -1
    if pairs is not None:
        ip = torch.from_numpy(np.ascontiguousarray(pairs[0], dtype=np.int64)).to(dev)
        it = torch.from_numpy(np.ascontiguousarray(pairs[1], dtype=np.int64)).to(dev)
        npairs = ip.shape[0]
    vp = ctypes.c_void_p
    st = N.Stats()
    best = None
    for r in range(reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tot = [0.0, 0.0, 0.0]
        for _ in range(repeat):
            if pieces is not None:
                _raise(ctx.lib.sphbi_evaluate_piecewise(
                    ctx.handle, len(pieces), descs, vp(scales.ctypes.data), float(h), n, vp(p.data_ptr()), T,
                    vp(t.data_ptr()), vp(vals.data_ptr()) if vals is not None else None, npairs,
                    vp(ip.data_ptr()) if ip is not None else None, vp(it.data_ptr()) if it is not None else None,
                    vp(ov.data_ptr()), vp(og.data_ptr()), None, None, ctypes.byref(st), N.MEM_DEVICE))
            else:
                _raise(fn(ctx.handle, ctypes.byref(desc), float(h), n, vp(p.data_ptr()), T, vp(t.data_ptr()),
                          vp(vals.data_ptr()) if vals is not None else None, npairs,
                          vp(ip.data_ptr()) if ip is not None else None,
                          vp(it.data_ptr()) if it is not None else None,
                          vp(ov.data_ptr()), vp(og.data_ptr()), None, None, ctypes.byref(st), N.MEM_DEVICE))
            tot[0] += st.ms_pairs
            tot[1] += st.ms_eval
            tot[2] += st.ms_reduce
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3 / repeat
        rec = {"pairs": int(st.n_pairs), "ms_pairs": tot[0] / repeat, "ms_eval": tot[1] / repeat,
               "ms_reduce": tot[2] / repeat, "ms_wall": wall}
        if r == 0:
            continue  # warm-up (scratch allocation)
        if best is None or rec["ms_pairs"] + rec["ms_eval"] + rec["ms_reduce"] < \
                best["ms_pairs"] + best["ms_eval"] + best["ms_reduce"]:
            best = rec
    return best


def run_sweep(ctx, sc, kernel, h, reps, pairs=None, variant=1):
    """Vertex-basis cache (sphbi_bases_create) + field sweeps (sphbi_bases_apply,
    difference variant) with device-resident inputs; the apply kernel is
    HBM-bound: algorithmic bytes = 76 per pair (9 cached doubles + triangle id)
    + 40 per particle (row pointer, a0, rho0, value, gradient) + 48 per triangle."""
    desc = table1_terms(PolyKernel(list(kernel.coefficients), kernel.normalization)).desc()
    vp = ctypes.c_void_p
    p = torch.from_numpy(np.ascontiguousarray(sc.particles)).to(dev)
    t = torch.from_numpy(np.ascontiguousarray(sc.triangles)).to(dev)
    n, T = p.shape[0], t.shape[0]
    ip = it = None
    npairs = -1
    if pairs is not None:
        ip = torch.from_numpy(np.ascontiguousarray(pairs[0], dtype=np.int64)).to(dev)
        it = torch.from_numpy(np.ascontiguousarray(pairs[1], dtype=np.int64)).to(dev)
        npairs = ip.shape[0]
    st = N.Stats()
    cache = vp()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _raise(ctx.lib.sphbi_bases_create(ctx.handle, ctypes.byref(desc), float(h), n, vp(p.data_ptr()), T,
                                      vp(t.data_ptr()), npairs, vp(ip.data_ptr()) if ip is not None else None,
                                      vp(it.data_ptr()) if it is not None else None, ctypes.byref(st),
                                      N.MEM_DEVICE, ctypes.byref(cache)), "bases_create")
    torch.cuda.synchronize()
    create_ms = (time.perf_counter() - t0) * 1e3
    m = ctypes.c_int64(0)
    ctx.lib.sphbi_bases_info(cache, None, None, ctypes.byref(m))
    g = torch.Generator(device="cpu").manual_seed(5)
    A = torch.randn((T, 3), generator=g, dtype=torch.float64).to(dev)
    rho = (0.5 + 1.5 * torch.rand((T, 3), generator=g, dtype=torch.float64)).to(dev)
    a0 = torch.randn(n, generator=g, dtype=torch.float64).to(dev)
    rho0 = (0.5 + 1.5 * torch.rand(n, generator=g, dtype=torch.float64)).to(dev)
    ov = torch.empty(n, dtype=torch.float64, device=dev)
    og = torch.empty((n, 2), dtype=torch.float64, device=dev)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    best = None
    for r in range(reps + 2):
        flush.fill_(float(r))  # L2 flush between sweeps
        ms = ctypes.c_double(0.0)
        _raise(ctx.lib.sphbi_bases_apply(cache, variant, vp(A.data_ptr()), vp(rho.data_ptr()), vp(a0.data_ptr()),
                                         vp(rho0.data_ptr()), vp(ov.data_ptr()), vp(og.data_ptr()),
                                         ctypes.byref(ms), N.MEM_DEVICE), "bases_apply")
        if r >= 1 and (best is None or ms.value < best):
            best = ms.value
    ctx.lib.sphbi_bases_destroy(cache)
    mp = int(m.value)
    algo = 76.0 * mp + 40.0 * n + 48.0 * T
    return {"pairs": mp, "ms_create_wall": create_ms, "ms_create_eval": st.ms_eval, "ms_apply": best,
            "sweep_pair_evals_per_s": mp / (best * 1e-3), "apply_GBps_algorithmic": algo / (best * 1e-3) / 1e9,
            "apply_bytes_algorithmic": algo}


def cpu_rate(sc, kernel, h, pairs, sample):
    """Reference (oracle/_ref, all host cores) on a seeded pair sample."""
    import oracle_lib as OL
    L = OL.ref()
    rng = np.random.default_rng(7)
    m = pairs[0].shape[0]
    idx = np.sort(rng.choice(m, size=min(sample, m), replace=False))
    pp = np.ascontiguousarray(pairs[0][idx], dtype=np.int64)
    pt = np.ascontiguousarray(pairs[1][idx], dtype=np.int64)
    c = np.ascontiguousarray(kernel.coefficients, dtype=np.float64)
    out = np.zeros((pp.shape[0], 4))
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    if sc.values is not None and sc.values.shape[1] == 10:
        O = OL.oracle()  # the reference has no P3 path: extended oracle
        fail = ctypes.c_int64(-1)
        O.oracle_eval_pairs_p3(pp.shape[0], OL.ptr(pp), OL.ptr(pt), OL.ptr(OL.arr(sc.particles)),
                               OL.ptr(OL.arr(sc.triangles)), OL.ptr(OL.arr(sc.values)), OL.ptr(c), c.shape[0],
                               kernel.normalization, h, threads, OL.ptr(out), ctypes.byref(fail))
        kind = "port (extended oracle; the reference has no P3 path)"
    else:
        # field == 1 as vertex values (1, 1, 1): the reference needs a value array
        vals = OL.arr(np.ones((sc.triangles.shape[0], 3)) if sc.values is None else sc.values)
        L.sphbi_ref_eval_pairs(pp.shape[0], OL.ptr(pp), OL.ptr(pt), OL.ptr(OL.arr(sc.particles)),
                               OL.ptr(OL.arr(sc.triangles)), OL.ptr(vals), OL.ptr(c),
                               c.shape[0], kernel.normalization, h, threads, OL.ptr(out),
                               ctypes.byref(ctypes.c_int64(-1)))
        kind = "reference"
    dt = time.perf_counter() - t0
    return {"value": pp.shape[0] / dt, "cores": threads, "kind": kind, "sample": int(pp.shape[0]),
            "seconds": dt}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--cpu", action="store_true")
    ap.add_argument("--configs", default="cfg1,cfg2A,cfg2B,cfg3,cfg4,cfg5_c2,cfg5_cubic,cfg5_cubic_1pass,cfg2A_sweep,cfg5_sweep")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    ctx = Context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    rows = []
    want = a.configs.split(",")
    cfg5 = None
    for name in want:
        t0 = time.time()
        pairs_for_cpu = None
        if name == "cfg1":
            sc = scenes.cfg1()
            k = sc.kernels[0]
            r = run_device(ctx, sc, k, sc.h, a.reps, repeat=200)
            note = "latency-bound (2.5k pairs): mean of 200 back-to-back calls"
        elif name == "cfg2A":
            sc = scenes.cfg2()
            k = sc.kernels[0]
            r = run_device(ctx, sc, k, sc.h, a.reps, pairs=sc.pairs)
            note = "own-triangle pairs (mode A), explicit pair list"
            pairs_for_cpu = sc.pairs
        elif name == "cfg2B":
            full = scenes.cfg2()
            sc = scenes.subsample(full, 16384, seed=2)
            sc.pairs = None
            k = sc.kernels[0]
            r = run_device(ctx, sc, k, sc.h, a.reps)
            note = "full cell-list pairing (mode B) on a seeded 16,384-particle subsample (rate)"
        elif name in ("cfg3", "cfg4"):
            sc = scenes.cfg3() if name == "cfg3" else scenes.cfg4()
            k = sc.kernels[0]
            r = run_device(ctx, sc, k, sc.h, a.reps)
            note = "device cell list over all particles; P3 field" if name == "cfg4" else "device cell list"
        elif name.startswith("cfg5") and not name.endswith("_sweep"):
            if cfg5 is None:
                cfg5 = scenes.cfg5()
            sc = cfg5
            ks = [sc.kernels[0]] if name == "cfg5_c2" else sc.kernels[1:]
            if name == "cfg5_cubic_1pass":
                r = run_device(ctx, sc, ks[0], sc.h, a.reps, pieces=ks)
                note = ("cubic spline in one pass (sphbi_evaluate_piecewise): one pair search at h, "
                        "inner piece on the pairs within h/2, one reduction; pairs = evaluations of both pieces")
            else:
                rs = [run_device(ctx, sc, kk, sc.h * kk.support_scale, a.reps) for kk in ks]
                r = {key: sum(x[key] for x in rs) for key in rs[0]}
                r["pairs"] = sum(x["pairs"] for x in rs)
                note = ("Wendland C2, h = 0.1" if name == "cfg5_c2" else
                        "cubic spline as outer (h) + inner (h/2) passes; pairs summed over both passes")
            k = ks[0]
        elif name.endswith("_sweep"):
            base = name[: -len("_sweep")]
            if base == "cfg2A":
                sc = scenes.cfg2()
                pr = sc.pairs
            elif base == "cfg5":
                if cfg5 is None:
                    cfg5 = scenes.cfg5()
                sc, pr = cfg5, None
            else:
                raise SystemExit(f"unknown sweep config {name}")
            k = sc.kernels[0]
            r = run_sweep(ctx, sc, k, sc.h, a.reps, pairs=pr)
            row = {"config": name, "particles": int(sc.particles.shape[0]), "triangles": int(sc.triangles.shape[0]),
                   "kernel": k.name, "h": sc.h, **r,
                   "note": "basis cache built once (integrate_triangle_bases per pair), then field sweeps "
                           "(difference variant) re-combining cached bases; best of reps, L2 flushed"}
            rows.append(row)
            print(json.dumps(row), flush=True)
            print(f"  [{name} took {time.time() - t0:.1f} s]", file=sys.stderr, flush=True)
            continue
        else:
            raise SystemExit(f"unknown config {name}")
        dev_ms = r["ms_pairs"] + r["ms_eval"] + r["ms_reduce"]
        row = {"config": name, "particles": int(sc.particles.shape[0]), "triangles": int(sc.triangles.shape[0]),
               "kernel": k.name, "h": sc.h, "pairs": r["pairs"], "ms_pairs": r["ms_pairs"], "ms_eval": r["ms_eval"],
               "ms_reduce": r["ms_reduce"], "ms_device": dev_ms, "ms_wall": r["ms_wall"],
               "device_pair_evals_per_s": r["pairs"] / (dev_ms * 1e-3) if dev_ms > 0 else None,
               "eval_pair_evals_per_s": r["pairs"] / ((r["ms_eval"] + r["ms_reduce"]) * 1e-3),
               "note": note}
        if name in ("cfg3", "cfg4"):
            # pair finding reads every particle (16 B) and writes its cell / pair count (12 B):
            # algorithmic bytes of K1-K3 over the device pair-finding time
            row["pair_finding_GBps_algorithmic"] = 28.0 * sc.particles.shape[0] / (r["ms_pairs"] * 1e-3) / 1e9
        if a.cpu and name != "cfg1" and name != "cfg2B":
            hh = sc.h * k.support_scale
            if pairs_for_cpu is None:  # cell-list configs: CPU pair finder on a particle subsample
                import oracle_lib as OL
                rng = np.random.default_rng(11)
                sub = np.sort(rng.choice(sc.particles.shape[0], min(200_000, sc.particles.shape[0]), replace=False))
                pr = OL.cpu_pairs_grid(OL.oracle(), np.ascontiguousarray(sc.particles[sub]), sc.triangles, hh)
                pairs_for_cpu = (sub[pr[:, 0]], pr[:, 1])
            row["cpu_baseline"] = cpu_rate(sc, k, hh, pairs_for_cpu, 65536 if name != "cfg4" else 8192)
            row["gpu_over_cpu_device"] = row["device_pair_evals_per_s"] / row["cpu_baseline"]["value"]
        rows.append(row)
        print(json.dumps(row), flush=True)
        print(f"  [{name} took {time.time() - t0:.1f} s]", file=sys.stderr, flush=True)
    if a.out:
        Path(a.out).write_text(json.dumps(rows, indent=1) + "\n")
    ctx.close()


if __name__ == "__main__":
    main()
