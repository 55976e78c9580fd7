#!/usr/bin/env python3
"""Benchmark of the B200 boundary-integral hot path (BASELINE.json metric:
particle-triangle integral+gradient evals/sec (FP64) and % of FP64 peak).

Headline workload (--workload cfg5, default; BASELINE.json configs[4], the
north-star 1/2/4/8-GPU configuration): 16,000,000 particles uniform in
[0,100]^2, ~2,000,000 boundary triangles (Delaunay triangulations of Bridson
Poisson-disk points, min spacing 0.05, inside 500 obstacle discs), Wendland C2,
h = 0.1, field == 1. Seeded synthetic scene (scenes.cfg5; no dataset exists).

One step = the whole scene through sphbi_evaluate: device cell-list pair
finding (K1-K3) -> pair-integral pipeline (K4) -> per-particle reduction (K5),
and for N > 1 the all-gather of the per-particle records.
  value : inputs resident in HBM; CUDA events on the launching stream; the
          mesh (96 MB) and particles (256 MB) exceed the 126 MB L2 and the L2
          is flushed (256 MB write) between steps.
  e2e   : the same step through the C-ABI from pinned HOST buffers: H2D of the
          (shard's) particles and the mesh, D2H of the full per-particle
          result, every step.
Multi-GPU (torchrun, one rank per GPU, NCCL): strong scaling of ONE scene --
particles cut into contiguous ranges at equal pair counts (device count pass
sphbi_pair_counts, sharded, once at setup), mesh replicated, each rank
evaluates its range straight into its slice of an in-place NCCL all-gather
buffer (paper_2507_21686_b200/shard.py); max step time over ranks.

--workload cfg2a: the round-1 line (cfg2 own-triangle pairs, 4,194,304 pair
evaluations, Wendland C4, h = 0.05; weak scaling, one scene per rank).
--impl reference: the reference's own CPU implementation (oracle/_ref, the
unmodified headers compiled here) on all host cores, bounded samples of the
same workload; rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import platform
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "particle-triangle integral+gradient evals/sec (FP64) and % of FP64 peak"
UNIT = "pair-evals/s"
PROFILES = ROOT / "profiles"
# ncu FP64 instruction counts of the K4 kernels (tools/ncu_fp64.py); the frozen
# first-kernel F_pair of BASELINE.md §5 stays in F_pair.json
FP64_PROFILE = {"cfg5": PROFILES / "r02af_fp64_cfg5.json", "cfg2a": PROFILES / "r02af_fp64_cfg2a.json"}
F_PAIR_FILE = PROFILES / "F_pair.json"


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms during the
    timed region (one persistent `nvidia-smi -lms 100` process)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc is None:
            return
        time.sleep(0.15)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        for line in out.splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None

        sm = [v for v in (num(r[1]) for r in self.rows) if v is not None]
        mx = [v for v in (num(r[2]) for r in self.rows) if v is not None]
        busy = [v for v in sm if v > 500] or sm  # samples under load
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, n in enumerate(names):
                if r[5 + i].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# the CPU reference path (oracle/_ref: the unmodified reference headers)
# ---------------------------------------------------------------------------
def ref_library():
    """The reference CPU implementation: oracle/_ref/libsphbi_ref.so (unmodified
    headers) if it was built here, else the plain-C restatement (built on demand)."""
    ref = ROOT / "oracle" / "_ref" / "libsphbi_ref.so"
    if ref.exists():
        lib = ctypes.CDLL(str(ref))
        return lib, "reference", lib.sphbi_ref_eval_pairs
    port = ROOT / "oracle" / "_ref" / "libsphbi_oracle.so"
    if not port.exists():
        subprocess.run(["make", "-C", str(ROOT / "oracle"), "_ref/libsphbi_oracle.so"], check=True,
                       capture_output=True)
    lib = ctypes.CDLL(str(port))
    return lib, "port", lib.oracle_eval_pairs


def oracle_lib():
    p = ROOT / "oracle" / "_ref" / "libsphbi_oracle.so"
    if not p.exists():
        subprocess.run(["make", "-C", str(ROOT / "oracle"), "_ref/libsphbi_oracle.so"], check=True,
                       capture_output=True)
    L = ctypes.CDLL(str(p))
    V = ctypes.c_void_p
    L.oracle_find_pairs_grid.argtypes = [ctypes.c_int64, V, ctypes.c_int64, V, ctypes.c_double, V, ctypes.c_int64]
    L.oracle_find_pairs_grid.restype = ctypes.c_int64
    return L


def host_info():
    model = "unknown"
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    lib, kind, _ = ref_library()
    try:
        fn = lib.sphbi_ref_ldbl_mant_dig if kind == "reference" else lib.oracle_ldbl_mant_dig
        ldbl = int(fn())
    except AttributeError:
        ldbl = None
    return {"cpu_model": model, "machine": platform.machine(), "LDBL_MANT_DIG": ldbl,
            "compiler_flags": "g++ -O2 -std=gnu++20 -Dsphbi=sphbi_ref (oracle/Makefile; no -march=native)"}


def cpu_eval_pairs(particles, triangles, values, kernel, h, pp, pt, nthreads):
    """integrate_triangle per pair on the CPU reference; returns (seconds, kind, status)."""
    lib, kind, fn = ref_library()
    P = ctypes.c_void_p
    fn.argtypes = [ctypes.c_int64, P, P, P, P, P, P, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                   ctypes.c_int, P, P]
    pp = np.ascontiguousarray(pp, dtype=np.int64)
    pt = np.ascontiguousarray(pt, dtype=np.int64)
    coef = np.array(kernel.coefficients, dtype=np.float64)
    out = np.zeros((pp.shape[0], 4))
    fail = ctypes.c_int64(-1)
    vals = values if values is not None else np.ones((triangles.shape[0], 3))
    t0 = time.perf_counter()
    st = fn(pp.shape[0], pp.ctypes.data, pt.ctypes.data, np.ascontiguousarray(particles).ctypes.data,
            np.ascontiguousarray(triangles).ctypes.data, np.ascontiguousarray(vals).ctypes.data, coef.ctypes.data,
            coef.shape[0], kernel.normalization, h, nthreads, out.ctypes.data, ctypes.byref(fail))
    return time.perf_counter() - t0, kind, st


def cpu_find_pairs(particles, triangles, h):
    """The CPU pair finder (same exact predicate, grid-accelerated, 1 thread)."""
    L = oracle_lib()
    cap = 64 * particles.shape[0] + 1024
    buf = np.zeros((cap, 2), dtype=np.int64)
    P = np.ascontiguousarray(particles)
    T = np.ascontiguousarray(triangles)
    t0 = time.perf_counter()
    n = L.oracle_find_pairs_grid(P.shape[0], P.ctypes.data, T.shape[0], T.ctypes.data, h, buf.ctypes.data, cap)
    dt = time.perf_counter() - t0
    assert n <= cap
    return buf[:n], dt


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------
def load_scene(workload, rank=0):
    from paper_2507_21686_b200 import scenes
    if workload == "cfg5":
        return scenes.cfg5()
    return scenes.cfg2(seed_offset=rank)


def bench_config(workload, sc, world, total_pairs=None):
    if workload == "cfg5":
        return {"workload": "cfg5: 16M uniform particles, ~2M Delaunay obstacle triangles (BASELINE.json configs[4])",
                "particles": int(sc.particles.shape[0]), "triangles": int(sc.triangles.shape[0]),
                "pairs_per_step": total_pairs, "h": sc.h, "kernel": "wendland_c2", "field": "1",
                "pairing": "device cell list (pair finding inside the timed step)",
                "l2": "inputs > L2 (352 MB) and a 256 MB L2 flush between timed steps",
                "parallelism": (f"particle shards x{world} (equal pair counts), mesh replicated, NCCL all-gather"
                                if world > 1 else "1 GPU")}
    return {"workload": "cfg2 stress triangles, own-triangle pairs (mode A)", "pairs_per_gpu": int(sc.pairs[0].shape[0]),
            "triangles_per_gpu": int(sc.triangles.shape[0]), "particles_per_gpu": int(sc.particles.shape[0]),
            "h": sc.h, "kernel": "wendland_c4", "field": "1",
            "l2": "flushed between timed steps (256 MB write) + inputs > L2",
            "parallelism": f"weak x{world} (independent scenes, no collective)"}


def run_reference(args, rank, world):
    """--impl reference: the reference CPU path on the host cores (rank 0 only)."""
    if rank != 0:
        return 0
    sc = load_scene(args.workload)
    k = sc.kernels[0]
    threads = os.cpu_count() or 1
    rng = np.random.default_rng(123)
    times, find_s = [], []
    pairs_done = 0
    kind = "reference"
    if args.workload == "cfg5":
        per_step = 16384  # particles per step: ~180k pairs, ~3 s on 16 cores
        for s in range(args.warmup + args.steps):
            idx = np.sort(rng.choice(sc.particles.shape[0], per_step, replace=False))
            P = sc.particles[idx]
            pr, tf = cpu_find_pairs(P, sc.triangles, sc.h)
            dt, kind, st = cpu_eval_pairs(P, sc.triangles, None, k, sc.h, pr[:, 0], pr[:, 1], threads)
            if s >= args.warmup:
                times.append(dt + tf)
                find_s.append(tf)
                pairs_done += pr.shape[0]
        sample = (f"{per_step} seeded random particles of the 16M-particle cfg5 scene per step, all their "
                  f"pairs (CPU grid pair finder, 1 thread, {sum(find_s):.2f} s of the total, + reference "
                  f"integrate_triangle per pair on {threads} threads)")
    else:
        n = sc.pairs[0].shape[0]
        sample_n = 32768
        for s in range(args.warmup + args.steps):
            idx = np.sort(rng.choice(n, sample_n, replace=False))
            dt, kind, st = cpu_eval_pairs(sc.particles, sc.triangles, sc.values, k, sc.h, sc.pairs[0][idx],
                                          sc.pairs[1][idx], threads)
            if s >= args.warmup:
                times.append(dt)
                pairs_done += sample_n
        sample = f"{sample_n} seeded random pairs of the 4,194,304-pair cfg2 workload per step"
    total = sum(times)
    value = pairs_done / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "strong" if args.workload == "cfg5" else "weak",
        "vs_baseline": None, "dtype": "f64 (x87 f80 internal sums)", "data": "synthetic",
        "config": bench_config(args.workload, sc, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample,
                         **host_info()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def fp64_roofline(workload, pairs, k4_ms, fp64_peak):
    """Roofline of the K4 pipeline from the ncu FP64 instruction counts of the
    same kernels (profiles/r02af_fp64_<workload>.json): achieved = measured flops
    per pair x pairs / live K4 time; also the ncu time-weighted FP64-pipe
    fraction and the BASELINE.md frozen-F_pair fraction."""
    roof = {"bound": "fp64", "peak": fp64_peak, "unit": "TFLOP/s", "kernel_ms": k4_ms,
            "kernel": "K4 pair integrals: k_edge_pairs_f (FP64 constant-field path: closed-form edge sum, one "
                      "kernel, thread per pair)",
            "peak_source": "measured live: DFMA loop over all SMs (sphbi_measure_fp64_peak) in this run"}
    prof = FP64_PROFILE.get(workload)
    if prof is not None and prof.exists():
        d = json.loads(prof.read_text())
        fpp = float(d["flops_per_pair"])
        achieved = fpp * pairs / (k4_ms * 1e-3) / 1e12
        roof.update({"achieved": achieved, "frac": achieved / fp64_peak, "flops_per_pair_measured": fpp,
                     "fp64_pipe_frac_ncu": d.get("fp64_pipe_frac_time_weighted"),
                     "traffic": d.get("dram_bytes_per_pair") and d["dram_bytes_per_pair"] * pairs,
                     "algorithmic_bytes": 72 * pairs,
                     "source": f"{prof.relative_to(ROOT)} (ncu, same kernels and workload)"})
    else:
        roof.update({"achieved": None, "frac": None, "source": "no ncu FP64 profile committed for this workload"})
    if workload == "cfg2a" and F_PAIR_FILE.exists():
        f = json.loads(F_PAIR_FILE.read_text())
        roof["frac_frozen_f_pair"] = f["f_pair"] * pairs / (k4_ms * 1e-3) / 1e12 / fp64_peak
    return roof


def secondary_configs(ctx, names):
    """The other BASELINE.json configs measured in the same run (N = 1, rank
    0): device pair-evals/s through sphbi_evaluate with device-resident inputs
    (pair finding + evaluation + reduction, best of 3 after a warm-up), and
    the reference CPU path on a bounded seeded pair sample of the same scene
    (cfg4: the extended oracle; the reference has no P3 path)."""
    sys.path.insert(0, str(ROOT / "tools"))
    sys.path.insert(0, str(ROOT / "tests"))
    import bench_configs as BC
    import oracle_lib as OL
    from paper_2507_21686_b200 import scenes

    out = {}
    for name in names:
        t0 = time.perf_counter()
        repeat, pairs, note = 1, None, ""
        if name == "cfg1":
            sc = scenes.cfg1()
            repeat = 200
            note = "single triangle, 4,096 particles: latency-bound, mean of 200 back-to-back calls"
        elif name == "cfg2a":
            sc = scenes.cfg2()
            pairs = sc.pairs
            note = "own-triangle pairs (mode A, explicit pair list)"
        elif name == "cfg2b":
            sc = scenes.subsample(scenes.cfg2(), 16384, seed=2)
            sc.pairs = None
            note = "full cell-list pairing (mode B, ~12.5k pairs per particle) on a seeded 16,384-particle subsample"
        elif name == "cfg5cubic":
            sc = scenes.cfg5()
            note = ("cfg5 scene with the 2-piece cubic spline in one pass (sphbi_evaluate_piecewise: one pair search "
                    "at h, inner piece on the pairs within h/2); pairs = pair evaluations over both pieces; CPU: the "
                    "outer piece's pairs through the reference")
        elif name == "cfg3":
            sc = scenes.cfg3()
            note = "1M particles, boundary strip: pair finding dominates"
        else:
            sc = scenes.cfg4()
            note = "4M particles, P3 (cubic) field, degree-12 kernel"
        k = sc.kernels[0]
        pieces = None
        if name == "cfg5cubic":
            pieces = sc.kernels[1:]
            k = pieces[0]
        r = BC.run_device(ctx, sc, k, sc.h, 3, pairs=pairs, repeat=repeat, pieces=pieces)
        dev_ms = r["ms_pairs"] + r["ms_eval"] + r["ms_reduce"]
        row = {"pairs": r["pairs"], "ms_device": dev_ms, "ms_pair_finding": r["ms_pairs"],
               "value": r["pairs"] / (dev_ms * 1e-3), "unit": UNIT, "kernel": k.name, "h": sc.h,
               "particles": int(sc.particles.shape[0]), "triangles": int(sc.triangles.shape[0]), "note": note}
        if name in ("cfg3", "cfg4"):
            row["pair_finding_GBps_algorithmic"] = 28.0 * sc.particles.shape[0] / (r["ms_pairs"] * 1e-3) / 1e9
        if pairs is None:
            m = 256 if name == "cfg2b" else 65536  # cfg2b: ~12.5k pairs per particle
            idx = np.sort(np.random.default_rng(11).choice(sc.particles.shape[0], min(m, sc.particles.shape[0]),
                                                           replace=False))
            pr = OL.cpu_pairs_grid(OL.oracle(), np.ascontiguousarray(sc.particles[idx]), sc.triangles, sc.h)
            pairs = (idx[pr[:, 0]], pr[:, 1])
        if pairs[0].shape[0]:
            row["cpu_baseline"] = BC.cpu_rate(sc, k, sc.h, pairs, 8192 if name in ("cfg4", "cfg2b") else 32768)
            row["gpu_over_cpu"] = row["value"] / row["cpu_baseline"]["value"]
        row["wall_s"] = time.perf_counter() - t0
        out[name] = row
    return out


def allreduce_scalar(dist, dev, value, op, dtype):
    """all_reduce of one number (NCCL on the device, gloo on the host)."""
    import torch
    on_dev = dist.get_backend() == "nccl"
    t = torch.tensor([value], dtype=dtype, device=dev if on_dev else "cpu")
    dist.all_reduce(t, op=op)
    return t.item()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg5", choices=["cfg5", "cfg2a"])
    ap.add_argument("--balance", default="pairs", choices=["pairs", "count"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--configs", default="cfg1,cfg2a,cfg2b,cfg3,cfg4,cfg5cubic",
                    help="secondary BASELINE.json configs measured in the same run at N = 1 ('' for none)")
    args = ap.parse_args()
    if args.impl == "ours":
        args.warmup = max(args.warmup, 3)

    rank = env_int("RANK", 0)
    world = env_int("WORLD_SIZE", 1)
    local = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    from paper_2507_21686_b200 import _native as N
    from paper_2507_21686_b200 import shard
    from paper_2507_21686_b200.sphbi import Context, PolyKernel, _raise, table1_terms

    if os.environ.get("SPHBI_BENCH_BACKEND", "nccl") != "nccl":
        local = local % torch.cuda.device_count()  # functional multi-rank check on fewer GPUs
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        # NCCL over NVLink (one process per GPU). SPHBI_BENCH_BACKEND=gloo runs
        # the same sharded path with several ranks on ONE GPU (NCCL refuses
        # that) -- a functional check of the multi-rank code, not a measurement
        backend = os.environ.get("SPHBI_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    sc = load_scene(args.workload, rank)
    k = sc.kernels[0]
    table = table1_terms(PolyKernel(k.coefficients, k.normalization))
    desc = table.desc()
    n = sc.particles.shape[0]
    T = sc.triangles.shape[0]
    p_d = torch.from_numpy(sc.particles).to(dev)
    t_d = torch.from_numpy(sc.triangles).to(dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2

    ctx = Context(local)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    lib = ctx.lib
    vp = ctypes.c_void_p

    peak = ctypes.c_double(0.0)
    _raise(lib.sphbi_measure_fp64_peak(ctx.handle, ctypes.byref(peak), None))
    fp64_peak = peak.value

    balance_ms = None
    if args.workload == "cfg5":
        t0 = time.perf_counter()
        S = shard.ShardedScene(p_d, t_d, table, sc.h, ctx=ctx, balance=args.balance if world > 1 else "count")
        torch.cuda.synchronize()
        balance_ms = 1e3 * (time.perf_counter() - t0)

        def step_device():
            S.evaluate()
            return S.stats

        def pairs_of(st):
            return st.n_pairs
    else:
        ip_d = torch.from_numpy(sc.pairs[0]).to(dev)
        it_d = torch.from_numpy(sc.pairs[1]).to(dev)
        ov_d = torch.empty(n, dtype=torch.float64, device=dev)
        og_d = torch.empty((n, 2), dtype=torch.float64, device=dev)
        stats = N.Stats()

        def step_device():
            _raise(lib.sphbi_evaluate(ctx.handle, ctypes.byref(desc), sc.h, n, vp(p_d.data_ptr()), T,
                                      vp(t_d.data_ptr()), None, ip_d.shape[0], vp(ip_d.data_ptr()),
                                      vp(it_d.data_ptr()), vp(ov_d.data_ptr()), vp(og_d.data_ptr()), None, None,
                                      ctypes.byref(stats), N.MEM_DEVICE), "evaluate")
            return stats

        def pairs_of(st):
            return st.n_pairs

    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = ctx.launch_count()
    k4_ms, find_ms, red_ms, local_pairs = [], [], [], 0
    sampler = ClockSampler(local)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with sampler:
        for s in range(args.steps):
            flush.zero_()  # L2 flush between timed iterations, outside the events
            ev[s][0].record(stream)
            st = step_device()
            ev[s][1].record(stream)
            k4_ms.append(st.ms_eval)
            find_ms.append(st.ms_pairs)
            red_ms.append(st.ms_reduce)
            local_pairs = pairs_of(st)
        torch.cuda.synchronize()
    launches = ctx.launch_count() - launches0
    arithmetic = ctx.last_precision()  # what the constant-field pipelines ran (sphbi_ctx_set_precision: auto)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    pairs_step = local_pairs
    if dist:
        total_ms = float(allreduce_scalar(dist, dev, total_ms, dist.ReduceOp.MAX, torch.float64))
        pairs_step = int(allreduce_scalar(dist, dev, local_pairs, dist.ReduceOp.SUM, torch.int64))
    ms_per_step = total_ms / args.steps
    value = pairs_step / (ms_per_step * 1e-3)

    # ---- e2e through the public C-ABI with pinned host buffers
    e2e = None
    if not args.no_e2e:
        if args.workload == "cfg5":
            b, e = S.ranges[S.rank]
            p_h = torch.from_numpy(np.ascontiguousarray(sc.particles[b:e])).pin_memory()
            t_h = torch.from_numpy(sc.triangles).pin_memory()
            ov_h = torch.empty(n, dtype=torch.float64).pin_memory()
            og_h = torch.empty((n, 2), dtype=torch.float64).pin_memory()
            ps_d = torch.empty((e - b, 2), dtype=torch.float64, device=dev)
            ts_d = torch.empty_like(t_d)

            def step_host():
                if world == 1:  # the C-ABI's own host-memory path (H2D, evaluate, D2H)
                    _raise(lib.sphbi_evaluate(ctx.handle, ctypes.byref(desc), sc.h, n, vp(p_h.data_ptr()), T,
                                              vp(t_h.data_ptr()), None, -1, None, None, vp(ov_h.data_ptr()),
                                              vp(og_h.data_ptr()), None, None, None, N.MEM_HOST), "evaluate")
                    return
                # H2D of this rank's particles and the mesh, shard evaluation
                # into the all-gather slice, gather, D2H of the full result
                ps_d.copy_(p_h, non_blocking=True)
                ts_d.copy_(t_h, non_blocking=True)
                ov, og = S.local_views()
                _raise(lib.sphbi_evaluate(ctx.handle, ctypes.byref(desc), sc.h, e - b, vp(ps_d.data_ptr()), T,
                                          vp(ts_d.data_ptr()), None, -1, None, None, vp(ov.data_ptr()),
                                          vp(og.data_ptr()), None, None, None, N.MEM_DEVICE), "evaluate")
                v, g = S.gather()
                ov_h.copy_(v, non_blocking=True)
                og_h.copy_(g, non_blocking=True)

            h2d = 16 * (e - b) + 48 * T
            d2h = 24 * n
        else:
            p_h = torch.from_numpy(sc.particles).pin_memory()
            t_h = torch.from_numpy(sc.triangles).pin_memory()
            ip_h = torch.from_numpy(sc.pairs[0]).pin_memory()
            it_h = torch.from_numpy(sc.pairs[1]).pin_memory()
            ov_h = torch.empty(n, dtype=torch.float64).pin_memory()
            og_h = torch.empty((n, 2), dtype=torch.float64).pin_memory()
            npairs = sc.pairs[0].shape[0]

            def step_host():
                _raise(lib.sphbi_evaluate(ctx.handle, ctypes.byref(desc), sc.h, n, vp(p_h.data_ptr()), T,
                                          vp(t_h.data_ptr()), None, npairs, vp(ip_h.data_ptr()),
                                          vp(it_h.data_ptr()), vp(ov_h.data_ptr()), vp(og_h.data_ptr()), None,
                                          None, None, N.MEM_HOST), "evaluate")

            h2d = 16 * n + 48 * T + 16 * npairs
            d2h = 24 * n
        for _ in range(2):
            step_host()
        torch.cuda.synchronize()
        e2e_ms = []
        if dist:
            dist.barrier()
        for s in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            bb = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            step_host()
            bb.record(stream)
            bb.synchronize()
            e2e_ms.append(a.elapsed_time(bb))
        e2e_total = sum(e2e_ms)
        if dist:
            e2e_total = float(allreduce_scalar(dist, dev, e2e_total, dist.ReduceOp.MAX, torch.float64))
        e2e = {"value": pairs_step / (e2e_total / args.steps * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": e2e_total / args.steps}

    k4 = statistics.mean(k4_ms) if k4_ms else float("nan")
    roof = fp64_roofline(args.workload, local_pairs, k4, fp64_peak)

    # ---- CPU baseline (rank 0, N = 1 only): the reference on a bounded sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        if args.workload == "cfg5":
            idx = np.sort(np.random.default_rng(5).choice(n, 65536, replace=False))
            P = sc.particles[idx]
            pr, tf = cpu_find_pairs(P, sc.triangles, sc.h)
            dt, kind, _ = cpu_eval_pairs(P, sc.triangles, None, k, sc.h, pr[:, 0], pr[:, 1], threads)
            cpu = {"value": pr.shape[0] / (dt + tf), "unit": UNIT, "cores": threads, "kind": kind,
                   "sample": f"65,536 seeded particles of the cfg5 scene: {pr.shape[0]} pairs; CPU pair finder "
                             f"{tf:.2f} s (1 thread), reference integrate_triangle {dt:.1f} s ({threads} threads)",
                   "eval_only_value": pr.shape[0] / dt, "pair_finding_s": tf, **host_info()}
        else:
            m = 262144
            idx = np.sort(np.random.default_rng(99).choice(sc.pairs[0].shape[0], m, replace=False))
            dt, kind, _ = cpu_eval_pairs(sc.particles, sc.triangles, None, k, sc.h, sc.pairs[0][idx],
                                         sc.pairs[1][idx], threads)
            cpu = {"value": m / dt, "unit": UNIT, "cores": threads, "kind": kind,
                   "sample": f"{m} seeded random pairs of the 4,194,304-pair cfg2 workload ({dt:.1f} s)",
                   **host_info()}

    clocks = sampler.summary()
    others = None
    if rank == 0 and world == 1 and args.configs and args.workload == "cfg5":
        others = secondary_configs(ctx, [c for c in args.configs.split(",") if c])
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if args.workload == "cfg5" else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded; scenes.py)",
            "config": dict(bench_config(args.workload, sc, world, pairs_step),
                           arithmetic={"fp64": "FP64 (a-priori error bound below the parity floor: fp64_path_ok)",
                                       "dd": "double-double"}[arithmetic]),
            "e2e": e2e,
            "gpu_launches": launches,
            "roofline": roof,
            "fp64_peak_tflops_measured": fp64_peak,
            "cpu_baseline": cpu,
            "clocks": clocks,
            "phases_ms_rank0": {"pair_finding": statistics.mean(find_ms), "k4_eval": k4,
                                "reduce": statistics.mean(red_ms)},
        }
        if balance_ms is not None:
            line["setup_ms"] = {"shard_cut": balance_ms, "count_pass": S.count_ms}
        if others:
            line["other_configs"] = others
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
