#!/usr/bin/env python3
"""Benchmark of the B200 boundary-integral hot path (BASELINE.json metric:
particle-triangle integral+gradient evals/sec (FP64) and % of FP64 peak).

Workload (BASELINE.json configs[1] = cfg2, SURVEY.md §8(d) mode A): 65,536
random triangles in U[0,1]^2 (20% slivers), 64 particles per triangle at
d/h in {0, 1e-12, U(0,1.2)}, Wendland C4, h = 0.05, each particle paired with
its own triangle: 4,194,304 (particle, triangle) pair evaluations per step,
summed per particle. Seeded synthetic data (no dataset exists).

One step = sphbi_evaluate over the whole scene (explicit pair list):
pair packing -> K4 pair-integral kernel -> K5 per-particle reduction.
  value : inputs resident in HBM, device events on the launching stream.
  e2e   : the public C-ABI with pinned HOST buffers: H2D of particles,
          triangles, pair list + D2H of the per-particle results every step.
Multi-GPU (torchrun): weak scaling, each rank evaluates its own cfg2 scene
(seed offset = rank); no data-path collective; max step time over ranks.
--impl reference: the reference's own CPU implementation (oracle/_ref,
the unmodified headers compiled here) on the host cores, bounded sample.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "particle-triangle integral+gradient evals/sec (FP64) and % of FP64 peak"
UNIT = "pair-evals/s"
# Algorithmic FP64 flops per pair evaluation on this workload, frozen from the
# first parity-passing kernel's ncu counters (2*DFMA + DADD + DMUL, thread
# level, predicated on) -- see BASELINE.md §5 / profiles/.
F_PAIR_FILE = ROOT / "profiles" / "F_pair.json"


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


def load_f_pair():
    if F_PAIR_FILE.exists():
        d = json.loads(F_PAIR_FILE.read_text())
        return float(d["f_pair"]), d
    return None, None


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


def cpu_eval_pairs(scene, idx, nthreads):
    """Evaluate the pairs `idx` of scene mode A on the CPU reference; returns seconds."""
    lib, kind, fn = ref_library()
    P = ctypes.c_void_p
    fn.argtypes = [ctypes.c_int64, P, P, P, P, P, P, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                   ctypes.c_int, P, P]
    pp = np.ascontiguousarray(scene.pairs[0][idx])
    pt = np.ascontiguousarray(scene.pairs[1][idx])
    k = scene.kernels[0]
    coef = np.array(k.coefficients, dtype=np.float64)
    out = np.zeros((idx.shape[0], 4))
    fail = ctypes.c_int64(-1)
    vals = scene.values if scene.values is not None else np.ones((scene.triangles.shape[0], 3))
    t0 = time.perf_counter()
    st = fn(idx.shape[0], pp.ctypes.data, pt.ctypes.data, scene.particles.ctypes.data, scene.triangles.ctypes.data,
            np.ascontiguousarray(vals).ctypes.data, coef.ctypes.data, coef.shape[0], k.normalization, scene.h,
            nthreads, out.ctypes.data, ctypes.byref(fail))
    dt = time.perf_counter() - t0
    return dt, kind, st, out


def bench_config(world, T=65536, n=4194304, npairs=4194304, h=0.05):
    """The workload description shared by both arms (ours / --impl reference)."""
    return {"workload": "cfg2 stress triangles, own-triangle pairs (mode A)", "pairs_per_gpu": npairs,
            "triangles_per_gpu": T, "particles_per_gpu": n, "h": h, "kernel": "wendland_c4", "field": "1",
            "l2": "flushed between timed steps (256 MB write) + inputs > L2",
            "parallelism": f"weak x{world} (independent scenes, no collective)"}


def run_reference(args, rank, world):
    """--impl reference: the reference CPU path on the host cores."""
    if rank != 0:
        return 0
    from paper_2507_21686_b200 import scenes
    sc = scenes.cfg2()
    n = sc.pairs[0].shape[0]
    threads = os.cpu_count() or 1
    sample = 32768  # pairs per step: ~0.2-1 s on 16 cores
    rng = np.random.default_rng(123)
    times = []
    kind = "reference"
    for s in range(args.warmup + args.steps):
        idx = np.sort(rng.choice(n, sample, replace=False))
        dt, kind, st, _ = cpu_eval_pairs(sc, idx, threads)
        if s >= args.warmup:
            times.append(dt)
    total = sum(times)
    value = sample * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64 (x87 f80 internal sums)",
        "data": "synthetic", "config": bench_config(world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"{sample} seeded random pairs of the 4,194,304-pair cfg2 workload per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=262144)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    rank = env_int("RANK", 0)
    world = env_int("WORLD_SIZE", 1)
    local = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    from paper_2507_21686_b200 import _native as N
    from paper_2507_21686_b200 import scenes
    from paper_2507_21686_b200.sphbi import Context, table1_terms, PolyKernel, _raise

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    sc = scenes.cfg2(seed_offset=rank)
    k = sc.kernels[0]
    table = table1_terms(PolyKernel(k.coefficients, k.normalization))
    desc = table.desc()
    n = sc.particles.shape[0]
    T = sc.triangles.shape[0]
    npairs = sc.pairs[0].shape[0]
    dev = torch.device("cuda", local)
    p_d = torch.from_numpy(sc.particles).to(dev)
    t_d = torch.from_numpy(sc.triangles).to(dev)
    ip_d = torch.from_numpy(sc.pairs[0]).to(dev)
    it_d = torch.from_numpy(sc.pairs[1]).to(dev)
    ov_d = torch.empty(n, dtype=torch.float64, device=dev)
    og_d = torch.empty((n, 2), dtype=torch.float64, device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2

    ctx = Context(local)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    lib = ctx.lib
    stats = N.Stats()

    def step_device():
        _raise(lib.sphbi_evaluate(ctx.handle, ctypes.byref(desc), sc.h, n, ctypes.c_void_p(p_d.data_ptr()), T,
                                  ctypes.c_void_p(t_d.data_ptr()), None, npairs, ctypes.c_void_p(ip_d.data_ptr()),
                                  ctypes.c_void_p(it_d.data_ptr()), ctypes.c_void_p(ov_d.data_ptr()),
                                  ctypes.c_void_p(og_d.data_ptr()), None, None, ctypes.byref(stats),
                                  N.MEM_DEVICE), "evaluate")

    # FP64 peak at the clocks of this run (roofline denominator)
    peak = ctypes.c_double(0.0)
    _raise(lib.sphbi_measure_fp64_peak(ctx.handle, ctypes.byref(peak), None))
    fp64_peak = peak.value

    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = ctx.launch_count()
    eval_ms = []
    sampler = ClockSampler(local)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with sampler:
        for s in range(args.steps):
            flush.zero_()  # L2 flush between timed iterations, outside the events
            ev[s][0].record(stream)
            step_device()
            ev[s][1].record(stream)
            eval_ms.append(stats.ms_eval)
        torch.cuda.synchronize()
    launches = ctx.launch_count() - launches0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    if dist:
        tt = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    ms_per_step = total_ms / args.steps
    value = world * npairs / (ms_per_step * 1e-3)

    # ---- e2e through the public C-ABI with pinned host buffers
    p_h = torch.from_numpy(sc.particles).pin_memory()
    t_h = torch.from_numpy(sc.triangles).pin_memory()
    ip_h = torch.from_numpy(sc.pairs[0]).pin_memory()
    it_h = torch.from_numpy(sc.pairs[1]).pin_memory()
    ov_h = torch.empty(n, dtype=torch.float64).pin_memory()
    og_h = torch.empty((n, 2), dtype=torch.float64).pin_memory()

    def step_host():
        _raise(lib.sphbi_evaluate(ctx.handle, ctypes.byref(desc), sc.h, n, ctypes.c_void_p(p_h.data_ptr()), T,
                                  ctypes.c_void_p(t_h.data_ptr()), None, npairs, ctypes.c_void_p(ip_h.data_ptr()),
                                  ctypes.c_void_p(it_h.data_ptr()), ctypes.c_void_p(ov_h.data_ptr()),
                                  ctypes.c_void_p(og_h.data_ptr()), None, None, None, N.MEM_HOST), "evaluate")

    for _ in range(2):
        step_host()
    e2e_ms = []
    if dist:
        dist.barrier()
    for s in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step_host()
        b.record(stream)
        b.synchronize()
        e2e_ms.append(a.elapsed_time(b))
    e2e_total = sum(e2e_ms)
    if dist:
        tt = torch.tensor([e2e_total], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_total = float(tt.item())
    e2e_value = world * npairs / (e2e_total / args.steps * 1e-3)
    h2d = 16 * n + 48 * T + 16 * npairs
    d2h = 24 * n

    # ---- roofline of the dominant kernel (K4 k_eval_scene_pairs)
    f_pair, f_info = load_f_pair()
    k_ms = statistics.mean(eval_ms) if eval_ms else float("nan")
    roof = None
    if f_pair:
        achieved = f_pair * npairs / (k_ms * 1e-3) / 1e12
        roof = {"bound": "fp64", "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": achieved / fp64_peak, "traffic": f_info.get("traffic_bytes_per_launch"),
                "kernel": "K4 pair-integral pipeline (k_pipe_count/emit/stub/sector/segment/combine)",
                "kernel_ms": k_ms, "f_pair": f_pair,
                "peak_source": "measured live: DFMA loop (sphbi_measure_fp64_peak) in this run"}

    # ---- CPU baseline (rank 0, N = 1 only): bounded sample of the same workload
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        m = min(args.cpu_sample, npairs)
        idx = np.sort(np.random.default_rng(99).choice(npairs, m, replace=False))
        dt, kind, st, _ = cpu_eval_pairs(sc, idx, threads)
        cpu = {"value": m / dt, "unit": UNIT, "cores": threads, "kind": kind,
               "sample": f"{m} seeded random pairs of the 4,194,304-pair cfg2 workload ({dt:.1f} s)"}

    clocks = sampler.summary()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(world, T, n, npairs, sc.h),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "roofline": roof,
            "fp64_peak_tflops_measured": fp64_peak,
            "cpu_baseline": cpu,
            "clocks": clocks,
            "phases_ms": {"eval_kernel": k_ms, "pairs_pack": stats.ms_pairs, "reduce": stats.ms_reduce},
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
