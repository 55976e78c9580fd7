"""Anatomy of the e2e (pinned host) cfg2 step: copy-engine bandwidths and the
device time of the pipeline on particle chunks of the streamed path."""
import ctypes
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_21686_b200 import _native as N  # noqa: E402
from paper_2507_21686_b200 import scenes  # noqa: E402
from paper_2507_21686_b200.sphbi import Context, PolyKernel, _raise, table1_terms  # noqa: E402

x = torch.empty(137_363_456 // 8, dtype=torch.float64).pin_memory()
y = torch.empty(100_663_296 // 8, dtype=torch.float64).pin_memory()
dx = torch.empty_like(x, device="cuda")
dy = torch.empty_like(y, device="cuda")
for name, f in (("h2d 137MB", lambda: dx.copy_(x, non_blocking=True)), ("d2h 100MB", lambda: y.copy_(dy, non_blocking=True))):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        f()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 10
    print(f"{name}: {dt*1e3:.3f} ms  {(x.numel() if 'h2d' in name else y.numel())*8/dt/1e9:.1f} GB/s")

sc = scenes.cfg2()
k = sc.kernels[0]
desc = table1_terms(PolyKernel(k.coefficients, k.normalization)).desc()
dev = torch.device("cuda", 0)
p = torch.from_numpy(sc.particles).to(dev)
t = torch.from_numpy(sc.triangles).to(dev)
ctx = Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
for nch in (1, 2, 4, 8):
    n = p.shape[0] // nch
    ip = torch.from_numpy(sc.pairs[0][:n]).to(dev)
    it = torch.from_numpy(sc.pairs[1][:n]).to(dev)
    ov = torch.empty(n, dtype=torch.float64, device=dev)
    og = torch.empty((n, 2), dtype=torch.float64, device=dev)
    def run():
        _raise(ctx.lib.sphbi_evaluate(ctx.handle, ctypes.byref(desc), sc.h, n, ctypes.c_void_p(p.data_ptr()), t.shape[0],
                                      ctypes.c_void_p(t.data_ptr()), None, n, ctypes.c_void_p(ip.data_ptr()),
                                      ctypes.c_void_p(it.data_ptr()), ctypes.c_void_p(ov.data_ptr()),
                                      ctypes.c_void_p(og.data_ptr()), None, None, None, N.MEM_DEVICE))
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        run()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 10
    print(f"device pipeline, {n} pairs: {dt*1e3:.3f} ms wall  x{nch} = {nch*dt*1e3:.3f} ms")
