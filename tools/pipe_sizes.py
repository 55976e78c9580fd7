"""Device time (CUDA events on the context's stream) of one sphbi_evaluate call
with device-resident inputs over the first n pairs of the cfg2 workload, for
several n: separates the pipeline's fixed per-call cost from its per-pair cost.
Usage: python tools/pipe_sizes.py [n ...]"""
import ctypes
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2507_21686_b200 import _native as N  # noqa: E402
from paper_2507_21686_b200 import scenes  # noqa: E402
from paper_2507_21686_b200.sphbi import Context, PolyKernel, _raise, table1_terms  # noqa: E402

sizes = [int(a) for a in sys.argv[1:]] or [1 << 16, 1 << 18, 1 << 19, 1 << 20, 1 << 21, 1 << 22]
sc = scenes.cfg2()
k = sc.kernels[0]
desc = table1_terms(PolyKernel(k.coefficients, k.normalization)).desc()
dev = torch.device("cuda", 0)
p = torch.from_numpy(sc.particles).to(dev)
t = torch.from_numpy(sc.triangles).to(dev)
ctx = Context(0)
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)
for n in sizes:
    ip = torch.from_numpy(sc.pairs[0][:n]).to(dev)
    it = torch.from_numpy(sc.pairs[1][:n]).to(dev)
    ov = torch.empty(n, dtype=torch.float64, device=dev)
    og = torch.empty((n, 2), dtype=torch.float64, device=dev)

    def run():
        _raise(ctx.lib.sphbi_evaluate(ctx.handle, ctypes.byref(desc), sc.h, n, ctypes.c_void_p(p.data_ptr()),
                                      t.shape[0], ctypes.c_void_p(t.data_ptr()), None, n,
                                      ctypes.c_void_p(ip.data_ptr()), ctypes.c_void_p(it.data_ptr()),
                                      ctypes.c_void_p(ov.data_ptr()), ctypes.c_void_p(og.data_ptr()), None, None,
                                      None, N.MEM_DEVICE))

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(8):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        run()
        b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    print(f"n={n:8d}  device ms median {ts[len(ts) // 2]:.3f}  min {ts[0]:.3f}  per-Mpair {ts[0] / n * 1e6:.3f}",
          flush=True)
ctx.close()
