"""e2e (pinned host buffers) wall time of the cfg2 workload through the C-ABI
for one library build: python tools/e2e_probe.py <lib.so>"""
import ctypes
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2507_21686_b200 import _native as N  # noqa: E402

if len(sys.argv) > 1:
    N.LIB_PATH = Path(sys.argv[1])
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_21686_b200 import scenes  # noqa: E402
from paper_2507_21686_b200.sphbi import Context, PolyKernel, _raise, table1_terms  # noqa: E402

sc = scenes.cfg2()
k = sc.kernels[0]
desc = table1_terms(PolyKernel(k.coefficients, k.normalization)).desc()


def pin(a):
    return torch.from_numpy(np.ascontiguousarray(a)).pin_memory()


P, T, ip, it = pin(sc.particles), pin(sc.triangles), pin(sc.pairs[0]), pin(sc.pairs[1])
n = P.shape[0]
ov = torch.empty(n, dtype=torch.float64).pin_memory()
og = torch.empty((n, 2), dtype=torch.float64).pin_memory()
ctx = Context(0)
vp = ctypes.c_void_p


def step():
    _raise(ctx.lib.sphbi_evaluate(ctx.handle, ctypes.byref(desc), sc.h, n, vp(P.data_ptr()), T.shape[0],
                                  vp(T.data_ptr()), None, ip.shape[0], vp(ip.data_ptr()), vp(it.data_ptr()),
                                  vp(ov.data_ptr()), vp(og.data_ptr()), None, None, None, N.MEM_HOST))


for _ in range(3):
    step()
ts = []
for _ in range(10):
    t0 = time.perf_counter()
    step()
    ts.append(time.perf_counter() - t0)
print(N.LIB_PATH.name, "e2e ms mean %.3f min %.3f" % (1e3 * sum(ts) / len(ts), 1e3 * min(ts)), flush=True)
