"""e2e (pinned host buffers) timing of the cfg2 workload for library variants."""
import ctypes, subprocess, sys
code = r'''
import sys, time, ctypes; sys.path.insert(0, '.')
from pathlib import Path
from paper_2507_21686_b200 import _native as N
N.LIB_PATH = Path(LIB)
import numpy as np, torch
from paper_2507_21686_b200 import scenes
from paper_2507_21686_b200.sphbi import Context, PolyKernel, table1_terms, _raise
sc = scenes.cfg2(); k = sc.kernels[0]; desc = table1_terms(PolyKernel(k.coefficients, k.normalization)).desc()
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
P, T, ip, it = pin(sc.particles), pin(sc.triangles), pin(sc.pairs[0]), pin(sc.pairs[1])
n = P.shape[0]; ov = torch.empty(n, dtype=torch.float64).pin_memory(); og = torch.empty((n, 2), dtype=torch.float64).pin_memory()
ctx = Context(0); vp = ctypes.c_void_p
def step():
    _raise(ctx.lib.sphbi_evaluate(ctx.handle, ctypes.byref(desc), sc.h, n, vp(P.data_ptr()), T.shape[0], vp(T.data_ptr()), None, ip.shape[0], vp(ip.data_ptr()), vp(it.data_ptr()), vp(ov.data_ptr()), vp(og.data_ptr()), None, None, None, N.MEM_HOST))
for _ in range(3): step()
ts = []
for _ in range(10):
    t0 = time.perf_counter(); step(); ts.append(time.perf_counter() - t0)
print(LIB, "e2e ms %.3f min %.3f" % (1e3 * sum(ts) / len(ts), 1e3 * min(ts)))
'''
for lib in sys.argv[1:]:
    r = subprocess.run([sys.executable, "-c", code.replace("LIB", repr(lib), 1).replace("Path(LIB)", f"Path({lib!r})")], capture_output=True, text=True)
    print((r.stdout.strip() or r.stderr[-500:]), flush=True)
