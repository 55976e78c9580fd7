"""e2e anatomy of the cfg5 host-memory call: raw PCIe copy times of the step's
buffers next to the sphbi_evaluate(MEM_HOST) call and the device-resident call."""
import ctypes, sys, time
from pathlib import Path
import numpy as np, torch
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2507_21686_b200 import scenes, sphbi as S, _native as N

sc = scenes.cfg5()
k = sc.kernels[0]
table = S.table1_terms(S.PolyKernel(list(k.coefficients), k.normalization))
desc = table.desc()
n, T = sc.particles.shape[0], sc.triangles.shape[0]
dev = torch.device("cuda:0")
p_h = torch.from_numpy(sc.particles).pin_memory()
t_h = torch.from_numpy(sc.triangles).pin_memory()
ov_h = torch.empty(n, dtype=torch.float64).pin_memory()
og_h = torch.empty((n, 2), dtype=torch.float64).pin_memory()
p_d = torch.empty_like(p_h, device=dev); t_d = torch.empty_like(t_h, device=dev)
ov_d = torch.empty(n, dtype=torch.float64, device=dev); og_d = torch.empty((n, 2), dtype=torch.float64, device=dev)
ctx = S.Context(0)
vp = ctypes.c_void_p

def timed(f, reps=5):
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(1e3 * (time.perf_counter() - t0))
    return min(ts)

print("H2D particles+triangles ms", timed(lambda: (p_d.copy_(p_h, non_blocking=True), t_d.copy_(t_h, non_blocking=True))))
print("D2H value+grad ms", timed(lambda: (ov_h.copy_(ov_d, non_blocking=True), og_h.copy_(og_d, non_blocking=True))))
def host():
    S._raise(ctx.lib.sphbi_evaluate(ctx.handle, ctypes.byref(desc), sc.h, n, vp(p_h.data_ptr()), T, vp(t_h.data_ptr()), None, -1, None, None,
                                    vp(ov_h.data_ptr()), vp(og_h.data_ptr()), None, None, None, N.MEM_HOST), "evaluate")
def devc():
    S._raise(ctx.lib.sphbi_evaluate(ctx.handle, ctypes.byref(desc), sc.h, n, vp(p_d.data_ptr()), T, vp(t_d.data_ptr()), None, -1, None, None,
                                    vp(ov_d.data_ptr()), vp(og_d.data_ptr()), None, None, None, N.MEM_DEVICE), "evaluate")
print("evaluate MEM_DEVICE ms", timed(devc))
print("evaluate MEM_HOST ms", timed(host))
stats = N.Stats()
def host_stats():
    S._raise(ctx.lib.sphbi_evaluate(ctx.handle, ctypes.byref(desc), sc.h, n, vp(p_h.data_ptr()), T, vp(t_h.data_ptr()), None, -1, None, None,
                                    vp(ov_h.data_ptr()), vp(og_h.data_ptr()), None, None, ctypes.byref(stats), N.MEM_HOST), "evaluate")
def dev_stats():
    S._raise(ctx.lib.sphbi_evaluate(ctx.handle, ctypes.byref(desc), sc.h, n, vp(p_d.data_ptr()), T, vp(t_d.data_ptr()), None, -1, None, None,
                                    vp(ov_d.data_ptr()), vp(og_d.data_ptr()), None, None, ctypes.byref(stats), N.MEM_DEVICE), "evaluate")
for name, f in (("host", host_stats), ("device", dev_stats)):
    t = timed(f)
    print(name, "total ms", t, "phases: pairs", stats.ms_pairs, "eval", stats.ms_eval, "reduce", stats.ms_reduce)
def host_no_out():
    S._raise(ctx.lib.sphbi_evaluate(ctx.handle, ctypes.byref(desc), sc.h, n, vp(p_h.data_ptr()), T, vp(t_h.data_ptr()), None, -1, None, None,
                                    None, None, None, None, None, N.MEM_HOST), "evaluate")
print("evaluate MEM_HOST without outputs ms", timed(host_no_out))
