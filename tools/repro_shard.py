import ctypes, sys
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
b, e = int(sys.argv[1]), int(sys.argv[2])
dev = torch.device("cuda:0")
p_d = torch.from_numpy(np.ascontiguousarray(sc.particles[b:e])).to(dev)
t_d = torch.from_numpy(sc.triangles).to(dev)
m = e - b
buf = torch.zeros(3 * m + 64, dtype=torch.float64, device=dev)
ov, og = buf[:m], buf[m:3 * m].view(m, 2)
ctx = S.Context(0)
vp = ctypes.c_void_p
use_stats = len(sys.argv) > 3
st = N.Stats()
for it in range(3):
    S._raise(ctx.lib.sphbi_evaluate(ctx.handle, ctypes.byref(desc), sc.h, m, vp(p_d.data_ptr()), T, vp(t_d.data_ptr()), None, -1, None, None,
                                    vp(ov.data_ptr()), vp(og.data_ptr()), None, None, ctypes.byref(st) if use_stats else None, N.MEM_DEVICE), "evaluate")
    torch.cuda.synchronize()
    print("ok", it, float(ov.sum()), flush=True)
