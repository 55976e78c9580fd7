"""Short profiling target: the cfg2 workload (4,194,304 own-triangle pairs)
through sphbi_evaluate with device-resident inputs, `--reps` times."""
import argparse
import ctypes
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2507_21686_b200 import _native as N  # noqa: E402
from paper_2507_21686_b200 import scenes  # noqa: E402
from paper_2507_21686_b200.sphbi import Context, PolyKernel, _raise, table1_terms  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--config", default="cfg2")
args = ap.parse_args()

if args.config == "cfg2":
    sc = scenes.cfg2()
    pairs = sc.pairs
elif args.config == "cfg3":
    sc = scenes.cfg3()
    pairs = None
else:
    raise SystemExit("unknown config")
k = sc.kernels[0]
desc = table1_terms(PolyKernel(k.coefficients, k.normalization)).desc()
dev = torch.device("cuda", 0)
p = torch.from_numpy(sc.particles).to(dev)
t = torch.from_numpy(sc.triangles).to(dev)
n, T = p.shape[0], t.shape[0]
ov = torch.empty(n, dtype=torch.float64, device=dev)
og = torch.empty((n, 2), dtype=torch.float64, device=dev)
if pairs is not None:
    ip = torch.from_numpy(pairs[0]).to(dev)
    it = torch.from_numpy(pairs[1]).to(dev)
    npairs = ip.shape[0]
ctx = Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
st = N.Stats()
for r in range(args.reps):
    _raise(ctx.lib.sphbi_evaluate(ctx.handle, ctypes.byref(desc), sc.h, n, ctypes.c_void_p(p.data_ptr()), T,
                                  ctypes.c_void_p(t.data_ptr()), None, npairs if pairs is not None else -1,
                                  ctypes.c_void_p(ip.data_ptr()) if pairs is not None else None,
                                  ctypes.c_void_p(it.data_ptr()) if pairs is not None else None,
                                  ctypes.c_void_p(ov.data_ptr()), ctypes.c_void_p(og.data_ptr()), None, None,
                                  ctypes.byref(st), N.MEM_DEVICE))
    print(f"rep {r}: pairs={st.n_pairs} ms_pairs={st.ms_pairs:.3f} ms_eval={st.ms_eval:.3f} "
          f"ms_reduce={st.ms_reduce:.3f}", flush=True)
torch.cuda.synchronize()
ctx.close()
