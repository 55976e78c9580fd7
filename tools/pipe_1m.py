"""One device-resident pipeline call on 1,048,576 cfg2 pairs (launch-list target)."""
import ctypes, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from paper_2507_21686_b200 import _native as N, scenes  # noqa: E402
from paper_2507_21686_b200.sphbi import Context, PolyKernel, _raise, table1_terms  # noqa: E402
sc = scenes.cfg2()
k = sc.kernels[0]
desc = table1_terms(PolyKernel(k.coefficients, k.normalization)).desc()
dev = torch.device("cuda", 0)
n = 1 << 20
p = torch.from_numpy(sc.particles).to(dev)
t = torch.from_numpy(sc.triangles).to(dev)
ip = torch.from_numpy(sc.pairs[0][:n]).to(dev)
it = torch.from_numpy(sc.pairs[1][:n]).to(dev)
ov = torch.empty(n, dtype=torch.float64, device=dev)
og = torch.empty((n, 2), dtype=torch.float64, device=dev)
ctx = Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 4):
    _raise(ctx.lib.sphbi_evaluate(ctx.handle, ctypes.byref(desc), sc.h, n, ctypes.c_void_p(p.data_ptr()), t.shape[0],
                                  ctypes.c_void_p(t.data_ptr()), None, n, ctypes.c_void_p(ip.data_ptr()),
                                  ctypes.c_void_p(it.data_ptr()), ctypes.c_void_p(ov.data_ptr()),
                                  ctypes.c_void_p(og.data_ptr()), None, None, None, N.MEM_DEVICE))
torch.cuda.synchronize()
