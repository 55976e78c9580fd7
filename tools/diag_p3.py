"""P3 path diagnosis: GPU (sphbi_integrate_pairs_p3) vs the host build of the
device core (core_host_eval_pair_p3) on simple routes."""
import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, ctypes
import oracle_lib as OL
from paper_2507_21686_b200 import sphbi as S
C = OL.core()
tab = S.table1_terms(S.wendland4())
coef = np.array(tab.kernel.coefficients if hasattr(tab, "kernel") else OL.W4); c2 = OL.C4
def host(q, h, tri, nodes):
    o = np.zeros(4)
    C.core_host_eval_pair_p3(OL.ptr(coef), coef.shape[0], c2, q[0], q[1], h, OL.ptr(OL.arr(tri)), OL.ptr(OL.arr(nodes)), OL.ptr(o))
    return o
cases = {
 "disc": (np.array([0.0, 0.0]), 1.0, np.array([-5, -5, 5, -5, 0, 5.0])),
 "wedge1": (np.array([0.0, 0.0]), 1.0, np.array([0.2, 0.1, 3, 0.3, 0.4, 2.5])),
 "t2": (np.array([0.0, 0.0]), 1.0, np.array([0.2, 0.1, 0.5, 0.3, 0.4, 2.5])),
 "t3": (np.array([0.0, 0.0]), 1.0, np.array([0.2, 0.1, 0.5, 0.3, 0.1, 0.5])),
 "outside": (np.array([0.0, 0.0]), 1.0, np.array([0.9, -2, 1.5, 2, 3, 0.0])),
}
for nm, (q, h, tri) in cases.items():
    for fn, nodes in (("one", np.ones(10)), ("x", OL.p3_nodes_from_poly(tri, lambda x, y: x)), ("xy2", OL.p3_nodes_from_poly(tri, lambda x, y: x * y * y + 0.3))):
        g = S.integrate_pairs_p3(q[None], h, tri[None], nodes[None], tab)[0]
        hh = host(q, h, tri, nodes)
        print(f"{nm:8s} {fn:4s} gpu {g[:3]} host {hh[:3]} diff {np.abs(g[:3]-hh[:3]).max():.3g}")
