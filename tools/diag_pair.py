"""Per-pair parity diagnosis: the pairs of one particle (GPU integrate_pairs vs
the C oracle and the reference build), for a cfg5-reduced scene with a linear field."""
import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import oracle_lib as OL
from paper_2507_21686_b200 import sphbi as S, scenes
O = OL.oracle(); R = OL.ref()
sc = scenes.cfg5(n_particles=60_000, n_discs=6, target_tris=20_000, domain=12.0)
k = sc.kernels[1]
vals = np.random.default_rng(2).standard_normal((sc.triangles.shape[0], 3))
tab = S.table1_terms(S.PolyKernel(list(k.coefficients), k.normalization))
pid = int(sys.argv[1]) if len(sys.argv) > 1 else 21602
pr = OL.cpu_pairs_grid(O, sc.particles, sc.triangles, sc.h)
sel = pr[pr[:, 0] == pid]
q = sc.particles[sel[:, 0]]; t = sc.triangles[sel[:, 1]]; a = vals[sel[:, 1]]
gpu = S.integrate_pairs(q, sc.h, t, a, tab)
st, ora = OL.oracle_pairs(O, np.arange(len(sel)), np.arange(len(sel)), q, t, a, k.coefficients, k.normalization, sc.h)
for j in range(len(sel)):
    _, rr = OL.ref_integrate(R, q[j], sc.h, t[j], a[j], k.coefficients, k.normalization) if R else (0, ora[j])
    d = gpu[j, :3] - rr[:3]
    nv = (t[j].reshape(3, 2) - q[j]) / sc.h
    print(j, sel[j, 1], "gpu", gpu[j, :3], "ref", rr[:3], "diff", d, "oracle-ref", ora[j, :3] - rr[:3])
    print("    nv", nv.ravel().tolist(), "vals", a[j].tolist(), "|v|", np.hypot(nv[:, 0], nv[:, 1]).tolist())
print("sum gpu", gpu[:, :3].sum(0), "sum oracle", ora[:, :3].sum(0))
