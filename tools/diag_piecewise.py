import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import oracle_lib as OL
from paper_2507_21686_b200 import sphbi as S, scenes
O = OL.oracle()
sc = scenes.cfg5(n_particles=60_000, n_discs=6, target_tris=20_000, domain=12.0)
ks = sc.kernels[1:]
vals = np.random.default_rng(2).standard_normal((sc.triangles.shape[0], 3))
tab = lambda k: S.table1_terms(S.PolyKernel(list(k.coefficients), k.normalization))
v, g, st = S.evaluate_piecewise(sc.particles, sc.h, sc.triangles, [(tab(k), k.support_scale) for k in ks], tri_values=vals)
tot_o = np.zeros((sc.particles.shape[0], 3)); tot_g = np.zeros_like(tot_o)
for k in ks:
    h = sc.h * k.support_scale
    pr = OL.cpu_pairs_grid(O, sc.particles, sc.triangles, h)
    s_, vo, go = OL.oracle_scene_sums(O, sc.particles, sc.triangles, vals, k.coefficients, k.normalization, h, pr[:, 0], pr[:, 1], threads=16)
    a, b, _ = S.evaluate(sc.particles, h, sc.triangles, tab(k), tri_values=vals)
    want = np.c_[vo, go]; got = np.c_[a, b]
    print(k.name, "piece ratio (own h floor)", OL.parity_ratio(got, want, k.normalization, h), "ratio w/ cfg floor", OL.parity_ratio(got, want, ks[0].normalization, sc.h))
    tot_o += want; tot_g += got
one = np.c_[v, g]
print("onepass vs oracle", OL.parity_ratio(one, tot_o, ks[0].normalization, sc.h))
print("twopass gpu vs oracle", OL.parity_ratio(tot_g, tot_o, ks[0].normalization, sc.h))
print("onepass vs twopass", OL.parity_ratio(one, tot_g, ks[0].normalization, sc.h))
tol = np.maximum(1e-11*np.maximum(abs(one), abs(tot_o)), 1e-13*ks[0].normalization/sc.h**2)
r = abs(one - tot_o)/tol
i, c = np.unravel_index(np.argmax(r), r.shape)
print("worst", i, c, one[i], tot_o[i], tot_g[i], r[i])
