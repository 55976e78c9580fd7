"""cfg4 (P3 field) timing on the device: full scene through the cell list."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_2507_21686_b200 import sphbi as S, scenes

sc = scenes.cfg4()
k = sc.kernels[0]
table = S.table1_terms(S.PolyKernel(list(k.coefficients), k.normalization))
ctx = S.Context(0)
import os
for it in range(int(os.environ.get("REPS", "4"))):
    t0 = time.time()
    v, g, st = S.evaluate(sc.particles, sc.h, sc.triangles, table, tri_values=sc.values, ctx=ctx)
    t1 = time.time()
    print(f"cfg4 particles {sc.particles.shape[0]} pairs {st.n_pairs} ms_pairs {st.ms_pairs:.3f} "
          f"ms_eval {st.ms_eval:.3f} ms_reduce {st.ms_reduce:.3f} wall {1e3*(t1-t0):.1f} ms "
          f"-> {st.n_pairs/(st.ms_eval*1e-3)/1e6:.2f} M pair-evals/s (eval)", flush=True)
