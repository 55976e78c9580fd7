"""Profiling target: one evaluation of a workload through the product path
(sphbi_evaluate), for ncu runs (tools/ncu_fp64.py, launch lists).
  cfg5 [--particles N]: the cfg5 scene (full 2M-triangle mesh), the first N of
                        its 16M uniform particles (a uniform sample of the scene)
  cfg2a:                cfg2 own-triangle pairs (4,194,304 pairs)
Prints one JSON line with the pair count and the device phase times."""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2507_21686_b200 import scenes  # noqa: E402
from paper_2507_21686_b200 import sphbi as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload", choices=["cfg5", "cfg2a", "cfg3", "cfg4"])
ap.add_argument("--particles", type=int, default=0)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
pairs = None
if a.workload == "cfg5":
    sc = scenes.cfg5()
    P = sc.particles[: a.particles] if a.particles else sc.particles
elif a.workload == "cfg2a":
    sc = scenes.cfg2()
    P, pairs = sc.particles, sc.pairs
else:
    sc = scenes.cfg3() if a.workload == "cfg3" else scenes.cfg4()
    P = sc.particles
k = sc.kernels[0]
table = S.table1_terms(S.PolyKernel(list(k.coefficients), k.normalization))
ctx = S.Context(0)
for r in range(a.reps):
    v, g, st = S.evaluate(P, sc.h, sc.triangles, table, tri_values=sc.values, pairs=pairs, ctx=ctx)
    print(json.dumps({"workload": a.workload, "particles": int(P.shape[0]), "pairs": int(st.n_pairs),
                      "ms_pairs": st.ms_pairs, "ms_eval": st.ms_eval, "ms_reduce": st.ms_reduce}), flush=True)
