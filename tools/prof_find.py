"""Profiling target for the device pair finder (K1-K3) and the evaluation on
cfg5 (16M particles, ~2M triangles, Wendland C2, h = 0.1) or cfg3."""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2507_21686_b200 import scenes  # noqa: E402
from paper_2507_21686_b200 import sphbi as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg5")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
sc = scenes.cfg5() if a.config == "cfg5" else scenes.cfg3()
k = sc.kernels[0]
table = S.table1_terms(S.PolyKernel(list(k.coefficients), k.normalization))
ctx = S.Context(0)
for r in range(a.reps):
    v, g, st = S.evaluate(sc.particles, sc.h, sc.triangles, table, ctx=ctx)
    print(f"rep {r}: pairs {st.n_pairs} ms_pairs {st.ms_pairs:.3f} ms_eval {st.ms_eval:.3f} "
          f"ms_reduce {st.ms_reduce:.3f}", flush=True)
