"""Bitwise digests of product-path outputs (regression check between builds):
cfg2 mode A (linear field), cfg5 (first 1M particles, field 1), cfg4 (P3).
Usage: python tools/digest.py [lib.so]   (default: the in-tree library)"""
import hashlib
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2507_21686_b200 import _native as N  # noqa: E402

if len(sys.argv) > 1:
    N.LIB_PATH = Path(sys.argv[1])
from paper_2507_21686_b200 import scenes  # noqa: E402
from paper_2507_21686_b200 import sphbi as S  # noqa: E402


def dig(*arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(a.tobytes())
    return h.hexdigest()[:16]


REPS = 4
ctx = S.Context(0)
for name in ("cfg2a_lin", "cfg5_1m", "cfg4"):
    if name == "cfg2a_lin":
        sc = scenes.cfg2(linear_field=True)
        P, pairs, vals = sc.particles, sc.pairs, sc.values
    elif name == "cfg5_1m":
        sc = scenes.cfg5()
        P, pairs, vals = sc.particles[:1_000_000], None, None
    else:
        sc = scenes.cfg4()
        P, pairs, vals = sc.particles, None, sc.values
    k = sc.kernels[0]
    t = S.table1_terms(S.PolyKernel(list(k.coefficients), k.normalization))
    ms = []
    for _ in range(REPS):
        v, g, st = S.evaluate(P, sc.h, sc.triangles, t, tri_values=vals, pairs=pairs, ctx=ctx)
        ms.append(st.ms_eval)
    print(name, st.n_pairs, dig(v, g), f"{min(ms):.3f} ms eval (min of {REPS})", flush=True)
