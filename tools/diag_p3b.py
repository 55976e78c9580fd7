import sys; sys.path.insert(0, ".")
from pathlib import Path
from paper_2507_21686_b200 import _native as N
N.LIB_PATH = Path("_variants/dbg.so")
import numpy as np
from paper_2507_21686_b200 import sphbi as S
tab = S.table1_terms(S.wendland4())
tri = np.array([-5, -5, 5, -5, 0, 5.0])
print(S.integrate_pairs_p3(np.zeros((1, 2)), 1.0, tri[None], np.ones((1, 10)), tab)[0], flush=True)
