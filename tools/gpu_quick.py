"""First GPU bring-up: device core vs the compiled reference on random configs."""
import ctypes, math, sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_2507_21686_b200 import sphbi as S

REF = ctypes.CDLL("oracle/_ref/libsphbi_ref.so")
D = ctypes.POINTER(ctypes.c_double)
W4 = np.array([3, 0, -28, 0, 210, -448, 420, -192, 35], dtype=np.float64) / 3.0
C4 = 9 / math.pi
tab = S.table1_terms(S.wendland4())

r = S.integrate_triangle(S.Point2(0.05, -0.03), 0.8, S.Triangle(S.Point2(0.31, -0.12), S.Point2(1.1, 0.55), S.Point2(-0.2, 0.9)), [2.0, -0.5, 1.3], tab)
print("frozen", r, "want 0.205764905431204284 1.31244878196802651 0.992047827773107329", flush=True)

rng = np.random.default_rng(1)
n = 20000
Q = np.zeros((n, 2)); T = np.zeros((n, 6)); V = np.zeros((n, 3)); H = np.zeros(n)
for it in range(n):
    while True:
        t = rng.uniform(-2.2, 2.2, 6)
        a = ((t[2]-t[0])*(t[5]-t[1]) - (t[3]-t[1])*(t[4]-t[0]))/2
        if abs(a) >= 0.05: break
    T[it] = t; V[it] = rng.uniform(-2, 2, 3); Q[it] = rng.uniform(-0.4, 0.4, 2); H[it] = rng.uniform(0.5, 2.0)
worst = 0
for hval in [0.5, 1.0, 2.0]:
    t0 = time.time()
    G = S.integrate_pairs(Q, hval, T, V, tab)
    t1 = time.time()
    R = np.zeros((n, 4))
    for k in range(n):
        REF.sphbi_ref_integrate_triangle(ctypes.c_double(Q[k,0]), ctypes.c_double(Q[k,1]), ctypes.c_double(hval),
            T[k].ctypes.data_as(D), V[k].ctypes.data_as(D), W4.ctypes.data_as(D), 9, ctypes.c_double(C4), R[k:k+1].ctypes.data_as(D))
    tol = np.maximum(1e-11*np.maximum(abs(R[:, :3]), abs(G[:, :3])), 1e-13*C4/hval**2)
    e = (abs(R[:, :3]-G[:, :3])/tol).max()
    worst = max(worst, e)
    print(f"h={hval} gpu {t1-t0:.3f}s worst/tol {e:.4f}", flush=True)
print("counters", S.branch_counters())
print("WORST", worst)
