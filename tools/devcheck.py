"""Dev loop: host-compiled device core vs the compiled reference (oracle/_ref)."""
import ctypes, math, sys
import numpy as np

REF = ctypes.CDLL("oracle/_ref/libsphbi_ref.so")
CORE = ctypes.CDLL("tests/native/_build/libcore_host.so")
D = ctypes.POINTER(ctypes.c_double)

def dp(a):
    return a.ctypes.data_as(D)

W4 = np.array([1, 0, -28/3, 0, 70, -448/3, 140, -64, 35/3], dtype=np.float64)
# exact wendland4 as the reference builds it (integers over 3)
W4 = np.array([3, 0, -28, 0, 210, -448, 420, -192, 35], dtype=np.float64) / 3.0
C4 = 9 / math.pi

def ref_eval(coef, c2, q, h, tri, vals):
    out = np.zeros(4)
    st = REF.sphbi_ref_integrate_triangle(ctypes.c_double(q[0]), ctypes.c_double(q[1]), ctypes.c_double(h),
                                          dp(tri), dp(vals), dp(coef), len(coef), ctypes.c_double(c2), dp(out))
    return st, out

def core_eval(coef, c2, q, h, tri, vals, mode=0):
    out = np.zeros(4 if mode == 0 else 12)
    nreg = ctypes.c_int(0)
    st = CORE.core_host_eval_pair(dp(coef), len(coef), ctypes.c_double(c2), ctypes.c_double(q[0]), ctypes.c_double(q[1]),
                                  ctypes.c_double(h), dp(tri), dp(vals), mode, dp(out), None, ctypes.byref(nreg))
    return st, out

if __name__ == "__main__":
    tri = np.array([0.31, -0.12, 1.1, 0.55, -0.2, 0.9])
    vals = np.array([2.0, -0.5, 1.3])
    print("ref ", ref_eval(W4, C4, (0.05, -0.03), 0.8, tri, vals))
    print("core", core_eval(W4, C4, (0.05, -0.03), 0.8, tri, vals))
    print("want", 0.205764905431204284207329245948, 1.31244878196802651342971672596, 0.992047827773107328591119006664)
    # random invariant-style configs
    rng = np.random.default_rng(1)
    worst = 0
    for it in range(20000):
        while True:
            t = rng.uniform(-2.2, 2.2, 6)
            a = ((t[2]-t[0])*(t[5]-t[1]) - (t[3]-t[1])*(t[4]-t[0]))/2
            if abs(a) >= 0.05: break
        v = rng.uniform(-2, 2, 3); q = rng.uniform(-0.4, 0.4, 2); h = rng.uniform(0.5, 2.0)
        s1, r = ref_eval(W4, C4, q, h, t, v)
        s2, c = core_eval(W4, C4, q, h, t, v)
        tol = np.maximum(1e-11*np.maximum(abs(r[:3]), abs(c[:3])), 1e-13*C4/h**2)
        e = np.max(abs(r[:3]-c[:3])/tol)
        if e > worst:
            worst = e
            print(it, "worst/tol", e, r[:3], c[:3], s1, s2)
    print("done worst", worst)
