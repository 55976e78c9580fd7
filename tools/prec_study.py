"""Precision study of the constant-field FP64 path (CPU only; host build of the
device core): per pair and per particle, FP64 (piece_*3f) vs double-double
(piece_*3) vs the compiled reference, in units of the parity tolerance.

    python tools/prec_study.py [cfg1 cfg2a cfg2b cfg3 cfg5 ...]

Prints, per configuration: kappa = sum |b_k|, the worst per-pair
difference FP64 - dd in the unit-disc frame as a multiple of u * kappa (the
constant of fp64_path_ok), and the per-particle parity ratios of both paths
against the reference.
"""
import ctypes
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import oracle_lib as OL  # noqa: E402
from paper_2507_21686_b200 import scenes  # noqa: E402

P, D, I64 = ctypes.c_void_p, ctypes.c_double, ctypes.c_int64
U = 2.0 ** -53
FAST = 2  # 1: FP64 piece kernels' math, 2: the FP64 edge form (the product's FP64 path)


def f1(C, pp, pt, pxy, tri, coef, c2, h, fast, decomp=2, threads=16):
    pp = OL.arr(pp, np.int64)
    pt = OL.arr(pt, np.int64)
    out = np.zeros((pp.shape[0], 3))
    c = OL.arr(coef)
    C.core_host_eval_pairs_f1.argtypes = [I64, P, P, P, P, P, ctypes.c_int, D, D, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_int, P]
    C.core_host_eval_pairs_f1(pp.shape[0], OL.ptr(pp), OL.ptr(pt), OL.ptr(OL.arr(pxy)), OL.ptr(OL.arr(tri)),
                              OL.ptr(c), c.shape[0], c2, h, threads, decomp, fast, OL.ptr(out))
    return out


def sums(n, pp, pt, out):
    order = np.lexsort((pt, pp))
    acc = np.zeros((n, 3))
    for c in range(3):  # ascending triangle id per particle, sequential adds
        np.add.at(acc[:, c], pp[order], out[order, c])
    return acc


def study(name, sc, O, R, C, max_pairs=None, ref_check=True):
    k = sc.kernels[0]
    coef, c2, h = list(k.coefficients), k.normalization, sc.h
    if sc.pairs is not None:
        pp, pt = sc.pairs
    else:
        pl = OL.cpu_pairs_grid(O, sc.particles, sc.triangles, h, cap=60_000_000)
        pp, pt = pl[:, 0].copy(), pl[:, 1].copy()
    if max_pairs and pp.shape[0] > max_pairs:
        pp, pt = pp[:max_pairs], pt[:max_pairs]
    C.core_host_kappa.restype = D
    C.core_host_kappa.argtypes = [P, ctypes.c_int]
    ca = OL.arr(coef)
    kappa = C.core_host_kappa(OL.ptr(ca), ca.shape[0])
    t0 = time.time()
    a = f1(C, pp, pt, sc.particles, sc.triangles, coef, c2, h, 0)
    t1 = time.time()
    b = f1(C, pp, pt, sc.particles, sc.triangles, coef, c2, h, FAST)
    t2 = time.time()
    # unit-disc frame: value / C2, gradient * h / C2
    scale = np.array([1.0 / c2, h / c2, h / c2])
    dn = abs(a - b) * scale
    worst = dn.max()
    n = sc.particles.shape[0]
    rows = np.bincount(pp, minlength=n)
    sa, sb = sums(n, pp, pt, a), sums(n, pp, pt, b)
    tol = np.maximum(1e-11 * np.maximum(abs(sa), abs(sb)), 1e-13 * abs(c2) / h ** 2)
    r_ab = (abs(sa - sb) / tol).max()
    line = (f"{name:8s} pairs {pp.shape[0]:9d} max_row {rows.max():6d} kappa {kappa:9.1f}  per-pair |f64-dd| "
            f"{worst:.2e} = {worst / (U * kappa):6.2f} u kappa  per-particle f64 vs dd {r_ab:.4f} tol"
            f"  (dd {t1 - t0:.1f}s f64 {t2 - t1:.1f}s)")
    if ref_check and R is not None:
        vals = np.ones((sc.triangles.shape[0], 3))
        out = np.zeros((pp.shape[0], 4))
        fail = I64(-1)
        ppc, ptc = OL.arr(pp, np.int64), OL.arr(pt, np.int64)
        R.sphbi_ref_eval_pairs(ppc.shape[0], OL.ptr(ppc), OL.ptr(ptc), OL.ptr(OL.arr(sc.particles)),
                               OL.ptr(OL.arr(sc.triangles)), OL.ptr(vals), OL.ptr(ca), ca.shape[0], c2, h, 16,
                               OL.ptr(out), ctypes.byref(fail))
        sr = sums(n, pp, pt, out[:, :3])
        ra = max(OL.parity_ratio(sa[:, 0], sr[:, 0], c2, h), OL.parity_ratio(sa[:, 1:], sr[:, 1:], c2, h))
        rb = max(OL.parity_ratio(sb[:, 0], sr[:, 0], c2, h), OL.parity_ratio(sb[:, 1:], sr[:, 1:], c2, h))
        line += f"  vs reference: dd {ra:.4f}  f64 {rb:.4f}"
    print(line, flush=True)


def main():
    which = sys.argv[1:] or ["cfg1", "cfg2a", "cfg3", "cfg5", "cfg2b"]
    O, R, C = OL.oracle(), OL.ref(), OL.core()
    for w in which:
        if w == "cfg1":
            study(w, scenes.cfg1(), O, R, C)
        elif w == "cfg2a":
            study(w, scenes.cfg2(T=8192), O, R, C)
        elif w == "cfg2b":
            sc = scenes.cfg2()
            sub = scenes.subsample(sc, 64, seed=7)
            sub.pairs = None
            study(w, sub, O, R, C)
        elif w == "cfg3":
            study(w, scenes.cfg3(), O, R, C)
        elif w == "cfg5":
            sc = scenes.cfg5(n_particles=400_000, n_discs=20, target_tris=80_000, domain=20.0)
            study(w, sc, O, R, C)
        elif w == "rand":
            # the reference suites' random configurations (h in [0.5, 2], Wendland C4)
            rng = np.random.default_rng(31337)
            n = 20000
            tri = np.zeros((n, 6))
            q = np.zeros((n, 2))
            for i in range(n):
                t, v, qq, hh = OL.random_config(rng)
                tri[i], q[i] = t, qq
            for hh in (0.5, 1.0, 2.0):
                sc = scenes.Scene("rand", q, tri, None, [scenes.wendland_c4()], hh,
                                  pairs=(np.arange(n, dtype=np.int64), np.arange(n, dtype=np.int64)))
                study(f"rand h={hh}", sc, O, R, C)


if __name__ == "__main__":
    main()
