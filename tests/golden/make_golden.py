"""Generates tests/golden/*.npz by running the REFERENCE ITSELF.

    make -C oracle all ref && python tests/golden/make_golden.py

Runs /root/reference/proj compiled unchanged into oracle/_ref/libimqfast_ref.so
(oracle/Makefile) through its own C ABI (imqfast.h).  Only this container has
/root/reference; the fixtures are committed so tests on the GPU box (which has
no reference) can pin both the C oracle and the CUDA product against them.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)
from oracle import Reference  # noqa: E402

from paper_2205_04194_b200 import inputs  # noqa: E402  (pure numpy generators)

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    R = Reference()
    R.set_threads(8)
    cases = {}

    # generator pins: random_vector / halton / auto_level / cost bound
    cases["gen"] = dict(
        rv42=R.random_vector(64, 42), rv0=R.random_vector(64, 0), rv1000=R.random_vector(64, 1000),
        halton=R.halton2d(64),
        auto=np.array([[n, m, R.auto_level(n, m)] for n in (16, 1000, 4096, 20000, 40000, 65536,
                                                           100000, 1048576, 4194304, 16777216)
                       for m in (4, 10, 12, 16, 20)]),
    )

    # config 1 exactly
    xy = R.random_vector(2 * 4096, 0) * 0.5 + 0.5
    u = R.random_vector(4096, 42)
    cases["cfg1"] = dict(xy=xy, u=u, t=0.1, m=10, L=2, b_fast=R.fast_matvec(xy, 0.1, 10, 2, u),
                         b_dense=R.dense_matvec(xy, 0.1, u))

    # test_fastmv.cpp:124-144 families (Halton / random, t, L) at N = 600
    hal = R.halton2d(600)
    rnd = R.random_vector(4000, 7)
    rpts = 0.5 + 0.5 * rnd[:1200]
    u600 = R.random_vector(600, 42)
    fam = {}
    for name, pts in (("halton", hal), ("random", rpts)):
        for t in (0.5, 1.0, 2.0):
            for L in (1, 2):
                fam[f"{name}_t{t}_L{L}"] = R.fast_matvec(pts, t, 10, L, u600)
    cases["family600"] = dict(halton=hal, random=rpts, u=u600, **fam)

    # clustered (config-3 generator, small N), M = 14, L = 3
    cl = inputs.gaussian_mixture(3000, 1)
    ucl = R.random_vector(3000, 42)
    cases["clustered"] = dict(xy=cl, u=ucl, t=0.02, m=14, L=3,
                              b_fast=R.fast_matvec(cl, 0.02, 14, 3, ucl),
                              b_dense=R.dense_matvec(cl, 0.02, ucl))

    # order sweep (config-5 shape, small N): p x c grid at L = 3
    xy5 = R.random_vector(2 * 2048, 0) * 0.5 + 0.5
    u5 = R.random_vector(2048, 42)
    sweep = {}
    for c in (0.001, 0.01, 0.1, 1.0):
        for p in (4, 8, 12, 16, 20):
            sweep[f"c{c}_p{p}"] = R.fast_matvec(xy5, c, p, 3, u5)
    cases["sweep2048"] = dict(xy=xy5, u=u5, b_dense_c0001=R.dense_matvec(xy5, 0.001, u5),
                              b_dense_c1=R.dense_matvec(xy5, 1.0, u5), **sweep)

    # high order (test_solver.cpp uses M = 30), auto L
    h500 = R.halton2d(500)
    u500 = R.random_vector(500, 5)
    cases["highm"] = dict(xy=h500, u=u500, t=0.03, b_m30=R.fast_matvec(h500, 0.03, 30, 0, u500),
                          b_m0=R.fast_matvec(h500, 0.03, 0, 2, u500),
                          b_m1=R.fast_matvec(h500, 0.03, 1, 2, u500))

    # degenerate trees (test_fastmv.cpp:37-41, 98-122)
    same = np.tile([0.3, 0.4], 12)
    u12 = R.random_vector(12, 6)
    cases["degenerate"] = dict(same=same, u12=u12, b_same=R.fast_matvec(same, 0.7, 10, 1, u12),
                               single=R.fast_matvec(np.array([0.3, 0.4]), 2.0, 10, 1,
                                                    np.array([3.0])))

    # GMRES (cli solve default-ish and the config-2 shape at small N)
    h400 = R.halton2d(400)
    f400 = R.random_vector(400, 11)
    s = R.iterative_solve(h400, 0.03, 12, 0, f400, 1e-10, 300, 50)
    xy2 = R.random_vector(2 * 4096, 0) * 0.5 + 0.5
    f2 = inputs.cfg2_rhs(xy2)
    s2 = R.iterative_solve(xy2, 0.05, 12, 0, f2, 1e-8, 100, 50)
    cases["gmres"] = dict(xy400=h400, f400=f400, c400=s["c"], it400=s["iterations"],
                          res400=s["final_relative_residual"], conv400=s["converged"],
                          xy2=xy2, f2=f2, c2=s2["c"], it2=s2["iterations"],
                          res2=s2["final_relative_residual"], conv2=s2["converged"])

    for k, v in cases.items():
        np.savez_compressed(os.path.join(OUT, f"{k}.npz"), **v)
        print(k, os.path.getsize(os.path.join(OUT, f"{k}.npz")))


if __name__ == "__main__":
    main()
