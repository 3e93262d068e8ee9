"""Full-size goldens made by running the REFERENCE ITSELF (test infrastructure).

    make -C oracle all ref && python tests/golden/make_golden_big.py cfg4 [--full-out PATH]
    python tests/golden/make_golden_big.py cfg2

cfg4: /root/reference/proj compiled unchanged (oracle/_ref/libimqfast_ref.so)
builds the config-4 operator (N = 16,777,216 uniform seed 0, c = 0.01, p = 16,
L = 8; ~37 GB of trig cache) and applies it once to u = random_vector(N, 1000)
(`fastmv.cpp:184-217` through `capi.cpp:130-138`).  The whole vector is too
big to commit (134 MB), so the committed fixture `cfg4_ref.npz` pins it by

* 65,536 rows b[r*N/65536] (r = 0..65535), stored exactly;
* per-chunk checksums over 4,096 contiguous chunks of 4,096 rows (original
  order): sum b, sum |b|, sum b^2 -- a GPU vector that differs anywhere by
  more than ~1e-12 relative moves at least one chunk checksum;
* global fingerprints (b[0], b[N-1], sum, sum|b|, max|b|) and the reference's
  build / apply wall times on this container's cores.

`--full-out` also writes the whole vector (float64 .npy, git-ignored) for a
one-off full-vector comparison.

cfg2: GMRES(50) on config 2 (N = 65,536, c = 0.05, p = 12, L = auto = 2,
x0 = 0, tol 1e-8) capped at 100 iterations; the coefficient vector c and the
residual are stored (`solver.cpp:41-159`), for the coefficient-difference
check BASELINE config 2 asks for.
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)
from oracle import Reference  # noqa: E402

from paper_2205_04194_b200 import inputs  # noqa: E402  (pure numpy generators)

OUT = os.path.dirname(os.path.abspath(__file__))
CHUNK = 4096


def checksums(b):
    c = b.reshape(-1, CHUNK)
    return np.sum(c, axis=1), np.sum(np.abs(c), axis=1), np.sum(c * c, axis=1)


def cfg4(full_out=None, threads=None):
    R = Reference()
    R.set_threads(threads or os.cpu_count())
    n = 1 << 24
    xy = inputs.uniform_points(n, 0)
    u = inputs.random_vector(n, 1000)
    t0 = time.perf_counter()
    h = R.create(xy, 0.01, 16, 8)
    t1 = time.perf_counter()
    b = R.apply(h, u)
    t2 = time.perf_counter()
    R.destroy(h)
    rows = (np.arange(65536, dtype=np.int64) * n) // 65536
    s, sa, s2 = checksums(b)
    np.savez_compressed(os.path.join(OUT, "cfg4_ref.npz"), rows=rows, b_rows=b[rows],
                        chunk_sum=s, chunk_abs=sa, chunk_sq=s2,
                        fp=np.array([b[0], b[-1], b.sum(), np.abs(b).sum(), np.abs(b).max()]),
                        build_s=t1 - t0, apply_s=t2 - t1, threads=threads or os.cpu_count())
    if full_out:
        np.save(full_out, b)
    print(f"cfg4: build {t1 - t0:.1f} s, apply {t2 - t1:.1f} s, b[0]={b[0]!r}")


def cfg2(cap=100):
    R = Reference()
    R.set_threads(os.cpu_count())
    xy = inputs.uniform_points(65536, 0)
    f = inputs.cfg2_rhs(xy)
    t0 = time.perf_counter()
    s = R.iterative_solve(xy, 0.05, 12, 0, f, 1e-8, cap, 50)
    dt = time.perf_counter() - t0
    np.savez_compressed(os.path.join(OUT, f"cfg2_ref_it{cap}.npz"), c=s["c"],
                        iterations=s["iterations"], res=s["final_relative_residual"],
                        converged=s["converged"], time_s=dt, threads=os.cpu_count())
    print(f"cfg2: {s['iterations']} its, res {s['final_relative_residual']:.6e}, {dt:.1f} s")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["cfg4", "cfg2"])
    ap.add_argument("--full-out", default=None)
    ap.add_argument("--threads", type=int, default=None)
    ap.add_argument("--cap", type=int, default=100)
    a = ap.parse_args()
    if a.what == "cfg4":
        cfg4(a.full_out, a.threads)
    else:
        cfg2(a.cap)
