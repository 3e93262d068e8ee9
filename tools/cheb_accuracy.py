"""Deviation of the GPU product (Chebyshev coarse far field on) from the
oracle's reference-order product on sampled rows, across shapes, orders and
point sets; also reports the same with IMQ_FAR_NOCHEB semantics absent."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2205_04194_b200 as P
from paper_2205_04194_b200 import inputs
from oracle.oracle import Oracle
o = Oracle()
rng = np.random.default_rng(0)
cases = []
n = 1 << 22
xy = inputs.uniform_points(n, 0)
for p, c in ((4, 0.001), (8, 1e-5), (12, 0.1), (16, 0.01), (20, 1.0), (20, 40.0),
             (20, 0.01), (16, 0.003), (20, 0.001), (16, 1e-5)):
    cases.append((f"uniform 4M L7 p={p} c={c}", xy, c, p, 7))
cases.append(("cfg4 16M L8 p=16 c=0.01", inputs.uniform_points(1 << 24, 0), 0.01, 16, 8))
g = inputs.gaussian_mixture(1 << 20, 1)
cases.append(("gaussian 1M L6 p=14 c=0.02", g, 0.02, 14, 6))
cases.append(("gaussian 1M L7 p=16 c=0.001", g, 0.001, 16, 7))
for name, pts, t, m, L in cases:
    N = pts.size // 2
    u = inputs.random_vector(N, 42)
    op = P.FastOperator(pts, t, m, L)
    b = op.apply(u)
    rows = np.unique(rng.integers(0, N, 200))
    ref = o.fast_matvec_rows(pts, t, m, L, u, rows)
    print(f"{name:36s} rel dev {float(np.max(np.abs(b[rows] - ref)) / np.max(np.abs(ref))):.2e}",
          flush=True)
    op.close()
