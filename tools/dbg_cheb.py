import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2205_04194_b200 as P
from paper_2205_04194_b200 import inputs
from oracle.oracle import Oracle
o = Oracle()
for name, xy, t, m, L in [("uni65k L4", inputs.uniform_points(1 << 16, 0), 0.02, 10, 4),
                          ("uni262k L5", inputs.uniform_points(1 << 18, 0), 0.02, 12, 5),
                          ("gm262k L5", inputs.gaussian_mixture(1 << 18, 1), 0.02, 14, 5),
                          ("gm1M L6", inputs.gaussian_mixture(1 << 20, 1), 0.02, 14, 6)]:
    n = xy.size // 2
    try:
        op = P.FastOperator(xy, t, m, L)
        u = inputs.random_vector(n, 42)
        b = op.apply(u)
        rows = np.unique(np.random.default_rng(0).integers(0, n, 300))
        ref = o.fast_matvec_rows(xy, t, m, L, u, rows)
        print(name, "err", float(np.max(np.abs(b[rows] - ref)) / np.max(np.abs(ref))), flush=True)
    except Exception as e:
        print(name, "FAIL", e, flush=True)
        break
