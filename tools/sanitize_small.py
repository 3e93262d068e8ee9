"""Small end-to-end run for compute-sanitizer (memcheck / racecheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2205_04194_b200 as P
from paper_2205_04194_b200 import inputs
xy = inputs.uniform_points(3000, 0); u = inputs.random_vector(3000, 1)
for m, L in ((16, 3), (12, 2), (30, 2), (0, 1)):
    with P.FastOperator(xy, 0.05, m, L) as op:
        b = op.apply(u)
        r = op.solve(u, 1e-6, 30, 10)
cl = inputs.gaussian_mixture(5000, 1)
with P.FastOperator(cl, 0.02, 14, 4) as op:
    op.apply(inputs.random_vector(5000, 2))
P.dense_matvec(xy, 0.1, u)
print("ok", float(np.abs(b).max()))
