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
# Chebyshev coarse pass (level-(L-2) boxes >= 600 targets) and sharded ranks
import torch
from paper_2205_04194_b200.parallel import ShardedOperator
big = inputs.uniform_points(120000, 0)
ub = torch.tensor(inputs.random_vector(120000, 3), device="cuda")
with P.FastOperator(big, 0.01, 8, 4) as op:
    assert op.stats()["cheb_levels"] > 0, op.stats()
    bb = torch.empty_like(ub)
    op.apply_device(ub, bb)
    torch.cuda.synchronize()
for r in range(2):
    sh = ShardedOperator(P.FastOperator(big, 0.01, 8, 4), r, 2)
    sh.moments(ub, reduce=False)   # single process: the all-reduce is skipped
    sh.op.moments_finish()
    sh.evaluate(torch.zeros_like(ub))
    torch.cuda.synchronize()
    sh.op.close()
g = inputs.gaussian_mixture(60000, 1)
with P.FastOperator(g, 0.02, 10, 3) as op:   # large leaves: chunk-pair near field
    assert op.stats()["near_mode"] == 2, op.stats()
    op.apply(inputs.random_vector(60000, 4))
print("ok2")
