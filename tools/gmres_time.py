"""Config-2 GMRES(50), 2,000-iteration cap: wall time of imq_ext_iterative_solve."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_04194_b200 as P
from paper_2205_04194_b200 import inputs
xy = inputs.uniform_points(65536, 0)
f = inputs.cfg2_rhs(xy)
with P.FastOperator(xy, 0.05, 12, 0) as op:
    op.solve(f, 1e-8, 100, 50)
    t0 = time.perf_counter()
    r = op.solve(f, 1e-8, 2000, 50)
    dt = time.perf_counter() - t0
print(f"GMRES cfg2: {r.iterations} its in {dt:.3f} s ({dt * 1e3 / r.iterations:.3f} ms/it), "
      f"residual {r.final_relative_residual:.6e}")
