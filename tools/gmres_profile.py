"""Config-2 GMRES: a few Arnoldi steps for launch lists / timing."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2205_04194_b200 as P
from paper_2205_04194_b200 import inputs
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 60
xy = inputs.uniform_points(65536, 0)
f = inputs.cfg2_rhs(xy)
op = P.FastOperator(xy, 0.05, 12, 0)
u = torch.tensor(f, device="cuda"); b = torch.empty_like(u)
for _ in range(3): op.apply_device(u, b)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20): op.apply_device(u, b)
torch.cuda.synchronize()
print(f"matvec {1e3*(time.perf_counter()-t0)/20:.3f} ms")
op.solve(f, 1e-8, 10, 50)
t0 = time.perf_counter(); r = op.solve(f, 1e-8, iters, 50); dt = time.perf_counter() - t0
print(f"gmres {iters} its {dt*1e3:.1f} ms -> {dt*1e3/iters:.3f} ms/it, res {r.final_relative_residual:.4e}")
