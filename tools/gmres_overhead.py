"""Where does a GMRES step's time go at config 2?  (development aid)"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2205_04194_b200 as P
from paper_2205_04194_b200 import inputs
xy = inputs.uniform_points(65536, 0)
f = inputs.cfg2_rhs(xy)
op = P.FastOperator(xy, 0.05, 12, 0)
u = torch.tensor(f, device="cuda"); b = torch.empty_like(u)
for _ in range(5): op.apply_sorted_device(u, b)
torch.cuda.synchronize()
n = 100
t0 = time.perf_counter()
for _ in range(n): op.apply_sorted_device(u, b)
t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"batched: enqueue {1e3*(t1-t0)/n:.3f} ms/apply, total {1e3*(t2-t0)/n:.3f} ms/apply")
t0 = time.perf_counter()
for _ in range(n):
    op.apply_sorted_device(u, b); torch.cuda.synchronize()
print(f"apply+sync: {1e3*(time.perf_counter()-t0)/n:.3f} ms")
h = torch.empty(64, dtype=torch.float64).pin_memory()
t0 = time.perf_counter()
for _ in range(n):
    op.apply_sorted_device(u, b); h[:1].copy_(b[:1], non_blocking=True); torch.cuda.synchronize()
print(f"apply+d2h+sync: {1e3*(time.perf_counter()-t0)/n:.3f} ms")
