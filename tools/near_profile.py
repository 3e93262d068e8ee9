"""Build one operator and run a few fast products (ncu target for the near kernels).

    python tools/near_profile.py N L t M [uniform|cfg3]
"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2205_04194_b200 as P
from paper_2205_04194_b200 import inputs

n, L, t, m = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4])
kind = sys.argv[5] if len(sys.argv) > 5 else "uniform"
xy = inputs.config_points(3, n) if kind == "cfg3" else inputs.uniform_points(n, 0)
op = P.FastOperator(xy, t, m, L)
u = torch.tensor(inputs.random_vector(n, 1000), device="cuda")
b = torch.empty_like(u)
s = torch.cuda.current_stream()
for _ in range(3):
    op.apply_device(u, b, s)
s.synchronize()
print("ok", op.levels, op.stats())
