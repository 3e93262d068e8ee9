"""One rank of an emulated W-rank sharded config-4 product (default rank 0 of
8), 3 products, for an ncu launch list of the per-rank moments and far/near."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2205_04194_b200 as P
from paper_2205_04194_b200 import inputs
from paper_2205_04194_b200.parallel import ShardedOperator
world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
rank = int(sys.argv[2]) if len(sys.argv) > 2 else 0
n = 1 << 24
xy = inputs.uniform_points(n, 0)
u = torch.tensor(inputs.random_vector(n, 1000), device="cuda")
b = torch.empty_like(u)
sh = ShardedOperator(P.FastOperator(xy, 0.01, 16, 8), rank, world)
for _ in range(3):
    sh.moments(u, reduce=False); sh.op.moments_finish(); sh.evaluate(b)
torch.cuda.synchronize()
print("ok")
