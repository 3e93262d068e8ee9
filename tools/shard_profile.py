"""One sharded rank (cfg 4, rank r of `world`, emulated on one GPU): build,
2 warm-up products and 1 measured (ncu target for the sharded launch list)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2205_04194_b200 as P
from paper_2205_04194_b200 import inputs
from paper_2205_04194_b200.parallel import ShardedOperator
world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
rank = int(sys.argv[2]) if len(sys.argv) > 2 else 3
n, t, m, L = 1 << 24, 0.01, 16, 8
xy = inputs.uniform_points(n, 0)
u = torch.tensor(inputs.random_vector(n, 1000), device="cuda")
b = torch.empty_like(u)
sh = ShardedOperator(P.FastOperator(xy, t, m, L), rank, world)
for _ in range(3):
    sh.moments(u, reduce=False); sh.op.moments_finish(); sh.evaluate(b)
torch.cuda.synchronize()
print("ok")
