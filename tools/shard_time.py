"""Per-rank cost of the sharded product, emulated on one GPU (cfg 4 by default):
every rank's moments_local + far/near evaluation timed alone with CUDA events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2205_04194_b200 as P
from paper_2205_04194_b200 import inputs
from paper_2205_04194_b200.parallel import ShardedOperator
world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
n, t, m, L = 1 << 24, 0.01, 16, 8
xy = inputs.uniform_points(n, 0)
u = torch.tensor(inputs.random_vector(n, 1000), device="cuda")
b = torch.empty_like(u)
times = []
for r in range(world):
    sh = ShardedOperator(P.FastOperator(xy, t, m, L), r, world)
    for _ in range(2):
        sh.moments(u, reduce=False); sh.op.moments_finish(); sh.evaluate(b)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record(); sh.moments(u, reduce=False); sh.op.moments_finish(); e[1].record()
    sh.evaluate(b); e[2].record(); torch.cuda.synchronize()
    st = sh.op.stats()
    times.append((e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2])))
    print(f"rank {r}: moments {times[-1][0]:.2f} ms, far+near {times[-1][1]:.2f} ms, "
          f"near_mode {st['near_mode']}", flush=True)
    sh.op.close()
    del sh
    torch.cuda.empty_cache()
print(f"max over ranks {max(a + c for a, c in times):.2f} ms (sum {sum(a + c for a, c in times):.2f} ms)")
