"""Config-5 sweep timing: N = 4,194,304 uniform, L = 7, p in {4..20}, c = 0.01."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2205_04194_b200 as P
from paper_2205_04194_b200 import inputs
n = 1 << 22
xy = inputs.uniform_points(n, 0)
u = torch.tensor(inputs.random_vector(n, 42), device="cuda")
b = torch.empty_like(u)
for p in (4, 8, 12, 16, 20):
    op = P.FastOperator(xy, 0.01, p, 7)
    for _ in range(2):
        op.apply_device(u, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        op.apply_device(u, b)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    st = op.stats()
    K = (p + 1) * (p + 2) // 2
    Ke = sum(k // 2 + 1 for k in range(p + 1))
    f = st["far_pairs"] * (4 * K + 6 * Ke + 6 * (p + 1) + 12) + st["near_pairs"] * 9
    print(f"p={p:2d}: {ms:7.3f} ms  {n / ms / 1e3:6.1f} Mpts/s  SURVEY-model {f / ms / 1e9:5.1f} TFLOP/s"
          f"  near_mode {st['near_mode']}", flush=True)
    op.close()
