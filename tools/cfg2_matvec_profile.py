"""Config-2 operator (N = 65,536, c = 0.05, p = 12, L = auto = 2): 3 device
products on one stream, for an ncu launch list (kernel share of a GMRES step)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2205_04194_b200 as P  # noqa: E402
from paper_2205_04194_b200 import inputs  # noqa: E402

xy = inputs.uniform_points(65536, 0)
op = P.FastOperator(xy, 0.05, 12, 0)
u = torch.tensor(inputs.random_vector(65536, 1), device="cuda")
b = torch.empty_like(u)
for _ in range(3):
    op.apply_device(u, b, torch.cuda.current_stream())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(100):
    op.apply_device(u, b, torch.cuda.current_stream())
e1.record()
torch.cuda.synchronize()
print(f"cfg2 product {e0.elapsed_time(e1) / 100 * 1e3:.1f} us, launches {op.stats()['kernel_launches']}")
