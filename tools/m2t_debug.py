"""Debug: config-5 corner (p = 4) build under CUDA_LAUNCH_BLOCKING."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_04194_b200 as P  # noqa: E402
from paper_2205_04194_b200 import inputs  # noqa: E402

n = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
p = int(sys.argv[2]) if len(sys.argv) > 2 else 4
xy = inputs.uniform_points(n, 0)
op = P.FastOperator(xy, 0.001, p, 7)
print(op.stats())
