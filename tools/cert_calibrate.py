"""Certificate calibration: for the bench configuration and the full-vector
test cases, the certificate's estimate (per interpolation kind) beside the
measured whole-vector (N <= 1M) or sampled-row deviation from the oracle, with
the certificate in report-only mode (the swept gates alone).  Test tool: the
oracle is the checker."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2205_04194_b200 as P
from paper_2205_04194_b200 import inputs
from oracle.oracle import Oracle

o = Oracle()
N1 = 1 << 20
cases = [("cfg4", inputs.uniform_points(1 << 24, 0), 0.01, 16, 8, 1000, "rows"),
         ("cfg3", inputs.gaussian_mixture(N1, 1), 0.02, 14, 6, 42, "full"),
         ("u1m_nodes", inputs.uniform_points(N1, 0), 0.001, 16, 6, 42, "full"),
         ("u1m_rings", inputs.uniform_points(N1, 0), 0.02, 16, 6, 42, "full"),
         ("u1m_cfg4mix", inputs.uniform_points(N1, 0), 0.04, 16, 6, 42, "full"),
         ("gate1.27", inputs.uniform_points(N1, 3), 1.27 / 64, 20, 6, 5, "full"),
         ("gate2.55", inputs.uniform_points(N1, 3), 2.55 / 64, 20, 6, 5, "full"),
         ("gate5.2", inputs.uniform_points(N1, 3), 5.2 / 128, 20, 6, 5, "full")]
only = sys.argv[1:]
for name, xy, t, m, L, seed, mode in cases:
    if only and name not in only:
        continue
    n = xy.size // 2
    u = inputs.random_vector(n, seed)
    op = P.FastOperator(xy, t, m, L, flags=["cert_report"])
    st = op.stats()
    b = op.apply(u)
    op.close()
    t0 = time.time()
    if mode == "full":
        ref = o.fast_matvec(xy, t, m, L, u)
        dev = float(np.max(np.abs(b - ref)) / np.max(np.abs(ref)))
    else:
        rows = (np.arange(4096) * n) // 4096
        ref = o.fast_matvec_rows(xy, t, m, L, u, rows)
        dev = float(np.max(np.abs(b[rows] - ref)) / np.max(np.abs(ref)))
    kinds = " ".join(f"{v:.1e}" for v in st["cert_by_kind"])
    print(f"{name:12s} cheb={st['cheb_levels']} ring={st['cheb_ring']} xring={st['cheb_xring']} "
          f"est {st['cert_estimate']:.2e} [nodes inner ring ring2 xring: {kinds}]  dev {dev:.2e} ({mode}, "
          f"oracle {time.time() - t0:.0f}s)", flush=True)
