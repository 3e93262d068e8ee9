"""Randomised check of the Chebyshev / ring / finest-split paths against the
oracle's reference-order rows: point sets (uniform, clusters, strips, rings,
duplicates), shapes, orders and levels drawn at random (seeded); prints the
worst deviation per case and which paths were active.  Test tool: the oracle
is the checker."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2205_04194_b200 as P
from paper_2205_04194_b200 import inputs
from oracle.oracle import Oracle

o = Oracle()
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
ncase = int(sys.argv[2]) if len(sys.argv) > 2 else 24
worst = 0.0
for c in range(ncase):
    n = int(rng.choice([1 << 17, 1 << 18, 1 << 19, 1 << 20]))
    kind = rng.choice(["uniform", "clusters", "strip", "annulus", "dups"])
    if kind == "uniform":
        xy = rng.random((n, 2))
    elif kind == "clusters":
        k = int(rng.integers(2, 12))
        cen = rng.random((k, 2))
        xy = cen[rng.integers(0, k, n)] + rng.normal(0, rng.uniform(0.01, 0.1), (n, 2))
    elif kind == "strip":
        xy = np.stack([rng.random(n), 0.5 + rng.uniform(0.002, 0.05) * rng.random(n)], 1)
    elif kind == "annulus":
        a = 2 * np.pi * rng.random(n)
        r = 0.3 + 0.05 * rng.random(n)
        xy = np.stack([0.5 + r * np.cos(a), 0.5 + r * np.sin(a)], 1)
    else:
        base = rng.random((n // 4, 2))
        xy = base[rng.integers(0, n // 4, n)]
    xy = np.ascontiguousarray(xy.reshape(-1))
    m = int(rng.choice([4, 6, 8, 10, 12, 14, 16, 18, 20]))
    t = float(10 ** rng.uniform(-4, 0))
    L = int(rng.integers(4, 8))
    if os.environ.get("STRESS_XGATE"):  # t just above the X-ring gate: t / h_X in [5, 5.4]
        m = int(rng.choice([12, 16, 20]))
        pts = xy.reshape(-1, 2)
        side = float(max(np.ptp(pts[:, 0]), np.ptp(pts[:, 1])))
        t = float(rng.uniform(5.0, 5.4) * side / 2 ** (L + 1))
    u = inputs.random_vector(n, 100 + c)
    # STRESS_REPORT=1: the certificate is estimated but not acted on, to
    # compare its estimate with the measured deviation of the swept gates
    op = P.FastOperator(xy, t, m, L, **({"flags": ["cert_report"]} if os.environ.get("STRESS_REPORT") else {}))
    st = op.stats()
    b = op.apply(u)
    rows = np.unique(rng.integers(0, n, 300))
    ref = o.fast_matvec_rows(xy, t, m, L, u, rows)
    err = float(np.max(np.abs(b[rows] - ref)) / np.max(np.abs(ref)))
    worst = max(worst, err)
    extra = ""
    if st["cheb_ring"] and os.environ.get("STRESS_COMPARE"):
        op2 = P.FastOperator(xy, t, m, L, flags=["no_ring"])  # same case without the rings
        b2 = op2.apply(u)
        extra = f"  (no rings: {float(np.max(np.abs(b2[rows] - ref)) / np.max(np.abs(ref))):.2e})"
        op2.close()
    print(f"{c:2d} {kind:8s} n={n:8d} L={L} m={m:2d} t={t:.2e}  cheb={st['cheb_levels']} "
          f"ring={st['cheb_ring']} xring={st['cheb_xring']} near={st['near_mode']}  "
          f"cert {st['cert_estimate']:.1e} [{' '.join(f'{v:.0e}' for v in st['cert_by_kind'])}] "
          f"fb={st['cert_fallbacks']}  dev {err:.2e}{extra}",
          flush=True)
    op.close()
print(f"worst {worst:.2e}")
