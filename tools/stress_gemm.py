"""Randomised check of the tensor-core node passes (k_node_gemm, TMA-staged)
against the oracle's reference-order rows: large point sets (uniform, clusters,
annulus, strip, duplicates -- empty and clipped boxes, partial 32-box tiles),
shapes around the ring / X-ring gates, orders 8..20; prints which passes ran
as GEMMs (gemm_node_pairs) and the worst deviation.  Test tool: the oracle is
the checker."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2205_04194_b200 as P
from paper_2205_04194_b200 import inputs
from oracle.oracle import Oracle

o = Oracle()
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
ncase = int(sys.argv[2]) if len(sys.argv) > 2 else 16
worst, ngemm = 0.0, 0
for c in range(ncase):
    n = int(rng.choice([1 << 21, 1 << 22, 3 << 21]))
    kind = rng.choice(["uniform", "clusters", "strip", "annulus", "dups"])
    if kind == "uniform":
        xy = rng.random((n, 2))
    elif kind == "clusters":
        k = int(rng.integers(3, 12))
        cen = rng.random((k, 2))
        xy = cen[rng.integers(0, k, n)] + rng.normal(0, rng.uniform(0.05, 0.2), (n, 2))
    elif kind == "strip":
        xy = np.stack([rng.random(n), 0.5 + rng.uniform(0.2, 0.6) * rng.random(n)], 1)
    elif kind == "annulus":
        a = 2 * np.pi * rng.random(n)
        r = 0.25 + 0.2 * rng.random(n)
        xy = np.stack([0.5 + r * np.cos(a), 0.5 + r * np.sin(a)], 1)
    else:
        base = rng.random((n // 4, 2))
        xy = base[rng.integers(0, n // 4, n)]
    xy = np.ascontiguousarray(xy.reshape(-1))
    pts = xy.reshape(-1, 2)
    side = float(max(np.ptp(pts[:, 0]), np.ptp(pts[:, 1])))
    L = int(rng.choice([7, 8]))
    m = int(rng.choice([8, 12, 16, 20]))
    hx = side / 2 ** L  # width of the level-(L-1) boxes
    t = float(rng.choice([0.8, 1.5, 2.2, 3.0, 5.2, 8.0]) * rng.uniform(0.9, 1.1) * hx)
    if os.environ.get("STRESS_X"):  # X-node GEMM on: L = 7, t / h_X in [5.05, 13]
        L = 7
        hx = side / 2 ** L
        t = float(rng.uniform(5.05, 13.0) * hx)
    u = inputs.random_vector(n, 300 + c)
    op = P.FastOperator(xy, t, m, L)
    st = op.stats()
    b = op.apply(u)
    rows = np.unique(rng.integers(0, n, 200))
    ref = o.fast_matvec_rows(xy, t, m, L, u, rows)
    err = float(np.max(np.abs(b[rows] - ref)) / np.max(np.abs(ref)))
    worst = max(worst, err)
    ngemm += st["gemm_node_pairs"] > 0
    print(f"{c:2d} {kind:8s} n={n:8d} L={L} m={m:2d} t={t:.2e} (t/hX {t / hx:.2f})  "
          f"cheb={st['cheb_levels']} ring={st['cheb_ring']} xring={st['cheb_xring']} "
          f"gemm_pairs={st['gemm_node_pairs']:.3g} of {st['cheb_node_pairs']:.3g}  "
          f"cert {st['cert_estimate']:.1e} fb={st['cert_fallbacks']}  dev {err:.2e}", flush=True)
    op.close()
print(f"worst {worst:.2e}; {ngemm} of {ncase} cases ran GEMM passes")
