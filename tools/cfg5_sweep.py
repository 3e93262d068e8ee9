"""Config 5 (BASELINE.json configs[4]): accuracy / throughput sweep.

N = 4,194,304 uniform points (seed 0), L = 7 (mean 64 per leaf), u =
random_vector(N, 42); p in {4,8,12,16,20} x c in {0.001,0.01,0.1,1.0}.  For
each cell: device time per fast product (CUDA events, 2 warm-up + 5 timed),
relative inf-norm error against the direct product on the 4,096-row subset
i_r = floor(r N / 4096) (direct rows from imq_evaluate_interpolant on the GPU,
checked against the oracle's dense rows on 64 of them), and the deviation from
the oracle's reference-order fast rows (ora_fast_matvec_rows) on the same
subset.  Then the direct O(N^2) product at N = 262,144 (c = 0.01).

Test/measurement tool: the oracle is the checker here, never the timed path.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2205_04194_b200 as P
from paper_2205_04194_b200 import inputs
from oracle.oracle import Oracle


def rel(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


o = Oracle()
n, L = 1 << 22, 7
xy = inputs.uniform_points(n, 0)
u_h = inputs.random_vector(n, 42)
u = torch.tensor(u_h, device="cuda")
b = torch.empty_like(u)
rows = (np.arange(4096) * n) // 4096
qxy = np.ascontiguousarray(xy.reshape(-1, 2)[rows]).reshape(-1)
peak, _ = P.api.fp64_peak(8192)
print(f"# cfg5 sweep: N={n} uniform seed 0, L={L}, u=random_vector(N,42); rows i_r=floor(rN/4096), "
      f"r<4096; FP64 DFMA peak {peak:.1f} TFLOP/s (live probe)")
print("p,c,ms_per_product,Mpoints_per_s,executed_TFLOPs,pipe_frac,err_gpu_vs_dense,"
      "err_oracle_vs_dense,dev_gpu_vs_oracle,gate_ok")
dense = {}
for c in (0.001, 0.01, 0.1, 1.0):
    d = P.evaluate_interpolant(xy, u_h, c, qxy)
    chk = o.dense_matvec(xy, c, u_h, rows[::64])
    assert rel(d[::64], chk) <= 1e-13, c
    dense[c] = d
for p in (4, 8, 12, 16, 20):
    for c in (0.001, 0.01, 0.1, 1.0):
        op = P.FastOperator(xy, c, p, L)
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
        ex = (st["far_pairs_direct"] + st["cheb_node_pairs"]) * 2 * (p * p + 4 * p + 12) \
            + st["near_pairs"] * 5.5
        bh = b.cpu().numpy()[rows]
        ref = o.fast_matvec_rows(xy, c, p, L, u_h, rows)
        e_g, e_o, dev = rel(bh, dense[c]), rel(ref, dense[c]), rel(bh, ref)
        ok = dev <= 1e-10 and np.max(np.abs(bh - dense[c])) <= \
            2 * np.max(np.abs(ref - dense[c])) + 1e-12 * np.max(np.abs(dense[c]))
        print(f"{p},{c},{ms:.3f},{n / ms / 1e3:.1f},{ex / ms / 1e9:.2f},{ex / ms / 1e9 / peak:.3f},"
              f"{e_g:.3e},{e_o:.3e},{dev:.2e},{int(ok)}", flush=True)
        op.close()

nd = 262144
xyd = inputs.uniform_points(nd, 0)
ud = torch.tensor(inputs.random_vector(nd, 42), device="cuda")
P.dense_matvec(xyd, 0.01, ud.cpu().numpy())
t0 = time.perf_counter()
bd = P.dense_matvec(xyd, 0.01, ud.cpu().numpy())
dt = time.perf_counter() - t0
rr = np.arange(0, nd, nd // 64)
print(f"# dense N={nd} c=0.01 (imq_dense_matvec, H2D/D2H included): {dt * 1e3:.2f} ms, "
      f"{float(nd) * nd / dt / 1e12:.3f} Tpairs/s; rel err vs oracle rows "
      f"{rel(bd[rr], o.dense_matvec(xyd, 0.01, ud.cpu().numpy(), rr)):.2e}")
