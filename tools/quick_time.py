"""Ad-hoc stage timing on one GPU (development aid, not the bench)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2205_04194_b200 as P
from paper_2205_04194_b200 import inputs

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = inputs.CONFIGS[cfg]
n = int(sys.argv[2]) if len(sys.argv) > 2 else c["n"]
t = c["t"] or 0.01
m = c["m"] or 16
xy = inputs.config_points(cfg, n)
t0 = time.time()
op = P.FastOperator(xy, t, m, c["levels"] if n == c["n"] else 0)
torch.cuda.synchronize(); print(f"build {time.time()-t0:.3f}s L={op.levels}", flush=True)
st = op.stats(); print(st, flush=True)
u = torch.tensor(inputs.random_vector(n, 1000), device="cuda")
b = torch.empty_like(u)
s = torch.cuda.current_stream()
perm = torch.tensor(op.permutation().astype(np.int64), device="cuda")
us = u[perm].contiguous()
for _ in range(2): op.apply_device(u, b, s)
s.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(10): op.apply_device(u, b, s)
e1.record(s); s.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"apply {ms:.3f} ms  -> {n/ms*1e3/1e6:.1f} Mpts/s", flush=True)
nf = len(op.items("far")); nn = len(op.items("near"))
e0.record(s); op.moments(us, s); e1.record(s); s.synchronize(); print(f"moments {e0.elapsed_time(e1):.3f} ms")
e0.record(s); op.far_near(us, b, (0, nf), (0, 0), s); e1.record(s); s.synchronize(); tf = e0.elapsed_time(e1); print(f"far {tf:.3f} ms")
e0.record(s); op.far_near(us, b, (0, 0), (0, nn), s); e1.record(s); s.synchronize(); print(f"near {e0.elapsed_time(e1):.3f} ms")
M = m; K = (M+1)*(M+2)//2; Ke = sum(k//2+1 for k in range(M+1))
fpair = 4*K + 6*Ke + 6*(M+1) + 12
print(f"far alg TFLOP/s {st['far_pairs']*fpair/tf/1e9:.2f}; issued ~{st['far_pairs']*2*(M*M+4*M)/tf/1e9:.2f}")
print("fp64 peak", P.api.fp64_peak())
