import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2205_04194_b200 as P
from paper_2205_04194_b200 import inputs
from oracle.oracle import Oracle
n = 1 << 26
xy = inputs.uniform_points(n, 0)
t0 = time.time(); op = P.FastOperator(xy, 0.01, 16, 9); torch.cuda.synchronize(); print("build", time.time() - t0, op.stats(), flush=True)
u = inputs.random_vector(n, 7)
du = torch.tensor(u, device="cuda"); db = torch.empty_like(du)
op.apply_device(du, db); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); op.apply_device(du, db); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1); print(f"apply {ms:.1f} ms {n/ms/1e3:.1f} Mpts/s", flush=True)
b = db.cpu().numpy()
rows = np.unique(np.random.default_rng(0).integers(0, n, 64))
ref = Oracle().fast_matvec_rows(xy, 0.01, 16, 9, u, rows)
print("err", float(np.max(np.abs(b[rows] - ref)) / np.max(np.abs(ref))))
print("mem GB", torch.cuda.max_memory_allocated() / 1e9)
