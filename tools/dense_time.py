"""Times imq_dense_matvec device kernel at config 5's dense point (N=262,144)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2205_04194_b200 as P
from paper_2205_04194_b200 import inputs
n = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
xy = inputs.uniform_points(n, 0); u = inputs.random_vector(n, 42)
P.dense_matvec(xy, 0.01, u)
t0 = time.perf_counter(); b = P.dense_matvec(xy, 0.01, u); dt = time.perf_counter() - t0
pairs = float(n) * n
print(f"dense N={n}: {dt*1e3:.2f} ms incl. H2D/D2H, {pairs/dt/1e12:.3f} Tpairs/s, "
      f"{pairs*9/dt/1e12:.2f} TFLOP/s (SURVEY 9 flop/pair)")
