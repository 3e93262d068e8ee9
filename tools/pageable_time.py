"""imq_operator_apply with pageable host buffers (what a reference caller
passes), config 4: e2e time per product, a few repeats."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2205_04194_b200 as P
from paper_2205_04194_b200 import inputs
n = 1 << 24
xy = inputs.uniform_points(n, 0)
op = P.FastOperator(xy, 0.01, 16, 8)
us = [inputs.random_vector(n, 1000 + k) for k in range(2)]
b = np.empty(n)
def step(k):
    P.capi.check(P.capi.lib().imq_operator_apply(op.handle, us[k % 2].ctypes.data_as(P.api._dp),
                                                 b.ctypes.data_as(P.api._dp)))
for k in range(3): step(k)
for rep in range(3):
    t0 = time.perf_counter()
    for k in range(10): step(k)
    dt = (time.perf_counter() - t0) / 10
    print(f"pageable e2e {dt * 1e3:.2f} ms per product -> {n / dt / 1e6:.1f} M points/s", flush=True)
print("threads", os.cpu_count())
