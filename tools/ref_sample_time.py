"""Sampled timing of the reference's own per-stage routines at a large
configuration (oracle/ref_sample.cpp): prints the estimated full-product time
and the raw stage times.  Measurement tool (the reference is the CPU baseline).

    python tools/ref_sample_time.py [N L n_mom n_tgt threads repeats]
"""
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2205_04194_b200 import inputs  # noqa: E402

a = [int(x) for x in sys.argv[1:]]
n, L, nm, nt, th, rep = (a + [1 << 24, 8, 4096, 4096, os.cpu_count(), 3][len(a):])[:6]
lib = C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libimqfast_ref.so"))
dp = C.POINTER(C.c_double)
f = lib.imqref_sample_time
f.argtypes = [dp, C.c_longlong, C.c_double, C.c_int, C.c_int, dp, C.c_int, C.c_int, C.c_ulonglong,
              C.c_int, dp]
xy = inputs.uniform_points(n, 0)
u = inputs.random_vector(n, 1000)
res = []
for k in range(rep):
    out = np.zeros(7)
    t0 = time.perf_counter()
    assert f(xy.ctypes.data_as(dp), n, 0.01, 16, L, u.ctypes.data_as(dp), nm, nt, 7 + k, th,
             out.ctypes.data_as(dp)) == 0
    res.append({"wall_s": time.perf_counter() - t0, "t_moments": out[0], "t_far": out[1],
                "t_near": out[2], "moment_points": out[3], "targets": out[4], "far_pairs": out[5],
                "est_full_s": out[6], "est_points_per_s": n / out[6]})
print(json.dumps({"n": n, "L": L, "threads": th, "samples": res}))
