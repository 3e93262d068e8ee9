"""One-off config-4 record on the GPU box: the unmodified reference
(oracle/_ref) builds the config-4 operator and applies it once on all host
cores (build and apply timed separately: the same-config CPU baseline, SURVEY
8(d) "for cfg 4, time 1-3 products"); then the GPU product of the same input
is compared with it over the WHOLE vector.  Prints one JSON object."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402

from paper_2205_04194_b200 import inputs  # noqa: E402

n = 1 << 24
xy = inputs.uniform_points(n, 0)
u = inputs.random_vector(n, 1000)
out = {"config": "cfg4: N=16777216 uniform seed 0, c=0.01, p=16, L=8, u=random_vector(N,1000)"}
from oracle import Reference  # noqa: E402
R = Reference()
cores = os.cpu_count()
R.set_threads(cores)
t0 = time.perf_counter()
h = R.create(xy, 0.01, 16, 8)
t1 = time.perf_counter()
b_ref = R.apply(h, u)
t2 = time.perf_counter()
R.destroy(h)
out["reference"] = {"cores": cores, "build_s": t1 - t0, "apply_s": t2 - t1,
                    "points_per_s": n / (t2 - t1)}
print(json.dumps(out), flush=True)
import paper_2205_04194_b200 as P  # noqa: E402
with P.FastOperator(xy, 0.01, 16, 8) as op:
    b = op.apply(u)
    st = op.stats()
scale = np.max(np.abs(b_ref))
d = np.abs(b - b_ref)
out["gpu_vs_reference"] = {"rel_inf": float(d.max() / scale), "argmax": int(d.argmax()),
                           "rel_rms": float(np.sqrt(np.mean(d * d)) / np.sqrt(np.mean(b_ref * b_ref))),
                           "rows_over_1e-13": int(np.sum(d > 1e-13 * scale)),
                           "certificate": st["cert_estimate"]}
g = np.load(os.path.join(ROOT, "tests", "golden", "cfg4_ref.npz"))
out["reference_vs_committed_golden_rows_bitwise"] = bool(np.array_equal(b_ref[g["rows"]], g["b_rows"]))
print(json.dumps(out), flush=True)
