"""Config-2 GMRES protocol (BASELINE config 2): N = 65,536
uniform points, c = 0.05, p = 12, L = auto (2), GMRES(50) from x0 = 0.

* iterations, wall time and final true residual to each tolerance of
  {1e-3, 5e-4, 2e-4} (each a separate solve with the reference's stopping
  rule), plus 1e-8 at the 2,000-iteration cap (not reachable: the reference
  stagnates at 1.058e-4);
* the relative inf-norm difference of the coefficient vector c against the
  reference's own c at matched caps (100 and 2,000 iterations,
  tests/golden/cfg2_ref_it*.npz made by tests/golden/make_golden_big.py);
* --ref: the same tolerance runs through the reference itself (oracle/_ref)
  on this host's cores, timed.

Prints one JSON object.  Test / measurement tool: the reference is the
checker and the CPU baseline, never part of the product path."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402

import paper_2205_04194_b200 as P  # noqa: E402
from paper_2205_04194_b200 import inputs  # noqa: E402

TOLS = (1e-3, 5e-4, 2e-4)
xy = inputs.uniform_points(65536, 0)
f = inputs.cfg2_rhs(xy)
out = {"config": "cfg2: N=65536 uniform seed 0, c=0.05, p=12, L=auto(2), GMRES(50), x0=0"}
with P.FastOperator(xy, 0.05, 12, 0) as op:
    op.solve(f, 1e-8, 50, 50)  # warm-up
    runs = []
    for tol in TOLS + (1e-8,):
        t0 = time.perf_counter()
        r = op.solve(f, tol, 2000, 50)
        dt = time.perf_counter() - t0
        runs.append({"tol": tol, "iterations": r.iterations, "time_s": dt,
                     "ms_per_iteration": dt * 1e3 / max(1, r.iterations),
                     "final_relative_residual": r.final_relative_residual,
                     "converged": r.converged})
    out["gpu"] = runs
    cdiff = {}
    for cap in (100, 2000):
        g = os.path.join(ROOT, "tests", "golden", f"cfg2_ref_it{cap}.npz")
        if not os.path.exists(g):
            continue
        ref = np.load(g)
        r = op.solve(f, 1e-8, cap, 50)
        c_ref = ref["c"]
        cdiff[str(cap)] = {
            "iterations": [r.iterations, int(ref["iterations"])],
            "residual": [r.final_relative_residual, float(ref["res"])],
            "c_rel_inf_diff": float(np.max(np.abs(r.c - c_ref)) / np.max(np.abs(c_ref))),
            "c_rel_2_diff": float(np.linalg.norm(r.c - c_ref) / np.linalg.norm(c_ref)),
            "reference_time_s": float(ref["time_s"]), "reference_threads": int(ref["threads"])}
    out["c_vs_reference"] = cdiff
if "--ref" in sys.argv:
    from oracle import Reference
    R = Reference()
    R.set_threads(os.cpu_count())
    rr = []
    for tol in TOLS:
        t0 = time.perf_counter()
        s = R.iterative_solve(xy, 0.05, 12, 0, f, tol, 2000, 50)
        rr.append({"tol": tol, "iterations": s["iterations"], "time_s": time.perf_counter() - t0,
                   "final_relative_residual": s["final_relative_residual"],
                   "converged": s["converged"]})
    out["reference"] = {"cores": os.cpu_count(), "runs": rr}
print(json.dumps(out))
