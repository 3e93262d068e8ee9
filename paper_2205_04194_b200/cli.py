"""Command-line harness over the C ABI.

    python -m paper_2205_04194_b200.cli --mode verify|bench|errtrend|solve [...]

Same modes, flags and CSV / '# config:' output schema as the reference CLI
(/root/reference/proj/tools/cli_main.cpp:82-90 config line, 139-185 bench,
186-215 errtrend, 217-284 solve, 288-304 flags), so runs of the two can be
compared line by line.  Everything is computed by libimqfast.so on the GPU.
"""
from __future__ import annotations

import argparse
import math
import sys
import time

import numpy as np

from . import api
from .capi import IMQError


def _levels(s: str) -> int:
    if s == "auto":
        return 0
    try:
        L = int(s)
    except ValueError:
        L = 0
    if L < 1:
        raise ValueError("--levels must be 'auto' or an integer >= 1")
    return L


def _ns(s: str, default):
    return [int(x) for x in s.split(",")] if s else list(default)


def _points(opt, n):
    return api.read_points(opt.points) if opt.points else api.halton2d(n)


def _g(x: float) -> str:
    """printf %g-like formatting (the reference streams doubles with defaults)."""
    return f"{x:g}"


def _config(opt, n_eff) -> str:
    line = (f"# config: mode={opt.mode} n={n_eff} t={_g(opt.t)} m={opt.m} levels={opt.levels} "
            f"seed={opt.seed} points={opt.points or '-'} "
            f"threads={opt.threads if opt.threads > 0 else 'default'}")
    if opt.mode == "solve":
        line += f" tol={_g(opt.tol)} max_iter={opt.max_iter} restart={opt.restart}"
    return line


def _rel_inf(a, b) -> float:
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / np.max(np.abs(b)))


def run_verify(opt, out) -> int:
    n = _ns(opt.n, [2000])[0]
    xy = _points(opt, n)
    n = xy.size // 2
    print(_config(opt, n), file=out)
    fails, rows = api.verify(xy, opt.t, opt.m, _levels(opt.levels), opt.seed)
    for name, ok, value in rows:
        print(f"[{'PASS' if ok else 'FAIL'}] {name} = {value:.6e}", file=out)
    print(f"# verify: {fails} of {len(rows)} checks failed", file=out)
    return fails


def run_bench(opt, out) -> int:
    ns = _ns(opt.n, [20000, 40000, 60000, 80000, 100000])
    print(_config(opt, ns[0] if len(ns) == 1 else 0), file=out)
    print("N,M,L,time_fast_s,time_dense_s,rel_err_inf", file=out)
    norm = []
    for n in ns:
        xy = _points(opt, n)
        n = xy.size // 2
        u = api.random_vector(n, opt.seed)
        with api.FastOperator(xy, opt.t, opt.m, _levels(opt.levels)) as op:
            tf = []
            for _ in range(3):
                t0 = time.perf_counter()
                bf = op.apply(u)
                tf.append(time.perf_counter() - t0)
            L = op.levels
        td = []
        for _ in range(3):
            t0 = time.perf_counter()
            bd = api.dense_matvec(xy, opt.t, u)
            td.append(time.perf_counter() - t0)
        fast, dense = sorted(tf)[1], sorted(td)[1]  # median of 3
        print(f"{n},{opt.m},{L},{fast:.6e},{dense:.6e},{_rel_inf(bf, bd):.3e}", file=out)
        norm.append(f"# normalized N={n} fast={fast / n:.3e} s/pt dense={dense / n:.3e} s/pt")
    for line in norm:
        print(line, file=out)
    return 0


def run_errtrend(opt, out) -> int:
    print(_config(opt, 0), file=out)
    print("rho_x,M,case,E,bound", file=out)
    pi = math.pi
    for M in (5, 10, 20):
        for cs in "ab":
            thx, thy = (pi / 3, pi / 3) if cs == "a" else (pi, pi / 4)
            omx, omy = pi / 3, (pi / 3 if cs == "a" else pi / 2)
            for i in range(100):
                rho = 1.1 + (21.0 - 1.1) * i / 99.0
                X = [rho * math.sin(thx) * math.cos(omx), rho * math.sin(thx) * math.sin(omx),
                     rho * math.cos(thx)]
                Y = [math.sin(thy) * math.cos(omy), math.sin(thy) * math.sin(omy), math.cos(thy)]
                e = abs(api.green_truncated(X, Y, M) - api.green_exact(X, Y))
                b = api.truncation_error_bound(rho, 1.0 / rho, M)
                print(f"{rho:.6f},{M},{cs},{e:.6e},{b:.6e}", file=out)
    return 0


def run_solve(opt, out) -> int:
    n = _ns(opt.n, [500])[0]
    xy = _points(opt, n)
    n = xy.size // 2
    print(_config(opt, n), file=out)
    x, y = xy[0::2], xy[1::2]
    f = np.exp(x) * np.sin(3.0 * y) + x * y
    fmax = float(np.max(np.abs(f)))
    with api.FastOperator(xy, opt.t, opt.m, _levels(opt.levels)) as op:
        r = op.solve(f, opt.tol, opt.max_iter, opt.restart)
        L = op.levels
    print(f"# solve: L={L} iterations={r.iterations} residual={r.final_relative_residual:.3e} "
          f"converged={int(r.converged)}", file=out)
    if n <= 5000:
        try:
            cd, res = api.dense_solve(xy, opt.t, f)
            print(f"# dense comparison: coeff dev {_rel_inf(r.c, cd):.3e}, dense residual "
                  f"{res:.3e}", file=out)
        except IMQError as e:
            if e.code != 2:
                raise
            print(f"# dense comparison skipped: {e.msg}", file=out)
    at = api.evaluate_interpolant(xy, r.c, opt.t, xy)
    print(f"# interpolant reproduction: {float(np.max(np.abs(at - f))) / fmax:.3e} relative",
          file=out)
    print("index,coefficient", file=out)
    for i, c in enumerate(r.c):
        print(f"{i},{c!r}", file=out)
    return 0 if r.converged else 1


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description="fast inverse-multiquadric kernel evaluator (B200)")
    ap.add_argument("--mode", default="verify", choices=("verify", "bench", "errtrend", "solve"))
    ap.add_argument("--n", default="", help="point count; comma list in bench mode")
    ap.add_argument("--t", type=float, default=1.0, help="kernel shape parameter t > 0")
    ap.add_argument("--m", type=int, default=10, help="truncation order M")
    ap.add_argument("--levels", default="auto", help="'auto' or a level count >= 1")
    ap.add_argument("--seed", type=int, default=42, help="seed for the test vector")
    ap.add_argument("--points", default="", help="two-column point file replacing the Halton set")
    ap.add_argument("--out", default="", help="output file (default stdout)")
    ap.add_argument("--threads", type=int, default=0, help="host worker thread cap")
    ap.add_argument("--tol", type=float, default=1e-10, help="solver relative residual tolerance")
    ap.add_argument("--max-iter", dest="max_iter", type=int, default=500)
    ap.add_argument("--restart", type=int, default=100)
    opt = ap.parse_args(argv)
    try:
        if opt.threads > 0:
            api.set_threads(opt.threads)
        out = open(opt.out, "w") if opt.out else sys.stdout
        try:
            fn = {"bench": run_bench, "errtrend": run_errtrend, "solve": run_solve,
                  "verify": run_verify}[opt.mode]
            return fn(opt, out)
        finally:
            if opt.out:
                out.close()
    except (IMQError, ValueError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
