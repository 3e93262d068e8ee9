"""Full-size configurations on the GPU: the product at BASELINE.json sizes is
checked against the oracle on sampled rows (same per-row arithmetic as the
reference, ora_fast_matvec_rows) and through size-independent properties."""
import os

import numpy as np
import pytest

from conftest import rel_err_inf

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def sampled_check(imq, oracle, xy, t, m, L, u, nrows, seed=0):
    n = u.size
    op = imq.FastOperator(xy, t, m, L)
    b = op.apply(u)
    rows = np.unique(np.random.default_rng(seed).integers(0, n, nrows))
    ref = oracle.fast_matvec_rows(xy, t, m, L, u, rows)
    err = float(np.max(np.abs(b[rows] - ref)) / np.max(np.abs(ref)))
    return op, b, rows, ref, err


def test_config3_clustered_full(imq, oracle):
    from paper_2205_04194_b200 import inputs
    xy = inputs.gaussian_mixture(1 << 20, 1)
    u = inputs.random_vector(1 << 20, 42)
    op, b, rows, ref, err = sampled_check(imq, oracle, xy, 0.02, 14, 6, u, 2048)
    assert err <= 1e-10
    d = oracle.dense_matvec(xy, 0.02, u, rows[:256])
    assert np.max(np.abs(b[rows[:256]] - d)) <= 2 * np.max(np.abs(ref[:256] - d)) + 1e-12 * np.max(np.abs(d))


def test_config4_full_size(imq, oracle):
    from paper_2205_04194_b200 import inputs
    n = 1 << 24
    xy = inputs.uniform_points(n, 0)
    u = inputs.random_vector(n, 1000)
    op, b, rows, ref, err = sampled_check(imq, oracle, xy, 0.01, 16, 8, u, 256)
    assert err <= 1e-10
    # linearity at full size (size-independent property)
    u2 = inputs.random_vector(n, 1001)
    b2 = op.apply(u2)
    bm = op.apply(0.25 * u - 2.0 * u2)
    assert rel_err_inf(bm, 0.25 * b - 2.0 * b2) <= 1e-12
    assert np.array_equal(op.apply(u), b)


def test_config5_sweep_sampled(imq, oracle):
    """4,194,304 uniform points, L=7: p x c corners of the sweep, sampled rows vs
    the oracle (<=1e-10) and vs the direct sum at the truncation error."""
    from paper_2205_04194_b200 import inputs
    n = 1 << 22
    xy = inputs.uniform_points(n, 0)
    u = inputs.random_vector(n, 42)
    rows = (np.arange(4096) * n) // 4096  # i_r = floor(r N / 4096)
    sub = rows[::64]
    dense = {}
    for p, c in ((4, 0.001), (12, 0.1), (16, 0.01), (20, 1.0)):
        op = imq.FastOperator(xy, c, p, 7)
        b = op.apply(u)
        ref = oracle.fast_matvec_rows(xy, c, p, 7, u, sub)
        assert np.max(np.abs(b[sub] - ref)) / np.max(np.abs(ref)) <= 1e-10, (p, c)
        if c not in dense:
            dense[c] = oracle.dense_matvec(xy, c, u, sub)
        d = dense[c]
        assert np.max(np.abs(b[sub] - d)) <= 2 * np.max(np.abs(ref - d)) + 1e-12 * np.max(np.abs(d))
        op.close()


@pytest.mark.parametrize("case", ["strip", "clustered_wide_t", "uniform_all_rings"])
def test_chebyshev_and_ring_paths_vs_oracle(imq, oracle, case):
    """Large inputs that switch on the Chebyshev coarse pass and the rings in
    different places: a thin strip (most boxes empty, full ones crowded), a
    clustered set with t large enough that every level 2..L-1 has a ring,
    and a uniform set with rings from level 3 on.  Sampled rows vs the
    oracle's reference-order rows (<= 1e-10, expected ~1e-14)."""
    from paper_2205_04194_b200 import inputs
    n = 1 << 20
    rng = np.random.default_rng(11)
    if case == "strip":
        xy = np.stack([rng.random(n), 0.3 + 0.01 * rng.random(n)], 1).reshape(-1)
        t, m, L = 0.05, 12, 6
    elif case == "clustered_wide_t":
        xy = inputs.gaussian_mixture(n, 1)
        t, m, L = 0.2, 10, 6
    else:
        xy = inputs.uniform_points(n, 5)
        t, m, L = 0.03, 14, 6
    u = inputs.random_vector(n, 9)
    op, b, rows, ref, err = sampled_check(imq, oracle, xy, t, m, L, u, 1024, seed=3)
    st = op.stats()
    if case != "strip":
        assert st["cheb_levels"] > 0 and st["cheb_ring"] == 1, st
    assert err <= 1e-10, (case, err)
    assert err <= 1e-12, (case, err)  # the interpolation keeps ~1e-14 in practice
    op.close()


def test_randomised_geometries_vs_oracle(imq, oracle):
    """tools/stress_paths.py at a fixed seed: random point sets (strips,
    annuli, clusters, duplicates), shapes, orders and levels through the
    Chebyshev / ring / finest-split paths; sampled rows vs the oracle."""
    import subprocess
    import sys
    from conftest import ROOT
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "stress_paths.py"), "11", "12"],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    worst = float(r.stdout.strip().splitlines()[-1].split()[-1])
    assert worst <= 1e-12, r.stdout


def test_dense_262144(imq, oracle):
    """Config 5's direct O(N^2) reference point at N = 262,144."""
    from paper_2205_04194_b200 import inputs
    n = 262144
    xy = inputs.uniform_points(n, 0)
    u = inputs.random_vector(n, 42)
    b = imq.dense_matvec(xy, 0.01, u)
    rows = np.arange(0, n, n // 256)
    ref = oracle.dense_matvec(xy, 0.01, u, rows)
    assert np.max(np.abs(b[rows] - ref)) / np.max(np.abs(ref)) <= 1e-12


def test_config2_gmres_iteration_matched(imq, oracle):
    """SURVEY 8(d) protocol: same cap, compare the restart-boundary residuals."""
    from paper_2205_04194_b200 import inputs
    xy = inputs.uniform_points(65536, 0)
    f = inputs.cfg2_rhs(xy)
    op = imq.FastOperator(xy, 0.05, 12, 0)
    assert op.levels == 2  # auto level of the reference for N = 65536, M = 12
    r = op.solve(f, 1e-8, 100, 50)
    ref = oracle.iterative_solve(xy, 0.05, 12, 0, f, 1e-8, 100, 50)
    assert r.iterations == ref["iterations"] == 100
    cr, rr = np.array(r.cycle_residuals), ref["cycle_residuals"]
    assert cr.size == rr.size
    assert np.max(np.abs(cr - rr) / rr) <= 1e-6
    # the coefficient vector against the REFERENCE's own c at matched caps
    # (tests/golden/cfg2_ref_it*.npz, make_golden_big.py; BASELINE config 2):
    # measured 3.3e-11 (100 iterations) and 6.2e-8 (2,000), where GMRES has
    # amplified the last-bit differences of the products for 40 cycles
    import os
    from conftest import GOLDEN
    for cap, bound in ((100, 1e-8), (2000, 1e-6)):
        g = np.load(os.path.join(GOLDEN, f"cfg2_ref_it{cap}.npz"))
        rc = r if cap == 100 else op.solve(f, 1e-8, cap, 50)
        assert rc.iterations == int(g["iterations"]) == cap
        assert abs(rc.final_relative_residual - float(g["res"])) <= 1e-6 * float(g["res"])
        assert float(np.max(np.abs(rc.c - g["c"])) / np.max(np.abs(g["c"]))) <= bound, cap
    # iterations to each tolerance of the protocol equal the reference's (87,
    # 182, 691: profiles/r02_gmres_protocol.json)
    for tol, its in ((1e-3, 87), (5e-4, 182), (2e-4, 691)):
        rt = op.solve(f, tol, 2000, 50)
        assert rt.converged and rt.iterations == its, (tol, rt.iterations)
