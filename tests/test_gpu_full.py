"""Full-size configurations on the GPU: the product at BASELINE.json sizes is
checked against the oracle on sampled rows (same per-row arithmetic as the
reference, ora_fast_matvec_rows) and through size-independent properties."""
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
