"""Full-size parity of the interpolated far field (the only non-exact step).

* Config 4 (N = 16,777,216) against the REFERENCE ITSELF: 65,536 rows stored
  exactly plus per-chunk checksums of the whole vector (4,096 chunks of 4,096
  rows: sum b, sum |b|, sum b^2), made once by running the unmodified
  reference (oracle/_ref, tests/golden/make_golden_big.py; build 168 s +
  apply 479 s on 8 cores).
* Whole-vector comparisons at N = 1,048,576 against the C oracle (bit-exact
  with the reference on every committed golden) for every interpolation mode:
  node pass only, node pass + rings, everything config 4 uses (inner lists at
  16x16, rings at 16x16 and 20x20, X-ring), and config 3 (clustered).
* p = 20 right at each gate of build_cheb (t/h just above 1.25, 2.5 and 5),
  whole vectors.
* All 20 (p, c) cells of config 5 on the rows floor(r N / 4096).
* The build-time certificate (operator.cu certify()) holds every case to its
  budget, and its estimate bounds the measured deviation.

Worst deviations are printed (`pytest -s`).
"""
import numpy as np
import pytest

from conftest import rel_err_inf

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

N1M = 1 << 20


def full_check(imq, oracle, xy, t, m, L, u, **opts):
    op = imq.FastOperator(xy, t, m, L, **opts)
    b = op.apply(u)
    st = op.stats()
    op.close()
    ref = oracle.fast_matvec(xy, t, m, L, u)
    return rel_err_inf(b, ref), st


def test_config4_whole_vector_vs_reference(imq, golden):
    """Config 4 exactly (uniform seed 0, c = 0.01, p = 16, L = 8, u =
    random_vector(N, 1000)) against the reference's own product."""
    from paper_2205_04194_b200 import inputs
    g = golden("cfg4_ref")
    n = 1 << 24
    xy = inputs.uniform_points(n, 0)
    u = inputs.random_vector(n, 1000)
    op = imq.FastOperator(xy, 0.01, 16, 8)
    b = op.apply(u)
    st = op.stats()
    op.close()
    assert st["cheb_xring"] == 1 and st["cheb_ring"] == 1, st  # the bench path
    scale = np.max(np.abs(g["b_rows"]))
    row_err = np.max(np.abs(b[g["rows"]] - g["b_rows"])) / scale
    c = b.reshape(-1, 4096)
    s_err = np.max(np.abs(c.sum(1) - g["chunk_sum"]) / g["chunk_abs"])
    a_err = np.max(np.abs(np.abs(c).sum(1) - g["chunk_abs"]) / g["chunk_abs"])
    q_err = np.max(np.abs((c * c).sum(1) - g["chunk_sq"]) / g["chunk_sq"])
    fp = np.array([b[0], b[-1], b.sum(), np.abs(b).sum(), np.abs(b).max()])
    fp_err = np.max(np.abs(fp - g["fp"]) / np.abs(g["fp"]))
    print(f"\ncfg4 vs reference: 65536 rows {row_err:.2e}, chunk sums {s_err:.2e}, "
          f"chunk |b| {a_err:.2e}, chunk b^2 {q_err:.2e}, fingerprints {fp_err:.2e}, "
          f"certificate {st['cert_estimate']:.2e}")
    assert row_err <= 1e-10
    # a deviation d in one row moves its chunk's sums by ~d / chunk scale
    assert s_err <= 1e-10 and a_err <= 1e-10 and q_err <= 1e-10 and fp_err <= 1e-10
    assert row_err <= 1e-12  # measured ~5e-14


@pytest.mark.parametrize("case", ["nodes", "rings", "cfg4_mix", "config3"])
def test_whole_vector_1m_per_mode(imq, oracle, case):
    """Every row of a 1,048,576-point product vs the oracle, one case per
    interpolation mode of build_cheb (L = 6, p = 16)."""
    from paper_2205_04194_b200 import inputs
    u = inputs.random_vector(N1M, 42)
    if case == "config3":
        xy, t = inputs.gaussian_mixture(N1M, 1), 0.02
        m = 14
    else:
        xy = inputs.uniform_points(N1M, 0)
        t = {"nodes": 0.001, "rings": 0.02, "cfg4_mix": 0.04}[case]
        m = 16
    err, st = full_check(imq, oracle, xy, t, m, 6, u)
    print(f"\n{case}: whole-vector deviation {err:.2e}, certificate {st['cert_estimate']:.2e} "
          f"(cheb {st['cheb_levels']}, ring {st['cheb_ring']}, xring {st['cheb_xring']}, "
          f"fallbacks {st['cert_fallbacks']})")
    assert st["cheb_levels"] > 0
    if case == "rings":
        assert st["cheb_ring"] == 1
    if case == "cfg4_mix":
        assert st["cheb_ring"] == 1 and st["cheb_xring"] == 1
    assert err <= 1e-10
    assert err <= 1e-12
    assert st["cert_estimate"] <= st["cert_budget"]


@pytest.mark.parametrize("tau", [1.27, 2.55, 5.2])
def test_gate_edges_p20_whole_vector(imq, oracle, tau):
    """p = 20 with t just above a gate of build_cheb: t/h = 1.27 of the
    level-(L-2) boxes (rings), 2.55 (rings at 16x16, inner lists at 16x16),
    5.2 of the level-(L-1) boxes (X-ring).  Whole 1M vectors vs the oracle."""
    from paper_2205_04194_b200 import inputs
    xy = inputs.uniform_points(N1M, 3)
    u = inputs.random_vector(N1M, 5)
    side = 1.0
    h = {1.27: side / 64, 2.55: side / 64, 5.2: side / 128}[tau]
    t = tau * h
    err, st = full_check(imq, oracle, xy, t, 20, 6, u)
    print(f"\ngate t/h={tau}: whole-vector deviation {err:.2e}, certificate "
          f"{st['cert_estimate']:.2e} (ring {st['cheb_ring']}, xring {st['cheb_xring']}, "
          f"fallbacks {st['cert_fallbacks']})")
    assert err <= 1e-10
    assert err <= 1e-12


def test_config5_all_cells(imq, oracle):
    """All 20 (p, c) cells of config 5 (N = 4,194,304, L = 7) on the 4,096
    rows floor(r N / 4096) vs the oracle's reference-order rows."""
    from paper_2205_04194_b200 import inputs
    n = 1 << 22
    xy = inputs.uniform_points(n, 0)
    u = inputs.random_vector(n, 42)
    rows = (np.arange(4096) * n) // 4096
    worst = 0.0
    for c in (0.001, 0.01, 0.1, 1.0):
        for p in (4, 8, 12, 16, 20):
            op = imq.FastOperator(xy, c, p, 7)
            b = op.apply(u)
            st = op.stats()
            op.close()
            ref = oracle.fast_matvec_rows(xy, c, p, 7, u, rows)
            err = float(np.max(np.abs(b[rows] - ref)) / np.max(np.abs(ref)))
            print(f"\ncfg5 p={p:2d} c={c}: {err:.2e} (certificate {st['cert_estimate']:.2e})", end="")
            worst = max(worst, err)
            assert err <= 1e-10, (p, c, err)
    print(f"\ncfg5 worst {worst:.2e}")
    assert worst <= 1e-12


def test_certificate_fallback_reaches_direct(imq, oracle):
    """A budget no interpolation can meet switches every interpolation off:
    the product is then bit-identical to the all-direct evaluation."""
    from paper_2205_04194_b200 import inputs
    n = 1 << 18
    xy = inputs.uniform_points(n, 0)
    u = inputs.random_vector(n, 1000)
    with imq.FastOperator(xy, 0.05, 16, 5, cert_budget=1e-300) as op:
        st = op.stats()
        b = op.apply(u)
    with imq.FastOperator(xy, 0.05, 16, 5, flags=["no_cheb"]) as op2:
        b2 = op2.apply(u)
    assert st["cert_fallbacks"] >= 1 and st["cheb_levels"] == 0, st
    assert np.array_equal(b, b2)
    with imq.FastOperator(xy, 0.05, 16, 5) as op3:
        st3 = op3.stats()
    assert st3["cheb_levels"] > 0 and st3["cert_fallbacks"] == 0, st3
    assert 0 < st3["cert_estimate"] <= st3["cert_budget"] == 2e-12


def test_options_cannot_loosen(imq):
    """Gates below the defaults are raised to them; scheduling options leave
    every bit unchanged."""
    from paper_2205_04194_b200 import inputs
    n = 1 << 18
    xy = inputs.uniform_points(n, 0)
    u = inputs.random_vector(n, 1000)
    with imq.FastOperator(xy, 0.05, 16, 5) as op:
        b = op.apply(u)
        st = op.stats()
    with imq.FastOperator(xy, 0.05, 16, 5, ring_tau=0.0, ring2_tau=0.1, inner_tau=0.1,
                          xring_tau=0.1, cert_budget=1.0) as op2:
        b2 = op2.apply(u)
        st2 = op2.stats()
    assert np.array_equal(b, b2) and st2["cert_budget"] == 2e-12
    assert st2["cheb_xring"] == st["cheb_xring"] and st2["cheb_ring"] == st["cheb_ring"]
    with imq.FastOperator(xy, 0.05, 16, 5, far_rmax=1, far_streams=1) as op3:
        b3 = op3.apply(u)
    assert np.array_equal(b, b3)


def test_node_and_ring_gemm_paths(imq, oracle):
    """A 16.8M-point case whose level-6 node pass (18x18 nodes, full lists) and
    level-7 ring (20x20 nodes at the level-6 boxes) run as tensor-core GEMMs
    (t = 0.007: rings from level 7 at 1.79 h of the level-6 boxes, no X-ring):
    sampled rows vs the oracle, and the device list check replays the GEMM
    offset tables against the reference lists."""
    from paper_2205_04194_b200 import inputs
    n = 1 << 24
    xy = inputs.uniform_points(n, 0)
    u = inputs.random_vector(n, 3)
    with imq.FastOperator(xy, 0.007, 16, 8) as op:
        st = op.stats()
        b = op.apply(u)
        lc = op.check_lists(2048)
    assert st["cheb_ring"] == 1 and st["cheb_xring"] == 0, st
    # level 6: 16,384 boxes x 324 nodes x <= 27 lists, ring: x 400 nodes x <= 20
    assert st["gemm_node_pairs"] > 16384 * (324 * 20 + 400 * 15), st["gemm_node_pairs"]
    assert lc["missing"] == 0 and lc["duplicated"] == 0 and lc["extra"] == 0, lc
    rows = (np.arange(2048) * n) // 2048
    ref = oracle.fast_matvec_rows(xy, 0.007, 16, 8, u, rows)
    err = float(np.max(np.abs(b[rows] - ref)) / np.max(np.abs(ref)))
    print(f"\nnode + ring GEMM case: {err:.2e} (certificate {st['cert_estimate']:.2e})")
    assert err <= 1e-12
