"""Pins the C oracle (oracle/imq_oracle.c) against the reference's own outputs.

The golden fixtures were produced by running the reference library itself
(tests/golden/make_golden.py); the oracle must reproduce them BIT FOR BIT.
When /root/reference is present the reference is also run live.
"""
import os

import numpy as np
import pytest

from conftest import ROOT, rel_err_inf


def test_generators_bitwise(oracle, golden):
    g = golden("gen")
    assert np.array_equal(oracle.random_vector(64, 42), g["rv42"])
    assert np.array_equal(oracle.random_vector(64, 0), g["rv0"])
    assert np.array_equal(oracle.random_vector(64, 1000), g["rv1000"])
    assert np.array_equal(oracle.halton2d(64), g["halton"])
    for n, m, L in g["auto"]:
        assert oracle.auto_level(int(n), int(m)) == L


def test_appendix_b_fingerprint(oracle, golden):
    c = golden("cfg1")
    b = oracle.fast_matvec(c["xy"], 0.1, 10, 2, c["u"])
    assert np.array_equal(b, c["b_fast"])
    assert b[0] == -4.2733848938270214
    assert b[-1] == 53.707507601630986
    sq = oracle.bounding_square(c["xy"])
    assert sq == (0.00026815667330509774, 0.00015237779721927192, 0.99980446419333591)
    d = oracle.dense_matvec(c["xy"], 0.1, c["u"])
    assert np.array_equal(d, c["b_dense"])
    assert abs(rel_err_inf(b, d) - 9.962661e-07) < 1e-12


def test_families_bitwise(oracle, golden):
    g = golden("family600")
    for name in ("halton", "random"):
        for t in (0.5, 1.0, 2.0):
            for L in (1, 2):
                b = oracle.fast_matvec(g[name], t, 10, L, g["u"])
                assert np.array_equal(b, g[f"{name}_t{t}_L{L}"]), (name, t, L)


def test_clustered_and_sweep_bitwise(oracle, golden):
    c = golden("clustered")
    assert np.array_equal(oracle.fast_matvec(c["xy"], 0.02, 14, 3, c["u"]), c["b_fast"])
    assert np.array_equal(oracle.dense_matvec(c["xy"], 0.02, c["u"]), c["b_dense"])
    s = golden("sweep2048")
    for cc in (0.001, 0.01, 0.1, 1.0):
        for p in (4, 8, 12, 16, 20):
            assert np.array_equal(oracle.fast_matvec(s["xy"], cc, p, 3, s["u"]), s[f"c{cc}_p{p}"])


def test_high_order_and_degenerate(oracle, golden):
    h = golden("highm")
    assert np.array_equal(oracle.fast_matvec(h["xy"], 0.03, 30, 0, h["u"]), h["b_m30"])
    assert np.array_equal(oracle.fast_matvec(h["xy"], 0.03, 0, 2, h["u"]), h["b_m0"])
    assert np.array_equal(oracle.fast_matvec(h["xy"], 0.03, 1, 2, h["u"]), h["b_m1"])
    d = golden("degenerate")
    assert np.array_equal(oracle.fast_matvec(d["same"], 0.7, 10, 1, d["u12"]), d["b_same"])
    assert np.array_equal(oracle.fast_matvec(np.array([0.3, 0.4]), 2.0, 10, 1, [3.0]),
                          d["single"])
    assert d["single"][0] == 1.5


def test_gmres_bitwise(oracle, golden):
    g = golden("gmres")
    s = oracle.iterative_solve(g["xy400"], 0.03, 12, 0, g["f400"], 1e-10, 300, 50)
    assert s["iterations"] == int(g["it400"])
    assert np.array_equal(s["c"], g["c400"])
    s2 = oracle.iterative_solve(g["xy2"], 0.05, 12, 0, g["f2"], 1e-8, 100, 50)
    assert s2["iterations"] == int(g["it2"])
    assert np.array_equal(s2["c"], g["c2"])
    assert s2["final_relative_residual"] == float(g["res2"])


def test_sampled_rows_equal_full_product(oracle, golden):
    c = golden("cfg1")
    rows = np.array([0, 1, 17, 2048, 4095])
    assert np.array_equal(oracle.fast_matvec_rows(c["xy"], 0.1, 10, 2, c["u"], rows),
                          c["b_fast"][rows])


def test_interaction_lists_match_partition_rules(oracle):
    # test_partition.cpp:93-114: 12 at the level-1 corner, 7 at (1,1), <= 27 below
    assert len(oracle.interaction_list(1, 0, 0)) == 12
    assert len(oracle.interaction_list(1, 1, 1)) == 7
    for l in (2, 3):
        g = 1 << (l + 1)
        assert max(len(oracle.interaction_list(l, i, j)) for i in range(g) for j in range(g)) <= 27


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libimqfast_ref.so")),
                    reason="reference not built here (needs /root/reference)")
def test_live_reference_agrees(oracle):
    from oracle import Reference
    R = Reference()
    xy = oracle.random_vector(2 * 1500, 3) * 0.5 + 0.5
    u = oracle.random_vector(1500, 4)
    for (t, m, L) in ((0.05, 12, 2), (0.3, 6, 3), (1.0, 16, 1)):
        assert np.array_equal(oracle.fast_matvec(xy, t, m, L, u), R.fast_matvec(xy, t, m, L, u))
