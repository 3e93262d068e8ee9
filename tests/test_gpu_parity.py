"""GPU parity of the CUDA product against the oracle and the reference's own
golden outputs.  Everything goes through the C ABI (libimqfast.so).

Tolerances: bit-exact for binning / bucket membership / ordering (integer
work); rel_err_inf <= 1e-10 for the fast product vs the reference fast product
(north_star); |gpu - dense| <= 2 |ref - dense| + 1e-12 against the direct sum.
"""
import numpy as np
import pytest

from conftest import rel_err_inf

pytestmark = pytest.mark.gpu
TOL = 1e-10


def morton(i, j):
    i = np.asarray(i, dtype=np.uint64)
    j = np.asarray(j, dtype=np.uint64)
    out = np.zeros_like(i)
    for b in range(16):
        out |= ((i >> np.uint64(b)) & np.uint64(1)) << np.uint64(2 * b + 1)
        out |= ((j >> np.uint64(b)) & np.uint64(1)) << np.uint64(2 * b)
    return out


def check_binning(imq, oracle, xy, t, m, L):
    op = imq.FastOperator(xy, t, m, L)
    L = op.levels
    perm = op.permutation()
    ls = op.leaf_start()
    n = xy.size // 2
    assert np.array_equal(np.sort(perm), np.arange(n))
    leaf_of_sorted = np.repeat(np.arange(ls.size - 1), np.diff(ls))
    leaf = np.empty(n, dtype=np.int64)
    leaf[perm] = leaf_of_sorted
    for lvl in range(1, L + 1):
        g = 1 << (lvl + 1)
        ids = oracle.block_ids(xy, lvl).astype(np.int64)
        want = morton(ids // g, ids % g).astype(np.int64)
        got = leaf >> (2 * (L - lvl))
        assert np.array_equal(got, want), f"level {lvl}"
    # within every bucket the points keep ascending original index
    # (BlockTree::buckets order, partition.cpp:53-54)
    for c in range(ls.size - 1):
        seg = perm[ls[c]:ls[c + 1]]
        assert np.all(np.diff(seg) > 0)
    return op


def test_binning_bit_exact(imq, oracle, golden):
    c = golden("cfg1")
    check_binning(imq, oracle, c["xy"], 0.1, 10, 2)
    cl = golden("clustered")
    check_binning(imq, oracle, cl["xy"], 0.02, 14, 5)
    # lattice points sitting exactly on cell edges (upper edges go up)
    g = np.linspace(0.0, 1.0, 33)
    X, Y = np.meshgrid(g, g, indexing="ij")
    xy = np.stack([X.ravel(), Y.ravel()], 1).ravel()
    check_binning(imq, oracle, xy, 0.5, 4, 4)
    # degenerate square (all points equal) and a thin strip (dy = 0)
    check_binning(imq, oracle, np.tile([0.3, 0.4], 50), 0.7, 4, 2)
    strip = np.stack([np.linspace(-3, 5, 400), np.full(400, 2.0)], 1).ravel()
    check_binning(imq, oracle, strip, 0.1, 6, 3)
    # the radix sort over many 4,096-key tiles with a partial last one, three
    # 8-bit passes (18-bit keys at L = 8) and two (14-bit keys at L = 6)
    rng = np.random.default_rng(5)
    check_binning(imq, oracle, rng.random(2 * 300_001), 0.05, 4, 8)
    check_binning(imq, oracle, rng.normal(0.5, 0.1, 2 * 123_457), 0.05, 4, 6)


def test_config1_fast_matches_reference(imq, golden):
    c = golden("cfg1")
    op = imq.FastOperator(c["xy"], 0.1, 10, 2)
    b = op.apply(c["u"])
    assert rel_err_inf(b, c["b_fast"]) <= TOL
    ref_err = rel_err_inf(c["b_fast"], c["b_dense"])
    assert abs(rel_err_inf(b, c["b_dense"]) - ref_err) <= ref_err  # same truncation error
    d = imq.dense_matvec(c["xy"], 0.1, c["u"])
    assert rel_err_inf(d, c["b_dense"]) <= 1e-13


def test_families_vs_golden(imq, golden):
    g = golden("family600")
    for name in ("halton", "random"):
        for t in (0.5, 1.0, 2.0):
            for L in (1, 2):
                b = imq.FastOperator(g[name], t, 10, L).apply(g["u"])
                assert rel_err_inf(b, g[f"{name}_t{t}_L{L}"]) <= TOL, (name, t, L)


def test_clustered_vs_golden(imq, golden):
    c = golden("clustered")
    b = imq.FastOperator(c["xy"], 0.02, 14, 3).apply(c["u"])
    assert rel_err_inf(b, c["b_fast"]) <= TOL
    ref = rel_err_inf(c["b_fast"], c["b_dense"])
    assert rel_err_inf(b, c["b_dense"]) <= 2 * ref + 1e-12


def test_order_shape_sweep_vs_golden(imq, golden):
    s = golden("sweep2048")
    for cc in (0.001, 0.01, 0.1, 1.0):
        for p in (4, 8, 12, 16, 20):
            b = imq.FastOperator(s["xy"], cc, p, 3).apply(s["u"])
            assert rel_err_inf(b, s[f"c{cc}_p{p}"]) <= TOL, (cc, p)


def test_generic_orders_vs_oracle(imq, oracle, golden):
    h = golden("highm")
    assert rel_err_inf(imq.FastOperator(h["xy"], 0.03, 30, 0).apply(h["u"]), h["b_m30"]) <= TOL
    assert rel_err_inf(imq.FastOperator(h["xy"], 0.03, 0, 2).apply(h["u"]), h["b_m0"]) <= TOL
    assert rel_err_inf(imq.FastOperator(h["xy"], 0.03, 1, 2).apply(h["u"]), h["b_m1"]) <= TOL
    xy = oracle.random_vector(2 * 3000, 9) * 0.5 + 0.5
    u = oracle.random_vector(3000, 10)
    for m in (3, 5, 7, 9, 11, 13, 15, 17, 19, 22, 25, 40):
        b = imq.FastOperator(xy, 0.2, m, 3).apply(u)
        assert rel_err_inf(b, oracle.fast_matvec(xy, 0.2, m, 3, u)) <= TOL, m


def test_degenerate_trees(imq, golden):
    d = golden("degenerate")
    b = imq.FastOperator(d["same"], 0.7, 10, 1).apply(d["u12"])
    assert rel_err_inf(b, d["b_same"]) <= 1e-14
    one = imq.FastOperator(np.array([0.3, 0.4]), 2.0, 10, 1).apply([3.0])
    assert one[0] == pytest.approx(1.5, rel=1e-15)


def test_linearity_determinism_symmetry(imq, oracle):
    xy = oracle.halton2d(3000)
    op = imq.FastOperator(xy, 1.0, 10, 2)
    u1, u2 = oracle.random_vector(3000, 7), oracle.random_vector(3000, 8)
    a, c = 0.7, -1.3
    b1, b2, bm = op.apply(u1), op.apply(u2), op.apply(a * u1 + c * u2)
    assert rel_err_inf(bm, a * b1 + c * b2) <= 1e-12
    assert np.array_equal(op.apply(u1), b1)
    op2 = imq.FastOperator(xy, 1.0, 10, 2)
    assert np.array_equal(op2.apply(u1), b1)
    utAv, vtAu = u1 @ b2, u2 @ b1
    scale = np.abs(u1 * b2).sum() + np.abs(u2 * b1).sum()
    assert abs(utAv - vtAu) <= 5e-8 * scale


def test_basis_columns_within_level1_bound(imq, oracle):
    # test_fastmv.cpp:146-164
    n = 400
    xy = oracle.halton2d(n)
    op = imq.FastOperator(xy, 1.0, 10, 1)
    for j in (0, 57, 399):
        e = np.zeros(n)
        e[j] = 1.0
        col = op.apply(e)
        d = xy.reshape(-1, 2) - xy.reshape(-1, 2)[j]
        exact = 1.0 / np.sqrt(1.0 + (d ** 2).sum(1))
        assert np.max(np.abs(col - exact)) <= 2.8668e-9 * (1 + 1e-6)


def test_dense_and_interpolant_vs_oracle(imq, oracle):
    xy = oracle.random_vector(2 * 5000, 3) * 0.5 + 0.5
    u = oracle.random_vector(5000, 4)
    assert rel_err_inf(imq.dense_matvec(xy, 0.01, u), oracle.dense_matvec(xy, 0.01, u)) <= 1e-13
    q = oracle.halton2d(777)
    got = imq.evaluate_interpolant(xy, u, 0.05, q)
    assert rel_err_inf(got, oracle.evaluate_interpolant(xy, u, 0.05, q)) <= 1e-13


def test_gmres_against_reference(imq, golden):
    g = golden("gmres")
    op = imq.FastOperator(g["xy400"], 0.03, 12, 0)
    r = op.solve(g["f400"], 1e-10, 300, 50)
    assert r.converged and r.final_relative_residual <= 1e-10
    assert abs(r.iterations - int(g["it400"])) <= 2
    assert rel_err_inf(r.c, g["c400"]) <= 1e-6
    # config-2 shape: iteration-matched comparison (SURVEY 8(d) protocol)
    op2 = imq.FastOperator(g["xy2"], 0.05, 12, 0)
    r2 = op2.solve(g["f2"], 1e-8, 100, 50)
    assert r2.iterations == int(g["it2"])
    assert abs(r2.final_relative_residual - float(g["res2"])) <= 1e-3 * float(g["res2"])
    assert r2.cycle_residuals == sorted(r2.cycle_residuals, reverse=True)


def test_gmres_semantics(imq, oracle):
    # test_solver.cpp:26-43, 93-123
    op = imq.FastOperator(np.array([0.4, 0.6]), 2.5, 4, 1)
    r = op.solve(np.array([3.0]), 1e-12)
    assert r.converged and r.iterations == 1 and r.c[0] == pytest.approx(7.5, rel=1e-12)
    op = imq.FastOperator(oracle.halton2d(50), 1.0, 6, 1)
    r = op.solve(np.ones(50), 1e-10, 0)
    assert not r.converged and r.iterations == 0 and np.all(r.c == 0.0)
    assert r.final_relative_residual == pytest.approx(1.0, rel=1e-15)
    f = np.ones(50)
    f[4] = np.nan
    with pytest.raises(imq.IMQError) as e:
        op.solve(f)
    assert "iteration" in e.value.msg and e.value.code == 4
    for bad in (dict(tol=0.0), dict(max_iter=-1), dict(restart=0)):
        with pytest.raises(imq.IMQError) as e:
            op.solve(np.ones(50), **{**dict(tol=1e-8, max_iter=10, restart=5), **bad})
        assert e.value.code == 1
    # restart-boundary residuals never increase (test_solver.cpp:93-105)
    op = imq.FastOperator(oracle.halton2d(300), 0.02, 30, 0)
    f = oracle.random_vector(300, 11)
    r = op.solve(f, 1e-12, 60, 10)
    cr = r.cycle_residuals
    assert len(cr) >= 2 and all(cr[i] <= cr[i - 1] * (1 + 1e-10) for i in range(1, len(cr)))
    assert r.final_relative_residual == pytest.approx(cr[-1], rel=1e-12)
    res = np.linalg.norm(f - op.apply(r.c)) / np.linalg.norm(f)
    assert res == pytest.approx(r.final_relative_residual, rel=1e-9)


def test_device_pointer_path_matches_host_path(imq, golden):
    torch = pytest.importorskip("torch")
    c = golden("cfg1")
    op = imq.FastOperator(c["xy"], 0.1, 10, 2)
    b_host = op.apply(c["u"])
    du = torch.tensor(c["u"], device="cuda")
    db = torch.empty_like(du)
    s = torch.cuda.current_stream()
    op.apply_device(du, db, s)
    s.synchronize()
    assert np.array_equal(db.cpu().numpy(), b_host)
    perm = torch.tensor(op.permutation().astype(np.int64), device="cuda")
    dbs = torch.empty_like(du)
    op.apply_sorted_device(du[perm].contiguous(), dbs, s)
    s.synchronize()
    out = torch.empty_like(du)
    out[perm] = dbs
    assert np.array_equal(out.cpu().numpy(), b_host)


def test_verify_suite_passes(imq, oracle):
    fails, rows = imq.verify(oracle.halton2d(2000), 1.0, 10, 0, 42)
    names = [r[0] for r in rows]
    assert names == ["separation_ratio", "separation_ratio_planar", "interaction_counts",
                     "exact_cover", "oracle_equivalence", "m0_sine_moments", "linearity",
                     "determinism"]
    assert fails == 0, rows


def test_operator_errors(imq):
    with pytest.raises(imq.IMQError) as e:
        imq.FastOperator(np.array([0.1, np.inf]), 1.0, 4, 1)
    assert e.value.code == 1 and "non-finite" in e.value.msg
    with pytest.raises(imq.IMQError) as e:
        imq.FastOperator(np.array([0.1, 0.2]), 1.0, -1, 1)
    assert e.value.code == 1
    op = imq.FastOperator(imq.halton2d(10), 1.0, 4, 0)
    assert op.size == 10 and op.levels == imq.auto_level(10, 4)
    with pytest.raises(imq.IMQError):
        op.apply(np.ones(9))
    # restrict: both ends must be level-(L-1) block boundaries
    xy = imq.halton2d(5000)
    with imq.FastOperator(xy, 0.1, 8, 4) as op:
        ls = op.leaf_start()
        cut = int(ls[4 * 37])
        assert imq.capi.lib().imq_ext_operator_restrict(op.handle, 0, cut) == 0
        inner = int(ls[4 * 37 + 1])
        assert inner != cut
        assert imq.capi.lib().imq_ext_operator_restrict(op.handle, 0, inner) == 1
        assert b"boundaries" in imq.capi.lib().imq_last_error()


@pytest.mark.parametrize("world", [2, 3, 5])
def test_sharded_application_emulated(imq, world):
    """The multi-GPU algorithm on one GPU: `world` restricted operators (own +
    halo moments, own-only coarse partials), the coarse all-reduce done by a
    sum, then each rank's far/near field; the union must equal the unsharded
    product.  (NCCL itself is exercised by bench.py under torchrun.)"""
    torch = pytest.importorskip("torch")
    from paper_2205_04194_b200 import inputs
    from paper_2205_04194_b200.parallel import ShardedOperator
    n, m, L = 1 << 18, 12, 5
    # t = 0.01: Chebyshev coarse levels, no rings (t < h); t = 0.05: the
    # level-(L-1) ring through the level-(L-2) boxes' nodes is on; t = 0.2:
    # also the X-ring (the fine pass is gone, the partial pass combines)
    for xy, t in ((inputs.uniform_points(n, 3), 0.01), (inputs.gaussian_mixture(n, 1), 0.01),
                  (inputs.uniform_points(n, 3), 0.05), (inputs.uniform_points(n, 3), 0.2)):
        u = torch.tensor(inputs.random_vector(n, 7), device="cuda")
        full = imq.FastOperator(xy, t, m, L)
        if t >= 0.05:
            assert full.stats()["cheb_ring"] == 1, full.stats()
        if t >= 0.2:  # t >= 5 h of the level-(L-1) boxes: the X-ring too
            assert full.stats()["cheb_xring"] == 1, full.stats()
        b_ref = torch.empty_like(u)
        full.apply_device(u, b_ref)
        torch.cuda.synchronize()
        ranks = [ShardedOperator(imq.FastOperator(xy, t, m, L), r, world) for r in range(world)]
        if xy is not None and full.stats()["near_mode"] == 1:
            # the ranks run the symmetric near field too (boundary slots pulled)
            assert all(sh.op.stats()["near_mode"] == 1 for sh in ranks)
        for sh in ranks:
            sh.moments(u, reduce=False)
        torch.cuda.synchronize()
        total = sum(sh.coarse.clone() for sh in ranks)   # the all-reduce
        b = torch.full_like(u, float("nan"))
        for sh in ranks:
            sh.coarse.copy_(total)
            sh.op.moments_finish()
            sh.evaluate(b)
        torch.cuda.synchronize()
        assert not torch.isnan(b).any()
        err = float((b - b_ref).abs().max() / b_ref.abs().max())
        assert err <= 1e-13, err
        owned = np.concatenate([sh.owned_original_indices() for sh in ranks])
        assert np.array_equal(np.sort(owned), np.arange(n))


@pytest.mark.parametrize("case", ["shifted_scaled", "strip", "duplicates", "two_points",
                                  "tiny_t", "large_t", "sparse_clusters"])
def test_unusual_geometry_vs_oracle(imq, oracle, case):
    """Edge geometries: far-from-origin squares, degenerate aspect ratios,
    coincident points, extreme shape parameters, mostly-empty trees."""
    rng = np.random.default_rng(5)
    if case == "shifted_scaled":
        xy, t, m, L = 1000.0 * rng.random(6000) - 12345.0, 7.5, 10, 3
    elif case == "strip":
        x = rng.random(3000)
        xy, t, m, L = np.stack([x, 1e-6 * x], 1).ravel(), 0.01, 12, 4
    elif case == "duplicates":
        base = rng.random(400)
        xy, t, m, L = np.concatenate([base, base, base]), 0.05, 8, 3
    elif case == "two_points":
        xy, t, m, L = np.array([0.1, 0.2, 0.9, 0.7]), 0.3, 6, 1
    elif case == "tiny_t":
        xy, t, m, L = rng.random(4000), 1e-5, 16, 3
    elif case == "large_t":
        xy, t, m, L = rng.random(4000), 40.0, 12, 3
    else:  # a few tight clusters in a large empty square
        c = rng.random((5, 2)) * 100.0
        xy = (c[rng.integers(0, 5, 3000)] + 0.01 * rng.standard_normal((3000, 2))).ravel()
        t, m, L = 0.002, 14, 6
    n = xy.size // 2
    u = rng.uniform(-1, 1, n)
    b = imq.FastOperator(xy, t, m, L).apply(u)
    ref = oracle.fast_matvec(xy, t, m, L, u)
    assert rel_err_inf(b, ref) <= 1e-10, case


def test_concurrent_apply_from_threads(imq, golden):
    """fastmv.hpp:17-18: the operator is safe for concurrent application to
    distinct vectors (ctypes releases the GIL; the library serialises)."""
    import threading
    c = golden("cfg1")
    op = imq.FastOperator(c["xy"], 0.1, 10, 2)
    us = [imq.random_vector(4096, 100 + k) for k in range(8)]
    want = [op.apply(u) for u in us]
    got = [None] * 8

    def work(k):
        for _ in range(3):
            got[k] = op.apply(us[k])

    ts = [threading.Thread(target=work, args=(k,)) for k in range(8)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for k in range(8):
        assert np.array_equal(got[k], want[k])


@pytest.mark.parametrize("case", ["sym_leaves", "pair_large_leaves", "pair_ragged",
                                  "pair_small_problem"])
def test_near_field_modes_vs_oracle(imq, oracle, case):
    """Each near-field evaluation strategy (imq_ext_stats.near_mode) against
    the oracle: the symmetric per-leaf kernel (leaves <= 128 and enough leaves
    to fill the GPU), the chunk-pair kernel for 1,024-point leaves, for ragged
    cluster leaves with partial chunks, and for a problem too small for the
    per-leaf kernel."""
    rng = np.random.default_rng(11)
    rows = None
    if case == "sym_leaves":
        xy, t, m, L, mode = rng.random(2 * (1 << 21)), 0.05, 8, 7, 1
        rows = np.unique(rng.integers(0, 1 << 21, 512))
    elif case == "pair_large_leaves":
        xy, t, m, L, mode = rng.random(2 * 16384), 0.05, 12, 1, 2
    elif case == "pair_ragged":
        c = rng.random((6, 2))
        k = rng.integers(0, 6, 12000)
        xy = np.clip(c[k] + 0.03 * rng.standard_normal((12000, 2)), 0, 1).ravel()
        t, m, L, mode = 0.02, 10, 2, 2
    else:
        xy, t, m, L, mode = rng.random(2 * 777), 0.3, 8, 1, 2
    n = xy.size // 2
    op = imq.FastOperator(xy, t, m, L)
    assert op.stats()["near_mode"] == mode
    u = rng.uniform(-1, 1, n)
    b = op.apply(u)
    if rows is None:
        ref = oracle.fast_matvec(xy, t, m, L, u)
        assert rel_err_inf(b, ref) <= TOL, case
    else:
        ref = oracle.fast_matvec_rows(xy, t, m, L, u, rows)
        assert float(np.max(np.abs(b[rows] - ref)) / np.max(np.abs(ref))) <= TOL, case
    assert np.array_equal(op.apply(u), b)  # deterministic reductions


@pytest.mark.parametrize("kind", ["pair", "sym_split"])
def test_device_applies_on_different_streams_do_not_race(imq, kind):
    """Entry points that use the operator's internal buffers are ordered on the
    device: interleaved apply_device calls on two streams give the same
    results as sequential ones."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(3)
    if kind == "pair":
        xy, t, m, L = rng.random(2 * 16384), 0.05, 12, 1
    else:
        xy, t, m, L = rng.random(2 * (1 << 20)), 0.02, 10, 6
    n = xy.size // 2
    op = imq.FastOperator(xy, t, m, L)
    us = [torch.tensor(rng.uniform(-1, 1, n), device="cuda") for _ in range(2)]
    want = []
    for u in us:
        b = torch.empty_like(u)
        op.apply_device(u, b)
        torch.cuda.synchronize()
        want.append(b.clone())
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [torch.full_like(us[0], float("nan")) for _ in range(2)]
    torch.cuda.synchronize()
    for _ in range(4):
        for k in range(2):
            op.apply_device(us[k], outs[k], streams[k])
    torch.cuda.synchronize()
    for k in range(2):
        assert torch.equal(outs[k], want[k])


def test_batch_and_pageable_host_paths_bitwise(imq):
    """imq_ext_operator_apply_batch (copy / compute pipeline, f4) and the
    pageable-buffer staging of imq_operator_apply give the same bits as the
    pinned single product, at a size with several staging chunks."""
    torch = pytest.importorskip("torch")
    from paper_2205_04194_b200 import inputs
    n = 1 << 21
    xy = inputs.uniform_points(n, 0)
    U = np.stack([inputs.random_vector(n, 100 + k) for k in range(3)])
    with imq.FastOperator(xy, 0.02, 12, 6) as op:
        ref = []
        pin_u = torch.empty(n, dtype=torch.float64).pin_memory()
        pin_b = torch.empty(n, dtype=torch.float64).pin_memory()
        for k in range(3):
            pin_u.copy_(torch.from_numpy(U[k]))
            imq.capi.check(imq.capi.lib().imq_operator_apply(
                op.handle, imq.api.C.cast(pin_u.data_ptr(), imq.api._dp),
                imq.api.C.cast(pin_b.data_ptr(), imq.api._dp)))
            ref.append(pin_b.numpy().copy())
        ref = np.stack(ref)
        assert np.array_equal(op.apply(U[1]), ref[1])          # pageable single
        assert np.array_equal(op.apply_batch(U), ref)          # pageable batch
        PU = torch.from_numpy(U).pin_memory()
        PB = torch.empty_like(PU).pin_memory()
        imq.capi.check(imq.capi.lib().imq_ext_operator_apply_batch(
            op.handle, 3, imq.api.C.cast(PU.data_ptr(), imq.api._dp),
            imq.api.C.cast(PB.data_ptr(), imq.api._dp)))
        assert np.array_equal(PB.numpy(), ref)                 # pinned batch
        assert np.array_equal(op.apply_batch(U[:1]), ref[:1])  # one row

def test_pageable_staging_odd_sizes_and_alignment(imq):
    """The streamed staging of pageable buffers (worker pool, non-temporal
    copies in 8 MB pieces): a length that leaves a partial last piece and
    parts that are not multiples of 64 bytes, and host pointers that are only
    8-byte aligned (the copy falls back to memcpy) -- same bits as the pinned
    product."""
    torch = pytest.importorskip("torch")
    from paper_2205_04194_b200 import inputs
    n = 1_300_003
    xy = inputs.uniform_points(n, 3)
    u = inputs.random_vector(n, 77)
    with imq.FastOperator(xy, 0.03, 8, 5) as op:
        pin_u = torch.from_numpy(u).pin_memory()
        pin_b = torch.empty(n, dtype=torch.float64).pin_memory()
        imq.capi.check(imq.capi.lib().imq_operator_apply(
            op.handle, imq.api.C.cast(pin_u.data_ptr(), imq.api._dp),
            imq.api.C.cast(pin_b.data_ptr(), imq.api._dp)))
        ref = pin_b.numpy().copy()
        assert np.array_equal(op.apply(u), ref)
        # 8-byte aligned but not 16-byte aligned views of pageable arrays
        base_u = np.empty(n + 3)
        off_u = 1 if base_u.ctypes.data % 16 == 0 else 0
        mu = base_u[off_u:off_u + n]
        mu[:] = u
        base_b = np.full(n + 3, np.nan)
        off_b = 1 if base_b.ctypes.data % 16 == 0 else 0
        mb = base_b[off_b:off_b + n]
        assert mu.ctypes.data % 16 == 8 and mb.ctypes.data % 16 == 8
        for _ in range(2):
            imq.capi.check(imq.capi.lib().imq_operator_apply(
                op.handle, mu.ctypes.data_as(imq.api._dp), mb.ctypes.data_as(imq.api._dp)))
            assert np.array_equal(mb, ref)
        # the guard elements around the output view are untouched
        assert np.isnan(base_b[:off_b]).all() and np.isnan(base_b[off_b + n:]).all()


@pytest.mark.parametrize("nrhs", [2, 3, 4, 7])
def test_block_product_bitwise_equals_single_products(imq, nrhs):
    """imq_ext_operator_apply_block (f4): groups of <= 4 vectors share the
    near field's kernel evaluations; every row equals the single product bit
    for bit (host matrices and device matrices), and the oracle rows to 1e-10."""
    torch = pytest.importorskip("torch")
    from paper_2205_04194_b200 import inputs
    n = 1 << 19
    xy = inputs.uniform_points(n, 3)
    U = np.stack([inputs.random_vector(n, 300 + k) for k in range(nrhs)])
    with imq.FastOperator(xy, 0.03, 12, 6) as op:
        ref = np.stack([op.apply(U[k]) for k in range(nrhs)])
        assert np.array_equal(op.apply_block(U), ref)            # pageable host matrices
        PU = torch.from_numpy(U).pin_memory()
        PB = torch.empty_like(PU).pin_memory()
        imq.capi.check(imq.capi.lib().imq_ext_operator_apply_block(
            op.handle, nrhs, imq.api.C.cast(PU.data_ptr(), imq.api._dp),
            imq.api.C.cast(PB.data_ptr(), imq.api._dp)))
        assert np.array_equal(PB.numpy(), ref)                   # pinned host matrices
        dU = torch.from_numpy(U).cuda()
        dB = torch.zeros_like(dU)
        op.apply_block_device(dU, dB, nrhs, torch.cuda.current_stream())
        torch.cuda.synchronize()
        assert np.array_equal(dB.cpu().numpy(), ref)             # device matrices
        assert np.array_equal(op.apply(U[0]), ref[0])            # single path intact afterwards


def test_block_product_other_near_modes(imq, oracle):
    """Operators whose near field is not the per-leaf symmetric kernel (large
    leaves: chunk pairs; tiny trees) take the block entry point vector by
    vector; rows equal the single products and the oracle."""
    from paper_2205_04194_b200 import inputs
    for n, levels in ((20000, 2), (3000, 1)):
        xy = inputs.uniform_points(n, 5)
        U = np.stack([inputs.random_vector(n, 40 + k) for k in range(3)])
        with imq.FastOperator(xy, 0.05, 10, levels) as op:
            B = op.apply_block(U)
            for k in range(3):
                assert np.array_equal(B[k], op.apply(U[k]))
        want = oracle.fast_matvec(xy, 0.05, 10, levels, U[2])
        assert np.max(np.abs(B[2] - want)) / np.max(np.abs(want)) <= 1e-10


@pytest.mark.parametrize("case", ["single_pass", "split_no_cheb", "cheb_nodes", "cheb_rings",
                                  "cheb_rings_xring", "clustered", "strip"])
def test_device_list_enumeration_matches_reference_lists(imq, case):
    """imq_verify's device check: every far pass of the operator (as built for
    the case) replayed per target through build_far_list gives each reference
    interaction-list entry (partition.cpp:56-72, non-empty blocks) exactly once
    -- in every enumeration mode (single pass; coarse + fine + per-leaf
    partial; Chebyshev node items; ring items; X-ring items)."""
    from paper_2205_04194_b200 import inputs
    rng = np.random.default_rng(17)
    n1 = 1 << 20
    cfg = {"single_pass": (inputs.uniform_points(4096, 0), 0.1, 10, 2, {}),
           "split_no_cheb": (inputs.uniform_points(20000, 1), 0.05, 8, 4, {}),
           "cheb_nodes": (inputs.uniform_points(n1, 0), 0.001, 16, 6, {"cheb_levels": 4, "cheb_ring": 0}),
           "cheb_rings": (inputs.uniform_points(n1, 0), 0.02, 16, 6, {"cheb_ring": 1, "cheb_xring": 0}),
           "cheb_rings_xring": (inputs.uniform_points(n1, 0), 0.04, 16, 6, {"cheb_ring": 1, "cheb_xring": 1}),
           "clustered": (inputs.gaussian_mixture(n1, 1), 0.02, 14, 6, {"cheb_ring": 1}),
           "strip": (np.stack([rng.random(n1), 0.3 + 0.01 * rng.random(n1)], 1).reshape(-1),
                     0.05, 12, 6, {})}[case]
    xy, t, m, L, want = cfg
    with imq.FastOperator(xy, t, m, L) as op:
        st = op.stats()
        for k, v in want.items():
            assert st[k] == v, (case, k, st[k])
        r = op.check_lists(4096)
    assert r["targets"] == min(4096, xy.size // 2)
    assert r["missing"] == 0 and r["duplicated"] == 0 and r["extra"] == 0, (case, r)
    assert r["max_entries"] > 0


def test_square_bits_match_oracle(imq, oracle):
    """The GPU bounding square (min/max reduction + host arithmetic,
    partition.cpp:9-23) equals the oracle's bit for bit."""
    from paper_2205_04194_b200 import inputs
    rng = np.random.default_rng(4)
    sets = [inputs.uniform_points(4096, 0), inputs.gaussian_mixture(50000, 1),
            1000.0 * rng.random(6000) - 12345.0,
            np.stack([rng.random(3000), 0.3 + 1e-7 * rng.random(3000)], 1).reshape(-1),
            np.tile([0.3, 0.4], 12)]
    for xy in sets:
        with imq.FastOperator(xy, 0.1, 6, 2) as op:
            st = op.stats()
        o = oracle.bounding_square(xy)
        got = (st["origin_x"], st["origin_y"], st["side"])
        assert all(np.float64(a).tobytes() == np.float64(b).tobytes() for a, b in zip(got, o)), (got, o)
