"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/imqfast.h declares, host utilities match the reference, and
argument validation / error codes follow reference capi.cpp."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT


def test_every_declared_symbol_is_exported(imq):
    from paper_2205_04194_b200 import capi
    declared = capi.header_symbols()
    out = subprocess.run(["nm", "-D", "--defined-only", capi.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    # the 22 entry points of the reference header are all present
    ref22 = ["imq_last_error", "imq_operator_create", "imq_operator_destroy", "imq_operator_size",
             "imq_operator_levels", "imq_operator_apply", "imq_dense_matvec", "imq_dense_solve",
             "imq_iterative_solve", "imq_evaluate_interpolant", "imq_green_exact",
             "imq_green_truncated", "imq_truncation_error_bound", "imq_auto_level",
             "imq_cost_upper_bound", "imq_halton2d", "imq_random_vector", "imq_read_points",
             "imq_write_points", "imq_free", "imq_set_threads", "imq_verify"]
    assert set(ref22) <= exported


def test_library_sources_read_no_environment_variable():
    # include/imqfast.h: "The library reads no environment variables" -- a
    # caller's environment cannot change a product (options go through
    # imq_ext_operator_create_opts); no library (CUB / cuBLAS) in the sources
    csrc = os.path.join(ROOT, "paper_2205_04194_b200", "csrc")
    for f in sorted(os.listdir(csrc)):
        text = open(os.path.join(csrc, f)).read()
        assert "getenv" not in text, f
        assert "#include <cub" not in text and "cublas" not in text.lower(), f


def test_library_is_sm100a(imq):
    from paper_2205_04194_b200 import capi
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", capi.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_generators_match_reference(imq, golden):
    g = golden("gen")
    assert np.array_equal(imq.random_vector(64, 42), g["rv42"])
    assert np.array_equal(imq.random_vector(64, 1000), g["rv1000"])
    assert np.array_equal(imq.halton2d(64), g["halton"])
    for n, m, L in g["auto"]:
        assert imq.auto_level(int(n), int(m)) == L


def test_inputs_module_matches_reference_stream(golden):
    from paper_2205_04194_b200 import inputs
    g = golden("gen")
    assert np.array_equal(inputs.random_vector(64, 42), g["rv42"])
    c = golden("cfg1")
    assert np.array_equal(inputs.uniform_points(4096, 0), c["xy"])
    cl = golden("clustered")
    assert np.array_equal(inputs.gaussian_mixture(3000, 1), cl["xy"])
    xy = inputs.gaussian_mixture(20000, 1)
    assert xy.min() >= 0.0 and xy.max() <= 1.0


def test_cost_model(imq, oracle):
    # test_fastmv.cpp:12-35
    assert [imq.auto_level(n, 10) for n in (20000, 40000, 60000, 80000, 100000)] == [1, 2, 2, 2, 2]
    assert imq.auto_level(16, 10) == 1
    assert imq.cost_upper_bound(1000, 10, 1) == pytest.approx(1000.0 * (109.0 * 66 + 9.0 * 1000 / 16),
                                                              rel=1e-15)
    for n, m, L in ((50000, 14, 3), (4096, 10, 2)):
        assert imq.cost_upper_bound(n, m, L) == oracle.cost_upper_bound(n, m, L)


def test_green_functions_and_bound(imq):
    # expansion.cpp:19-56 semantics
    assert imq.green_exact([1, 1, 0.5], [0, 0, -0.5]) == pytest.approx(1 / np.sqrt(3))
    X, Y = [0.3, 0.2, 1.1], [0.05, -0.02, 0.1]
    exact = imq.green_exact(X, Y)
    assert abs(imq.green_truncated(X, Y, 20) - exact) < 1e-8
    assert imq.truncation_error_bound(2.0, 0.0, 5) == 0.0
    assert imq.truncation_error_bound(2.0, 0.5, 3) == pytest.approx(0.5 ** 4 / (2.0 * 0.5))
    with pytest.raises(imq.IMQError) as e:
        imq.green_exact([0, 0, 0], [0, 0, 0])
    assert e.value.code == 1
    with pytest.raises(imq.IMQError) as e:
        imq.truncation_error_bound(1.0, 1.0, 3)
    assert e.value.code == 1


def test_argument_validation_codes(imq):
    from paper_2205_04194_b200 import capi
    L = capi.lib()
    h = C.c_void_p()
    xy = np.array([0.1, 0.2, 0.3, 0.4])
    dp = xy.ctypes.data_as(C.POINTER(C.c_double))
    assert L.imq_operator_create(None, 2, 1.0, 4, 1, C.byref(h)) == 1
    assert L.imq_operator_create(dp, 0, 1.0, 4, 1, C.byref(h)) == 1
    assert L.imq_operator_create(dp, 2, 0.0, 4, 1, C.byref(h)) == 1
    assert b"shape parameter" in L.imq_last_error()
    assert L.imq_operator_create(dp, 2, float("nan"), 4, 1, C.byref(h)) == 1
    assert L.imq_operator_apply(None, dp, dp) == 1
    assert L.imq_set_threads(0) == 1
    assert L.imq_set_threads(4) == 0
    assert L.imq_auto_level(0, 10, C.byref(C.c_int())) == 1
    assert L.imq_random_vector(0, 1, dp) == 1
    L.imq_operator_destroy(None)  # NULL is a no-op
    out = C.c_double()
    assert L.imq_dense_matvec(dp, 2, -1.0, dp, C.cast(C.byref(out), C.POINTER(C.c_double))) == 1
    # options: negative / NaN gates and budgets are rejected before any device work
    o = capi.imq_ext_options()
    o.ring_tau = -1.0
    assert L.imq_ext_operator_create_opts(dp, 2, 1.0, 4, 1, C.byref(o), C.byref(h)) == 1
    o = capi.imq_ext_options()
    o.cert_budget = float("nan")
    assert L.imq_ext_operator_create_opts(dp, 2, 1.0, 4, 1, C.byref(o), C.byref(h)) == 1
    assert L.imq_ext_operator_create_opts(None, 2, 1.0, 4, 1, None, C.byref(h)) == 1


def test_point_file_io(imq, tmp_path):
    p = tmp_path / "pts.txt"
    xy = imq.halton2d(17)
    imq.write_points(str(p), xy)
    back = imq.read_points(str(p))
    assert np.array_equal(back, xy)
    (tmp_path / "bad.txt").write_text("# c\n0.1 0.2\n0.3\n")
    with pytest.raises(imq.IMQError) as e:
        imq.read_points(str(tmp_path / "bad.txt"))
    assert e.value.code == 3 and "malformed line 3" in e.value.msg
    with pytest.raises(imq.IMQError) as e:
        imq.read_points(str(tmp_path / "missing.txt"))
    assert e.value.code == 3


def test_dense_solve_host(imq):
    # test_solver.cpp:72-91 style: small well-conditioned system
    xy = imq.halton2d(16)
    x, y = xy[0::2], xy[1::2]
    f = np.exp(x) * np.sin(3 * y) + x * y
    c, res = imq.dense_solve(xy, 1.0, f)
    assert res <= 1e-10
    with pytest.raises(imq.IMQError) as e:
        imq.dense_solve(xy, 1.0, np.zeros(16))
    assert e.value.code == 1


def test_no_cpu_fallback_without_gpu(imq):
    """Without a CUDA device the compute entry points fail loudly."""
    if imq.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(imq.IMQError) as e:
        imq.FastOperator(imq.halton2d(10), 1.0, 4, 1)
    assert e.value.code == 4 and "no CPU fallback" in e.value.msg
    with pytest.raises(imq.IMQError):
        imq.dense_matvec(imq.halton2d(10), 1.0, np.ones(10))
