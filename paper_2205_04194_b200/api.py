"""Python mirror of the reference C++ API over the C ABI (numpy / torch).

Names follow the reference (imq::build_operator / fast_matvec /
iterative_solve / dense_matvec / random_vector ..., proj/include/imq/*.hpp);
errors surface as ``IMQError`` carrying the reference's IMQ_ERR_* code.
All numerics run in libimqfast.so on the GPU; nothing here computes.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import capi
from .capi import IMQError, check, lib

_dp = C.POINTER(C.c_double)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


# ----------------------------------------------------------- host utilities
def random_vector(n: int, seed: int) -> np.ndarray:
    """reference.cpp:94-108: n uniform values on [-1, 1) from SplitMix64."""
    out = np.empty(n)
    check(lib().imq_random_vector(n, seed, _ptr(out)))
    return out


def halton2d(n: int) -> np.ndarray:
    out = np.empty(2 * n)
    check(lib().imq_halton2d(n, _ptr(out)))
    return out


def auto_level(n: int, m: int) -> int:
    o = C.c_int()
    check(lib().imq_auto_level(n, m, C.byref(o)))
    return o.value


def cost_upper_bound(n: int, m: int, levels: int) -> float:
    o = C.c_double()
    check(lib().imq_cost_upper_bound(n, m, levels, C.byref(o)))
    return o.value


def green_exact(x3, y3) -> float:
    x3, y3 = _f64(x3), _f64(y3)
    o = C.c_double()
    check(lib().imq_green_exact(_ptr(x3), _ptr(y3), C.byref(o)))
    return o.value


def green_truncated(x3, y3, m: int) -> float:
    x3, y3 = _f64(x3), _f64(y3)
    o = C.c_double()
    check(lib().imq_green_truncated(_ptr(x3), _ptr(y3), m, C.byref(o)))
    return o.value


def truncation_error_bound(rho_major: float, r: float, m: int) -> float:
    o = C.c_double()
    check(lib().imq_truncation_error_bound(rho_major, r, m, C.byref(o)))
    return o.value


def read_points(path: str) -> np.ndarray:
    p = _dp()
    n = C.c_size_t()
    check(lib().imq_read_points(path.encode(), C.byref(p), C.byref(n)))
    try:
        return np.ctypeslib.as_array(p, shape=(2 * n.value,)).copy() if n.value else np.empty(0)
    finally:
        lib().imq_free(C.cast(p, C.c_void_p))


def write_points(path: str, xy) -> None:
    xy = _f64(xy)
    check(lib().imq_write_points(path.encode(), _ptr(xy), xy.size // 2))


def set_threads(n: int) -> None:
    check(lib().imq_set_threads(n))


def device_count() -> int:
    o = C.c_int()
    check(lib().imq_ext_device_count(C.byref(o)))
    return o.value


def fp64_peak(iters: int = 4096):
    """(TFLOP/s, ms) of a dependency-free DFMA probe on the current device."""
    tf, ms = C.c_double(), C.c_double()
    check(lib().imq_ext_fp64_peak(iters, C.byref(tf), C.byref(ms)))
    return tf.value, ms.value


def set_device(d: int) -> None:
    check(lib().imq_ext_set_device(d))


# ------------------------------------------------------------- GPU compute
def dense_matvec(xy, t: float, u) -> np.ndarray:
    """reference.cpp:11-28 on the GPU (imq_dense_matvec)."""
    xy, u = _f64(xy), _f64(u)
    b = np.empty(u.size)
    check(lib().imq_dense_matvec(_ptr(xy), u.size, t, _ptr(u), _ptr(b)))
    return b


def evaluate_interpolant(centers_xy, c, t: float, x_xy) -> np.ndarray:
    """solver.cpp:161-172 on the GPU (imq_evaluate_interpolant)."""
    centers_xy, c, x_xy = _f64(centers_xy), _f64(c), _f64(x_xy)
    out = np.empty(x_xy.size // 2)
    check(lib().imq_evaluate_interpolant(_ptr(centers_xy), _ptr(c), c.size, t, _ptr(x_xy),
                                         out.size, _ptr(out)))
    return out


def dense_solve(xy, t: float, f):
    xy, f = _f64(xy), _f64(f)
    c = np.empty(f.size)
    r = C.c_double()
    check(lib().imq_dense_solve(_ptr(xy), f.size, t, _ptr(f), _ptr(c), C.byref(r)))
    return c, r.value


def verify(xy, t: float, m: int, levels: int = 0, seed: int = 42):
    """imq_verify: returns (n_failed, [(name, pass, value), ...])."""
    xy = _f64(xy)
    cfg = capi.imq_verify_config(_ptr(xy), xy.size // 2, t, m, levels, seed)
    rows = []

    def cb(name, ok, value, _ud):
        rows.append((name.decode(), bool(ok), value))

    cfun = capi.VERIFY_CB(cb)
    fails = lib().imq_verify(C.byref(cfg), cfun, None)
    if fails < 0:
        raise IMQError(-fails, lib().imq_last_error().decode())
    return fails, rows


@dataclass
class SolveReport:
    """solver.hpp:9-15"""
    c: np.ndarray
    iterations: int = 0
    final_relative_residual: float = 0.0
    converged: bool = False
    cycle_residuals: list = field(default_factory=list)


class FastOperator:
    """Device-resident fast IMQ operator (reference fastmv.hpp:19-38).

    ``levels <= 0`` selects auto_level(N, M) exactly like the reference.
    ``options`` (imq_ext_create_opts) may only disable approximations or make
    their gates stricter: ``flags`` is a list of names from ``capi.OPT``
    (e.g. ``["no_ring"]``), plus ``ring_tau`` / ``ring2_tau`` / ``inner_tau``
    / ``xring_tau`` and the scheduling-only ``far_rmax`` / ``far_streams``.
    """

    def __init__(self, xy, t: float, m: int, levels: int = 0, **options):
        xy = _f64(xy)
        h = C.c_void_p()
        if options:
            o = capi.imq_ext_options()
            for name in options.pop("flags", ()):
                o.flags |= capi.OPT[name]
            for k, v in options.items():
                setattr(o, k, v)
            check(lib().imq_ext_operator_create_opts(_ptr(xy), xy.size // 2, t, m, levels,
                                                     C.byref(o), C.byref(h)))
        else:
            check(lib().imq_operator_create(_ptr(xy), xy.size // 2, t, m, levels, C.byref(h)))
        self._h = h
        self.t = t
        self.m = m

    def close(self):
        if getattr(self, "_h", None):
            lib().imq_operator_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def handle(self):
        return self._h

    @property
    def size(self) -> int:
        o = C.c_size_t()
        check(lib().imq_operator_size(self._h, C.byref(o)))
        return o.value

    @property
    def levels(self) -> int:
        o = C.c_int()
        check(lib().imq_operator_levels(self._h, C.byref(o)))
        return o.value

    @property
    def order(self) -> int:
        """Truncation order M (imq_ext_stats.m)."""
        return int(self.stats()["m"])

    def apply(self, u) -> np.ndarray:
        """imq_operator_apply: host in, host out (fast_matvec, fastmv.cpp:184-217)."""
        u = _f64(u)
        if u.size != self.size:
            raise IMQError(capi.IMQ_ERR_INVALID_ARG, "fast_matvec: length mismatch")
        b = np.empty(u.size)
        check(lib().imq_operator_apply(self._h, _ptr(u), _ptr(b)))
        return b

    __call__ = apply

    def apply_batch(self, U) -> np.ndarray:
        """imq_ext_operator_apply_batch: rows of U (nrhs x N, host) -> rows of B,
        products pipelined with their host copies."""
        U = np.ascontiguousarray(np.atleast_2d(U), dtype=np.float64)
        if U.shape[1] != self.size:
            raise IMQError(capi.IMQ_ERR_INVALID_ARG, "apply_batch: length mismatch")
        B = np.empty_like(U)
        check(lib().imq_ext_operator_apply_batch(self._h, U.shape[0], _ptr(U), _ptr(B)))
        return B

    def apply_block(self, U) -> np.ndarray:
        """imq_ext_operator_apply_block: rows of U (nrhs x N, host) -> rows of B;
        groups of 4 vectors share the near field's kernel evaluations."""
        U = np.ascontiguousarray(np.atleast_2d(U), dtype=np.float64)
        if U.shape[1] != self.size:
            raise IMQError(capi.IMQ_ERR_INVALID_ARG, "apply_block: length mismatch")
        B = np.empty_like(U)
        check(lib().imq_ext_operator_apply_block(self._h, U.shape[0], _ptr(U), _ptr(B)))
        return B

    def apply_block_device(self, d_U, d_B, nrhs, stream=None) -> None:
        """Device matrices (nrhs x N row-major, original point order)."""
        check(lib().imq_ext_operator_apply_block_device(self._h, int(nrhs), _addr(d_U),
                                                        _addr(d_B), _stream(stream)))

    def apply_device(self, d_u, d_b, stream=None) -> None:
        """Device pointers (ints or torch CUDA tensors), original point order."""
        check(lib().imq_ext_operator_apply_device(self._h, _addr(d_u), _addr(d_b),
                                                  _stream(stream)))

    def apply_sorted_device(self, d_us, d_bs, stream=None) -> None:
        check(lib().imq_ext_operator_apply_sorted_device(self._h, _addr(d_us), _addr(d_bs),
                                                         _stream(stream)))

    def synchronize(self) -> None:
        check(lib().imq_ext_operator_synchronize(self._h))

    def permutation(self) -> np.ndarray:
        out = np.empty(self.size, dtype=np.int32)
        check(lib().imq_ext_operator_permutation(self._h, out.ctypes.data_as(C.POINTER(C.c_int))))
        return out

    def leaf_start(self) -> np.ndarray:
        n = (1 << (2 * (self.levels + 1))) + 1
        out = np.empty(n, dtype=np.int32)
        check(lib().imq_ext_operator_leaf_start(self._h, out.ctypes.data_as(C.POINTER(C.c_int)), n))
        return out

    def stats(self) -> dict:
        s = capi.imq_ext_stats()
        check(lib().imq_ext_operator_stats(self._h, C.byref(s)))
        out = {k: getattr(s, k) for k, _ in s._fields_}
        out["cert_by_kind"] = list(out["cert_by_kind"])
        return out

    def check_lists(self, max_targets: int = 4096) -> dict:
        """imq_ext_operator_check_lists: the device far-list enumeration of every
        pass vs the reference interaction lists."""
        o = (C.c_longlong * 5)()
        check(lib().imq_ext_operator_check_lists(self._h, max_targets, o))
        return dict(zip(("targets", "missing", "duplicated", "extra", "max_entries"), list(o)))

    def solve(self, f, tol: float = 1e-8, max_iter: int = 500, restart: int = 100) -> SolveReport:
        """imq_iterative_solve (solver.cpp:41-159) with the cycle residual history."""
        f = _f64(f)
        c = np.empty(f.size)
        st = capi.imq_solve_stats()
        cyc = np.empty(max(1, max_iter + 2))
        ncyc = C.c_int()
        check(lib().imq_ext_iterative_solve(self._h, _ptr(f), tol, max_iter, restart, _ptr(c),
                                            C.byref(st), _ptr(cyc), cyc.size, C.byref(ncyc)))
        return SolveReport(c=c, iterations=st.iterations,
                           final_relative_residual=st.final_relative_residual,
                           converged=bool(st.converged),
                           cycle_residuals=list(cyc[:min(ncyc.value, cyc.size)]))

    # --- stage-level access for sharded application (parallel.py)
    def moments(self, d_us, stream=None) -> None:
        check(lib().imq_ext_operator_moments(self._h, _addr(d_us), _stream(stream)))

    def coefficients(self):
        p = C.c_void_p()
        n = C.c_size_t()
        offs = (C.c_longlong * 16)()
        check(lib().imq_ext_operator_coefficients(self._h, C.byref(p), C.byref(n), offs, 16))
        return p.value, n.value, list(offs[: self.levels + 1])

    def items(self, which: str) -> np.ndarray:
        w = 0 if which == "far" else 1
        n = C.c_size_t()
        check(lib().imq_ext_operator_items(self._h, w, None, 0, C.byref(n)))
        out = np.empty((n.value, 4), dtype=np.int32)
        check(lib().imq_ext_operator_items(self._h, w, out.ctypes.data_as(C.POINTER(C.c_int)),
                                           n.value, C.byref(n)))
        return out

    def far_near(self, d_us, d_bs, far_range, near_range, stream=None, scatter=False) -> None:
        check(lib().imq_ext_operator_far_near(self._h, _addr(d_us), _addr(d_bs), far_range[0],
                                              far_range[1], near_range[0], near_range[1],
                                              1 if scatter else 0, _stream(stream)))

    def gather(self, d_u, d_us, stream=None) -> None:
        check(lib().imq_ext_operator_gather(self._h, _addr(d_u), _addr(d_us), _stream(stream)))

    def near_begin(self, d_us, stream=None) -> None:
        """Start the near field of d_us early (overlaps the moments); the next
        far_near uses it."""
        check(lib().imq_ext_operator_near_begin(self._h, _addr(d_us), _stream(stream)))

    def moments_local(self, d_us, stream=None) -> None:
        check(lib().imq_ext_operator_moments_local(self._h, _addr(d_us), _stream(stream)))

    def coarse_moments(self):
        """(device pointer, number of doubles) of the coarse moment region that
        sharded ranks all-reduce; 0 doubles when the operator is not sharded."""
        p = C.c_void_p()
        n = C.c_size_t()
        check(lib().imq_ext_operator_coarse_moments(self._h, C.byref(p), C.byref(n)))
        return p.value, n.value

    def moments_finish(self, stream=None) -> None:
        check(lib().imq_ext_operator_moments_finish(self._h, _stream(stream)))


def _addr(x) -> int:
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        if not x.is_cuda or not x.is_contiguous():
            raise ValueError("expected a contiguous CUDA tensor")
        return x.data_ptr()
    raise TypeError(f"cannot take a device address of {type(x)}")


def _stream(s):
    if s is None:
        return None
    if isinstance(s, int):
        return s
    return s.cuda_stream  # torch.cuda.Stream


def fast_matvec(op: FastOperator, u) -> np.ndarray:
    return op.apply(u)


def build_operator(xy, t: float, m: int, levels: int = 0) -> FastOperator:
    return FastOperator(xy, t, m, levels)


def iterative_solve(op: FastOperator, f, tol=1e-8, max_iter=500, restart=100) -> SolveReport:
    return op.solve(f, tol, max_iter, restart)
