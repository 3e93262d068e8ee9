"""ctypes bindings for the parity checkers (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs import this module.  The product package
(paper_2205_04194_b200) never imports it.

Two checkers are exposed:
  * ``Oracle``    -- our C restatement (oracle/liboracle.so, imq_oracle.c);
  * ``Reference`` -- the reference's own C ABI (oracle/_ref/libimqfast_ref.so),
                    compiled from /root/reference/proj/src by oracle/Makefile.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_ORACLE = os.path.join(HERE, "liboracle.so")
LIB_REF = os.path.join(HERE, "_ref", "libimqfast_ref.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)


def _d(a):
    return a.ctypes.data_as(_dp)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class Oracle:
    """C restatement of the reference algorithm (see oracle/imq_oracle.c)."""

    def __init__(self, path: str = LIB_ORACLE):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = C.CDLL(path)
        L.ora_last_error.restype = C.c_char_p
        L.ora_random_vector.argtypes = [C.c_int64, C.c_uint64, _dp]
        L.ora_halton2d.argtypes = [C.c_int64, _dp]
        L.ora_rel_err_inf.argtypes = [_dp, _dp, C.c_int64]
        L.ora_rel_err_inf.restype = C.c_double
        L.ora_auto_level.argtypes = [C.c_int, C.c_int]
        L.ora_cost_upper_bound.argtypes = [C.c_int, C.c_int, C.c_int]
        L.ora_cost_upper_bound.restype = C.c_double
        L.ora_bounding_square.argtypes = [_dp, C.c_int64, _dp]
        L.ora_block_ids.argtypes = [_dp, C.c_int64, C.c_int, _i32p]
        L.ora_interaction_list.argtypes = [C.c_int, C.c_int, C.c_int, _i32p]
        L.ora_resolved_levels.argtypes = [C.c_int64, C.c_int, C.c_int]
        L.ora_fast_matvec.argtypes = [_dp, C.c_int64, C.c_double, C.c_int, C.c_int, _dp, _dp]
        L.ora_fast_matvec_rows.argtypes = [_dp, C.c_int64, C.c_double, C.c_int, C.c_int, _dp,
                                           _i64p, C.c_int64, _dp]
        L.ora_block_moments.argtypes = [_dp, C.c_int64, C.c_double, C.c_int, C.c_int, _dp,
                                        C.c_int, C.c_int, _dp, _dp]
        L.ora_dense_rows.argtypes = [_dp, C.c_int64, C.c_double, _dp, _i64p, C.c_int64, _dp]
        L.ora_dense_matvec.argtypes = [_dp, C.c_int64, C.c_double, _dp, _dp]
        L.ora_iterative_solve.argtypes = [_dp, C.c_int64, C.c_double, C.c_int, C.c_int, _dp,
                                          C.c_double, C.c_int, C.c_int, _dp, _ip, _dp, _ip, _dp,
                                          C.c_int, _ip]
        L.ora_evaluate_interpolant.argtypes = [_dp, _dp, C.c_int64, C.c_double, _dp, C.c_int64,
                                               _dp]
        self.lib = L

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(self.lib.ora_last_error().decode())

    def random_vector(self, n: int, seed: int) -> np.ndarray:
        out = np.empty(n)
        self._check(self.lib.ora_random_vector(n, seed, _d(out)))
        return out

    def halton2d(self, n: int) -> np.ndarray:
        out = np.empty(2 * n)
        self._check(self.lib.ora_halton2d(n, _d(out)))
        return out

    def auto_level(self, n: int, m: int) -> int:
        return self.lib.ora_auto_level(n, m)

    def cost_upper_bound(self, n: int, m: int, L: int) -> float:
        return self.lib.ora_cost_upper_bound(n, m, L)

    def bounding_square(self, xy) -> tuple:
        xy = _f64(xy)
        sq = np.empty(3)
        self._check(self.lib.ora_bounding_square(_d(xy), xy.size // 2, _d(sq)))
        return float(sq[0]), float(sq[1]), float(sq[2])

    def block_ids(self, xy, level: int) -> np.ndarray:
        xy = _f64(xy)
        out = np.empty(xy.size // 2, dtype=np.int32)
        self._check(self.lib.ora_block_ids(_d(xy), xy.size // 2, level,
                                           out.ctypes.data_as(_i32p)))
        return out

    def interaction_list(self, level: int, i: int, j: int) -> list:
        out = np.empty(64, dtype=np.int32)
        c = self.lib.ora_interaction_list(level, i, j, out.ctypes.data_as(_i32p))
        return [int(v) for v in out[:c]]

    def levels(self, n: int, m: int, L: int) -> int:
        return self.lib.ora_resolved_levels(n, m, L)

    def fast_matvec(self, xy, t, m, L, u) -> np.ndarray:
        xy, u = _f64(xy), _f64(u)
        b = np.empty(u.size)
        self._check(self.lib.ora_fast_matvec(_d(xy), u.size, t, m, L, _d(u), _d(b)))
        return b

    def fast_matvec_rows(self, xy, t, m, L, u, rows) -> np.ndarray:
        xy, u = _f64(xy), _f64(u)
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        b = np.empty(rows.size)
        self._check(self.lib.ora_fast_matvec_rows(_d(xy), u.size, t, m, L, _d(u),
                                                  rows.ctypes.data_as(_i64p), rows.size, _d(b)))
        return b

    def block_moments(self, xy, t, m, L, u, level, block):
        xy, u = _f64(xy), _f64(u)
        K = (m + 1) * (m + 2) // 2
        v, w = np.empty(K), np.empty(K)
        self._check(self.lib.ora_block_moments(_d(xy), u.size, t, m, L, _d(u), level, block,
                                               _d(v), _d(w)))
        return v, w

    def dense_matvec(self, xy, t, u, rows=None) -> np.ndarray:
        xy, u = _f64(xy), _f64(u)
        if rows is None:
            b = np.empty(u.size)
            self._check(self.lib.ora_dense_matvec(_d(xy), u.size, t, _d(u), _d(b)))
            return b
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        b = np.empty(rows.size)
        self._check(self.lib.ora_dense_rows(_d(xy), u.size, t, _d(u),
                                            rows.ctypes.data_as(_i64p), rows.size, _d(b)))
        return b

    def iterative_solve(self, xy, t, m, L, f, tol=1e-8, max_iter=500, restart=100):
        xy, f = _f64(xy), _f64(f)
        n = f.size
        c = np.empty(n)
        it, conv, ncyc = C.c_int(), C.c_int(), C.c_int()
        rel = C.c_double()
        cyc = np.empty(max_iter + 2)
        self._check(self.lib.ora_iterative_solve(
            _d(xy), n, t, m, L, _d(f), tol, max_iter, restart, _d(c), C.byref(it),
            C.byref(rel), C.byref(conv), _d(cyc), cyc.size, C.byref(ncyc)))
        return dict(c=c, iterations=it.value, final_relative_residual=rel.value,
                    converged=bool(conv.value), cycle_residuals=cyc[:ncyc.value].copy())

    def evaluate_interpolant(self, cxy, c, t, qxy):
        cxy, c, qxy = _f64(cxy), _f64(c), _f64(qxy)
        out = np.empty(qxy.size // 2)
        self._check(self.lib.ora_evaluate_interpolant(_d(cxy), _d(c), c.size, t, _d(qxy),
                                                      qxy.size // 2, _d(out)))
        return out


class imq_solve_stats(C.Structure):
    _fields_ = [("iterations", C.c_int), ("final_relative_residual", C.c_double),
                ("converged", C.c_int)]


class Reference:
    """The reference library itself through its C ABI (proj/include/imqfast.h)."""

    def __init__(self, path: str = LIB_REF):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` "
                                    "(needs /root/reference)")
        L = C.CDLL(path)
        L.imq_last_error.restype = C.c_char_p
        L.imq_operator_create.argtypes = [_dp, C.c_size_t, C.c_double, C.c_int, C.c_int,
                                          C.POINTER(C.c_void_p)]
        L.imq_operator_destroy.argtypes = [C.c_void_p]
        L.imq_operator_levels.argtypes = [C.c_void_p, _ip]
        L.imq_operator_apply.argtypes = [C.c_void_p, _dp, _dp]
        L.imq_dense_matvec.argtypes = [_dp, C.c_size_t, C.c_double, _dp, _dp]
        L.imq_iterative_solve.argtypes = [C.c_void_p, _dp, C.c_double, C.c_int, C.c_int, _dp,
                                          C.POINTER(imq_solve_stats)]
        L.imq_random_vector.argtypes = [C.c_size_t, C.c_ulonglong, _dp]
        L.imq_halton2d.argtypes = [C.c_size_t, _dp]
        L.imq_auto_level.argtypes = [C.c_size_t, C.c_int, _ip]
        L.imq_cost_upper_bound.argtypes = [C.c_size_t, C.c_int, C.c_int, _dp]
        L.imq_set_threads.argtypes = [C.c_int]
        self.lib = L

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(f"reference error {rc}: {self.lib.imq_last_error().decode()}")

    def set_threads(self, n: int):
        self._check(self.lib.imq_set_threads(n))

    def random_vector(self, n, seed):
        out = np.empty(n)
        self._check(self.lib.imq_random_vector(n, seed, _d(out)))
        return out

    def halton2d(self, n):
        out = np.empty(2 * n)
        self._check(self.lib.imq_halton2d(n, _d(out)))
        return out

    def auto_level(self, n, m):
        o = C.c_int()
        self._check(self.lib.imq_auto_level(n, m, C.byref(o)))
        return o.value

    def create(self, xy, t, m, levels):
        xy = _f64(xy)
        h = C.c_void_p()
        self._check(self.lib.imq_operator_create(_d(xy), xy.size // 2, t, m, levels,
                                                 C.byref(h)))
        return h

    def destroy(self, h):
        self.lib.imq_operator_destroy(h)

    def levels(self, h):
        o = C.c_int()
        self._check(self.lib.imq_operator_levels(h, C.byref(o)))
        return o.value

    def apply(self, h, u):
        u = _f64(u)
        b = np.empty(u.size)
        self._check(self.lib.imq_operator_apply(h, _d(u), _d(b)))
        return b

    def fast_matvec(self, xy, t, m, L, u):
        h = self.create(xy, t, m, L)
        try:
            return self.apply(h, u)
        finally:
            self.destroy(h)

    def dense_matvec(self, xy, t, u):
        xy, u = _f64(xy), _f64(u)
        b = np.empty(u.size)
        self._check(self.lib.imq_dense_matvec(_d(xy), u.size, t, _d(u), _d(b)))
        return b

    def iterative_solve(self, xy, t, m, L, f, tol, max_iter, restart):
        h = self.create(xy, t, m, L)
        try:
            f = _f64(f)
            c = np.empty(f.size)
            st = imq_solve_stats()
            self._check(self.lib.imq_iterative_solve(h, _d(f), tol, max_iter, restart, _d(c),
                                                     C.byref(st)))
            return dict(c=c, iterations=st.iterations,
                        final_relative_residual=st.final_relative_residual,
                        converged=bool(st.converged))
        finally:
            self.destroy(h)


def uniform_points(oracle_or_ref, n: int, seed: int) -> np.ndarray:
    """Appendix-A uniform points: (0.5+0.5 r[2i], 0.5+0.5 r[2i+1])."""
    r = oracle_or_ref.random_vector(2 * n, seed)
    return 0.5 + 0.5 * r
