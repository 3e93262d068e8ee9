"""B200-native fast inverse-multiquadric matvec + GMRES (arXiv 2205.04194).

The product is libimqfast.so (CUDA, sm_100a) behind the reference's C ABI
(include/imqfast.h); this package is its Python mirror.
"""
from .api import (FastOperator, SolveReport, auto_level, build_operator, cost_upper_bound,
                  dense_matvec, dense_solve, device_count, evaluate_interpolant, fast_matvec,
                  green_exact, green_truncated, halton2d, iterative_solve, random_vector,
                  read_points, set_device, set_threads, truncation_error_bound, verify,
                  write_points)
from .capi import IMQError

__all__ = ["FastOperator", "SolveReport", "IMQError", "auto_level", "build_operator",
           "cost_upper_bound", "dense_matvec", "dense_solve", "device_count",
           "evaluate_interpolant", "fast_matvec", "green_exact", "green_truncated", "halton2d",
           "iterative_solve", "random_vector", "read_points", "set_device", "set_threads",
           "truncation_error_bound", "verify", "write_points"]
