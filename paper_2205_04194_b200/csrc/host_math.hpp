// host_math.hpp -- host-side numerics of the library (off the GPU hot path).
//
// These are B200-library re-implementations of the reference's small host
// utilities, with the reference's semantics and error behaviour:
//   random_vector / halton2d      reference.cpp:77-108
//   auto_level / cost_upper_bound fastmv.cpp:13-30
//   bounding square arithmetic    partition.cpp:18-22
//   Legendre table, d_{n,m}       specfun.cpp:26-37,73-91
//   Green's function helpers      expansion.cpp:19-56, geometry.cpp:21-37
//   point-file I/O                reference.cpp:110-136
//   dense LU solve                reference.cpp:30-64 (partial-pivot LU + 1 refinement)
// plus the tables the device pipeline needs (mu -> C transform, binomials).
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace imqh {

struct singular_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline int order_K(int M) { return (M + 1) * (M + 2) / 2; }
int order_Ke(int M);  // #{(n, m) : n - m even, 0 <= m <= n <= M}
int mu_offset(int M, int m);
// Far-field coefficient layout ("Horner order"): groups m = M..0, inside a
// group k = top(m)..m.  C_{m,M} vanishes identically when M - m is odd (no n
// with n = m mod 2 fits in [M, min(M, 2M - m)]), so such groups start at M-1.
inline int horner_top(int M, int m) { return M - ((M - m) & 1); }
inline int horner_count(int M) { return order_K(M) - (M + 1) / 2; }
inline int horner_index(int M, int m, int k) {
  int o = 0;
  for (int mm = M; mm > m; --mm) o += horner_top(M, mm) - mm + 1;
  return o + (horner_top(M, m) - k);
}

void check_t(double t);  // expansion.cpp:11-13
void check_M(int M);     // specfun.cpp:8-10

std::vector<double> random_vector(int64_t n, uint64_t seed);
std::vector<double> halton2d(int64_t n);

int auto_level(int N, int M);
double cost_upper_bound(int N, int M, int L);

// origin.x, origin.y, side from the coordinate extrema (partition.cpp:18-22).
void square_from_extrema(double minx, double maxx, double miny, double maxy, double sq[3]);

void legendre_table(int M, double x, double sin_theta, double* out);
double coeff_d(int n, int m);

double green_exact(const double* X, const double* Y);
double green_truncated(const double* X, const double* Y, int M);
double truncation_error_bound(double rho_major, double r, int M);

std::vector<double> read_points(const std::string& path);  // interleaved
void write_points(const std::string& path, const double* xy, size_t n);

// Transform table (CSR over Horner slots): C[o] = sum val[e] * mu[idx[e]].
struct Transform {
  std::vector<int> off, idx;
  std::vector<double> val;
};
Transform build_transform(int M, double t);
std::vector<double> binomials(int M);  // [(M+1) x (M+1)], C(a, p)
// Per-level tables of the fused M2M (k_m2m_tr), interleaved complex:
// V[c][a][p] = C(a,p) d_c^{a-p} (a, p <= M) followed by
// W[c][b][r] = C(b,r) conj(d_c)^{b-r} (b, r <= M/2), d_c = (+-h) + i (+-h)
// child c at x offset (c >> 1 ? +h : -h), y offset (c & 1 ? +h : -h), the
// Morton child order.  Evaluated in long double.
std::vector<double> m2m_tables(int M, double h);

// Dense solve: A = [1/sqrt(t^2+|xi-xj|^2)], n <= 5000 (reference.cpp:30-46),
// partial-pivot LU + one refinement step, residual guard 1e-10 (48-64).
std::vector<double> dense_solve(const double* xy, size_t n, double t, const double* f,
                                double* residual_out);

// Separation check of partition.cpp:117-141 for the uniform-depth grid.
struct Separation {
  double max_ratio, max_ratio_level1;
  bool valid;
};
Separation verify_separation(const double sq[3], int L, double t);

}  // namespace imqh
