// host_math.cpp -- see host_math.hpp.  Compiled with -ffp-contract=off so the
// bounding-square arithmetic matches the reference bit for bit.
#include "host_math.hpp"

#include <algorithm>
#include <cmath>
#include <fstream>
#include <sstream>

namespace imqh {

int order_Ke(int M) {
  int s = 0;
  for (int n = 0; n <= M; ++n) s += n / 2 + 1;
  return s;
}
int mu_offset(int M, int m) {
  int o = 0;
  for (int mm = 0; mm < m; ++mm) o += (M - mm) / 2 + 1;
  return o;
}

void check_t(double t) {
  if (!(t > 0.0) || !std::isfinite(t))
    throw std::invalid_argument("shape parameter t must be positive and finite");
}
void check_M(int M) {
  if (M < 0) throw std::invalid_argument("truncation index M must be >= 0");
}

// reference.cpp:94-108
std::vector<double> random_vector(int64_t n, uint64_t seed) {
  if (n < 1) throw std::invalid_argument("random_vector: N must be >= 1");
  std::vector<double> u((size_t)n);
  uint64_t state = seed;
  for (int64_t i = 0; i < n; ++i) {
    state += 0x9E3779B97F4A7C15ull;
    uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    u[(size_t)i] = 2.0 * ((double)(z >> 11) * 0x1.0p-53) - 1.0;
  }
  return u;
}

// reference.cpp:77-92
static double radical_inverse(int64_t index, int base) {
  double r = 0.0, denom = 1.0;
  while (index > 0) {
    denom *= base;
    r += (double)(index % base) / denom;
    index /= base;
  }
  return r;
}
std::vector<double> halton2d(int64_t n) {
  if (n < 1) throw std::invalid_argument("halton2d: N must be >= 1");
  std::vector<double> xy(2 * (size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    xy[2 * (size_t)i] = radical_inverse(i + 1, 2);
    xy[2 * (size_t)i + 1] = radical_inverse(i + 1, 3);
  }
  return xy;
}

// fastmv.cpp:13-24
int auto_level(int N, int M) {
  if (N < 1) throw std::invalid_argument("auto_level: N must be >= 1");
  check_M(M);
  const double alpha = 2.0 * 109.0 * order_K(M);
  const double beta = 2.25 * N;
  const double lam = std::log(beta * std::log(4.0) / alpha) / std::log(4.0);
  const int lmax =
      std::max(1, static_cast<int>(std::floor(std::log(static_cast<double>(N)) / std::log(4.0))) - 1);
  auto g = [&](int L) { return alpha * L + beta * std::pow(4.0, -L); };
  const int lo = std::clamp(static_cast<int>(std::floor(lam)), 1, lmax);
  const int hi = std::clamp(static_cast<int>(std::ceil(lam)), 1, lmax);
  return g(hi) < g(lo) ? hi : lo;
}
// fastmv.cpp:26-30
double cost_upper_bound(int N, int M, int L) {
  if (N < 1 || L < 1) throw std::invalid_argument("cost_upper_bound: need N >= 1, L >= 1");
  check_M(M);
  return N * (109.0 * order_K(M) * L + 9.0 * N / std::pow(4.0, L + 1));
}

// partition.cpp:18-22
void square_from_extrema(double minx, double maxx, double miny, double maxy, double sq[3]) {
  const double dx = maxx - minx, dy = maxy - miny;
  double side = std::max(dx, dy);
  side = side > 0.0 ? side * (1.0 + 1e-9) : 1e-9;
  sq[0] = minx - 0.5 * (side - dx);
  sq[1] = miny - 0.5 * (side - dy);
  sq[2] = side;
}

static inline int flat(int n, int m) { return n * (n + 1) / 2 + m; }

// specfun.cpp:73-91
void legendre_table(int M, double x, double sin_theta, double* out) {
  if (M < 0) throw std::invalid_argument("assoc_legendre_table: M < 0");
  if (!(x >= -1.0 && x <= 1.0))
    throw std::invalid_argument("Legendre argument must satisfy |x| <= 1");
  double pmm = 1.0;
  for (int m = 0; m <= M; ++m) {
    if (m > 0) pmm *= -(2.0 * m - 1.0) * sin_theta;
    out[flat(m, m)] = pmm;
    if (m == M) break;
    double prev2 = pmm;
    double prev1 = x * (2.0 * m + 1.0) * pmm;
    out[flat(m + 1, m)] = prev1;
    for (int n = m + 2; n <= M; ++n) {
      const double p = ((2.0 * n - 1.0) * x * prev1 - (n + m - 1.0) * prev2) / (n - m);
      out[flat(n, m)] = p;
      prev2 = prev1;
      prev1 = p;
    }
  }
}
// specfun.cpp:26-37
double coeff_d(int n, int m) {
  double d = m == 0 ? 1.0 : 2.0;
  for (int k = n - m + 1; k <= n + m; ++k) d /= static_cast<double>(k);
  return d;
}

// geometry.cpp:21-37 (to_spherical), expansion.cpp:19-48
struct Sph {
  double rho, theta, omega;
};
static Sph to_sph(const double* v) {
  const double rho = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
  if (rho == 0.0) return {0.0, 2.0 * std::atan(1.0), 0.0};
  double c = v[2] / rho;
  c = std::min(1.0, std::max(-1.0, c));
  const double theta = std::acos(c);
  double omega = std::atan2(v[1], v[0]);
  if (omega < 0.0) omega += 8.0 * std::atan(1.0);
  if (omega < 0.0) omega = 0.0;
  return {rho, theta, omega};
}
double green_exact(const double* X, const double* Y) {
  const double d[3] = {X[0] - Y[0], X[1] - Y[1], X[2] - Y[2]};
  const double r = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
  if (r == 0.0) throw std::invalid_argument("green_exact: X = Y is singular");
  return 1.0 / r;
}
double green_truncated(const double* X, const double* Y, int M) {
  if (M < 0) throw std::invalid_argument("green_truncated: M < 0");
  const Sph sx = to_sph(X), sy = to_sph(Y);
  if (sx.rho == sy.rho)
    throw std::invalid_argument("green_truncated: expansion undefined for ||X|| = ||Y||");
  double rmin = sx.rho, rmax = sy.rho;
  if (rmin > rmax) std::swap(rmin, rmax);
  std::vector<double> px((size_t)order_K(M)), py((size_t)order_K(M));
  legendre_table(M, std::cos(sx.theta), std::sin(sx.theta), px.data());
  legendre_table(M, std::cos(sy.theta), std::sin(sy.theta), py.data());
  const double dom = sx.omega - sy.omega;
  double sum = 0.0, ratio_pow = 1.0;
  const double inv_major = 1.0 / rmax;
  for (int n = 0; n <= M; ++n) {
    const double radial = ratio_pow * inv_major;
    for (int m = 0; m <= n; ++m) {
      const int k = flat(n, m);
      sum += coeff_d(n, m) * py[(size_t)k] * px[(size_t)k] * std::cos(m * dom) * radial;
    }
    ratio_pow *= rmin * inv_major;
  }
  return sum;
}
// expansion.cpp:50-56
double truncation_error_bound(double rho_major, double r, int M) {
  if (M < 0) throw std::invalid_argument("truncation_error_bound: M < 0");
  if (!(rho_major > 0.0))
    throw std::invalid_argument("truncation_error_bound: rho_major must be positive");
  if (r == 0.0) return 0.0;
  if (!(r > 0.0 && r < 1.0))
    throw std::invalid_argument("truncation_error_bound: need 0 <= r < 1");
  return std::pow(r, M + 1) / (rho_major * (1.0 - r));
}

// reference.cpp:110-136
std::vector<double> read_points(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("read_points: cannot open " + path);
  std::vector<double> xy;
  std::string line;
  int lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    const size_t pos = line.find_first_not_of(" \t\r");
    if (pos == std::string::npos || line[pos] == '#') continue;
    std::istringstream ss(line);
    double x, y;
    std::string extra;
    if (!(ss >> x >> y) || (ss >> extra))
      throw std::runtime_error("read_points: malformed line " + std::to_string(lineno) + " in " +
                               path);
    xy.push_back(x);
    xy.push_back(y);
  }
  return xy;
}
void write_points(const std::string& path, const double* xy, size_t n) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("write_points: cannot open " + path);
  out.precision(17);
  for (size_t i = 0; i < n; ++i) out << xy[2 * i] << ' ' << xy[2 * i + 1] << '\n';
  if (!out) throw std::runtime_error("write_points: write failure on " + path);
}

// -------------------------------------------------------- transform table --
// C_{m,k} = sum_{n} d_{n,m} P_n^m(0) pi_{n,m,n-k} t^{2k-n-m} mu_{m,(n-m)/2},
// n in [k, min(M, 2k-m)], n = m (mod 2), where pi_{n,m,j} is the coefficient of
// x^{n-m-2j} in (-1)^m d^m/dx^m P_n(x):
//   pi_{n,m,j} = (-1)^(m+j) C(n,j) C(2n-2j,n) (n-2j)!/(n-2j-m)! / 2^n.
// Derivation: P_n^m(x) = sin^m(theta) (-1)^m D^m P_n(x), x = t/rho,
// sin(theta) e^{-i m w} = conj(dx + i dy)/rho; see DESIGN.md §3.
Transform build_transform(int M, double t) {
  const int K = horner_count(M);
  std::vector<long double> pascal((size_t)(2 * M + 2) * (2 * M + 2), 0.0L);
  auto Cb = [&](int a, int b) -> long double & { return pascal[(size_t)a * (2 * M + 2) + b]; };
  for (int a = 0; a <= 2 * M + 1; ++a) {
    Cb(a, 0) = 1.0L;
    for (int b = 1; b <= a; ++b) Cb(a, b) = Cb(a - 1, b - 1) + (b <= a - 1 ? Cb(a - 1, b) : 0.0L);
  }
  std::vector<double> pn0((size_t)order_K(M));
  legendre_table(M, 0.0, 1.0, pn0.data());
  Transform T;
  T.off.assign((size_t)K + 1, 0);
  std::vector<std::vector<std::pair<int, double>>> rows((size_t)K);
  for (int m = 0; m <= M; ++m)
    for (int k = m; k <= horner_top(M, m); ++k) {
      const int o = horner_index(M, m, k);
      for (int n = k; n <= std::min(M, 2 * k - m); ++n) {
        if ((n - m) % 2) continue;
        const int j = n - k;
        long double pi = Cb(n, j) * Cb(2 * n - 2 * j, n);
        for (int s = 0; s < m; ++s) pi *= (long double)(n - 2 * j - s);
        pi = std::ldexp(pi, -n);
        if ((m + j) % 2) pi = -pi;
        long double v = pi * (long double)coeff_d(n, m) * (long double)pn0[(size_t)flat(n, m)] *
                        std::pow((long double)t, (long double)(2 * k - n - m));
        rows[(size_t)o].push_back({mu_offset(M, m) + (n - m) / 2, (double)v});
      }
    }
  for (int o = 0; o < K; ++o) {
    T.off[(size_t)o + 1] = T.off[(size_t)o] + (int)rows[(size_t)o].size();
    for (auto& e : rows[(size_t)o]) {
      T.idx.push_back(e.first);
      T.val.push_back(e.second);
    }
  }
  if (T.idx.empty()) {  // keep device allocations non-empty
    T.idx.push_back(0);
    T.val.push_back(0.0);
  }
  return T;
}

std::vector<double> binomials(int M) {
  std::vector<double> b((size_t)(M + 1) * (M + 1), 0.0);
  for (int a = 0; a <= M; ++a) {
    b[(size_t)a * (M + 1)] = 1.0;
    for (int p = 1; p <= a; ++p)
      b[(size_t)a * (M + 1) + p] =
          b[(size_t)(a - 1) * (M + 1) + p - 1] + (p <= a - 1 ? b[(size_t)(a - 1) * (M + 1) + p] : 0.0);
  }
  return b;
}

// mu'_{a,b} = sum_c sum_{p<=a, r<=b} C(a,p) C(b,r) d_c^{a-p} conj(d_c)^{b-r} N^c_{p,r},
// N_{p,r} = mu_{p-r,r} (p >= r) or conj(mu_{r-p,p}); a = m+i, b = i.  The m = 0
// outputs are real in exact arithmetic; their imaginary column is left zero.
std::vector<double> m2m_tables(int M, double h) {
  const int M1 = M + 1, H1 = M / 2 + 1;
  std::vector<double> out((size_t)2 * 4 * (M1 * M1 + H1 * H1), 0.0);
  std::vector<long double> bn((size_t)M1 * M1, 0.0L);
  for (int a = 0; a <= M; ++a) {
    bn[(size_t)a * M1] = 1.0L;
    for (int p = 1; p <= a; ++p)
      bn[(size_t)a * M1 + p] = bn[(size_t)(a - 1) * M1 + p - 1] + (p <= a - 1 ? bn[(size_t)(a - 1) * M1 + p] : 0.0L);
  }
  for (int c = 0; c < 4; ++c) {
    const long double dx = (c >> 1) ? h : -h, dy = (c & 1) ? h : -h;
    std::vector<long double> pr((size_t)M1), pi((size_t)M1);  // d^k
    pr[0] = 1.0L;
    pi[0] = 0.0L;
    for (int k = 1; k <= M; ++k) {
      pr[(size_t)k] = pr[(size_t)k - 1] * dx - pi[(size_t)k - 1] * dy;
      pi[(size_t)k] = pr[(size_t)k - 1] * dy + pi[(size_t)k - 1] * dx;
    }
    for (int a = 0; a <= M; ++a)
      for (int p = 0; p <= a; ++p) {
        const size_t o = 2 * ((size_t)c * M1 * M1 + (size_t)a * M1 + p);
        out[o] = (double)(bn[(size_t)a * M1 + p] * pr[(size_t)(a - p)]);
        out[o + 1] = (double)(bn[(size_t)a * M1 + p] * pi[(size_t)(a - p)]);
      }
    const size_t wbase = (size_t)4 * M1 * M1;
    for (int b = 0; b < H1; ++b)
      for (int r = 0; r <= b; ++r) {
        const size_t o = 2 * (wbase + (size_t)c * H1 * H1 + (size_t)b * H1 + r);
        out[o] = (double)(bn[(size_t)b * M1 + r] * pr[(size_t)(b - r)]);
        out[o + 1] = (double)(-bn[(size_t)b * M1 + r] * pi[(size_t)(b - r)]);
      }
  }
  return out;
}


// ----------------------------------------------------------- dense solve --
std::vector<double> dense_solve(const double* xy, size_t n, double t, const double* f,
                                double* residual_out) {
  check_t(t);
  if (n > 5000) throw std::invalid_argument("assemble_dense: N exceeds the memory cap");
  const size_t N = n;
  std::vector<double> A(N * N), LU;
  const double inv_t = 1.0 / t;
  for (size_t i = 0; i < N; ++i) {
    A[i * N + i] = inv_t;
    for (size_t j = i + 1; j < N; ++j) {
      const double dx = xy[2 * i] - xy[2 * j], dy = xy[2 * i + 1] - xy[2 * j + 1];
      const double v = 1.0 / std::sqrt(t * t + (dx * dx + dy * dy));
      A[i * N + j] = v;
      A[j * N + i] = v;
    }
  }
  LU = A;
  std::vector<size_t> piv(N);
  for (size_t k = 0; k < N; ++k) {
    size_t p = k;
    double best = std::fabs(LU[k * N + k]);
    for (size_t i = k + 1; i < N; ++i)
      if (std::fabs(LU[i * N + k]) > best) {
        best = std::fabs(LU[i * N + k]);
        p = i;
      }
    piv[k] = p;
    if (p != k)
      for (size_t j = 0; j < N; ++j) std::swap(LU[k * N + j], LU[p * N + j]);
    const double d = LU[k * N + k];
    for (size_t i = k + 1; i < N; ++i) {
      const double l = LU[i * N + k] / d;
      LU[i * N + k] = l;
      double* ri = &LU[i * N];
      const double* rk = &LU[k * N];
      for (size_t j = k + 1; j < N; ++j) ri[j] -= l * rk[j];
    }
  }
  auto lu_solve = [&](std::vector<double> b) {
    for (size_t k = 0; k < N; ++k) std::swap(b[k], b[piv[k]]);
    for (size_t i = 0; i < N; ++i)
      for (size_t j = 0; j < i; ++j) b[i] -= LU[i * N + j] * b[j];
    for (size_t i = N; i-- > 0;) {
      for (size_t j = i + 1; j < N; ++j) b[i] -= LU[i * N + j] * b[j];
      b[i] /= LU[i * N + i];
    }
    return b;
  };
  std::vector<double> fv(f, f + N);
  std::vector<double> c = lu_solve(fv);
  std::vector<double> r(N);
  for (size_t i = 0; i < N; ++i) {
    double s = 0.0;
    for (size_t j = 0; j < N; ++j) s += A[i * N + j] * c[j];
    r[i] = fv[i] - s;
  }
  std::vector<double> dc = lu_solve(r);
  for (size_t i = 0; i < N; ++i) c[i] += dc[i];
  double fnorm = 0.0, res = 0.0;
  for (size_t i = 0; i < N; ++i) fnorm = std::max(fnorm, std::fabs(fv[i]));
  if (fnorm == 0.0) throw std::invalid_argument("dense_solve: zero right-hand side");
  for (size_t i = 0; i < N; ++i) {
    double s = 0.0;
    for (size_t j = 0; j < N; ++j) s += A[i * N + j] * c[j];
    res = std::max(res, std::fabs(s - fv[i]));
  }
  res /= fnorm;
  if (!(res <= 1e-10))
    throw singular_error("dense_solve: numerically singular matrix (relative residual " +
                         std::to_string(res) + " exceeds 1e-10)");
  if (residual_out) *residual_out = res;
  return c;
}

// --------------------------------------------------------- separation ----
// partition.cpp:117-141 over the enumerated interaction lists.
Separation verify_separation(const double sq[3], int L, double t) {
  if (t < 0.0) throw std::invalid_argument("verify_separation: t must be >= 0");
  Separation rep{0.0, 0.0, true};
  for (int l = 1; l <= L; ++l) {
    const int grid = 1 << (l + 1);
    const double cell = sq[2] / grid;
    const double rho_yz = cell * std::sqrt(0.5);
    for (int pi = 0; pi < grid; ++pi)
      for (int pj = 0; pj < grid; ++pj) {
        const double zx = sq[0] + (pi + 0.5) * cell, zy = sq[1] + (pj + 0.5) * cell;
        int lo_i = 0, hi_i = grid - 1, lo_j = 0, hi_j = grid - 1;
        if (l >= 2) {
          lo_i = std::max(0, 2 * (pi / 2 - 1));
          hi_i = std::min(grid - 1, 2 * (pi / 2 + 1) + 1);
          lo_j = std::max(0, 2 * (pj / 2 - 1));
          hi_j = std::min(grid - 1, 2 * (pj / 2 + 1) + 1);
        }
        for (int qi = lo_i; qi <= hi_i; ++qi)
          for (int qj = lo_j; qj <= hi_j; ++qj) {
            if (std::max(std::abs(qi - pi), std::abs(qj - pj)) < 2) continue;
            const double x0 = sq[0] + qi * cell, y0 = sq[1] + qj * cell;
            const double dx = std::max({x0 - zx, 0.0, zx - (x0 + cell)});
            const double dy = std::max({y0 - zy, 0.0, zy - (y0 + cell)});
            const double planar = std::sqrt(dx * dx + dy * dy);
            const double rho_xz = std::sqrt(planar * planar + t * t);
            const double ratio = rho_yz / rho_xz;
            rep.max_ratio = std::max(rep.max_ratio, ratio);
            if (l == 1) rep.max_ratio_level1 = std::max(rep.max_ratio_level1, ratio);
          }
      }
  }
  rep.valid = rep.max_ratio < 0.5;
  return rep;
}

}  // namespace imqh
