// capi.cpp -- the C ABI (include/imqfast.h), replacing reference
// proj/src/capi.cpp.  Same validation order, error codes, thread-local error
// string and exception -> code mapping (capi.cpp:30-52); compute goes to the
// device operator, host utilities to host_math.
#include "imqfast.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "host_math.hpp"
#include "imq_kernels.hpp"
#include "operator.hpp"

struct imq_operator {
  std::unique_ptr<imqh::DeviceOperator> op;
};

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* msg) {
  g_last_error = msg;
  return code;
}

// reference capi.cpp:39-52
template <typename F>
int guard(F&& fn, int runtime_code = IMQ_ERR_INTERNAL) {
  try {
    return fn();
  } catch (const imqh::singular_error& e) {
    return fail(IMQ_ERR_SINGULAR, e.what());
  } catch (const std::invalid_argument& e) {
    return fail(IMQ_ERR_INVALID_ARG, e.what());
  } catch (const std::bad_alloc&) {
    return fail(IMQ_ERR_INTERNAL, "out of memory");
  } catch (const std::exception& e) {
    return fail(runtime_code, e.what());
  }
}

void require_device() {
  int nd = 0;
  if (cudaGetDeviceCount(&nd) != cudaSuccess || nd == 0) {
    cudaGetLastError();
    throw imqh::cuda_error("no CUDA device available: the B200 build has no CPU fallback");
  }
}

// Dense / interpolant product on the device: out[q] = sum_j c_j phi(x_q, y_j).
void direct_product(const double* sxy, const double* c, size_t ns, double t, const double* txy,
                    size_t nt, double* out) {
  require_device();
  if (nt == 0) return;
  cudaStream_t s = cudaStreamPerThread;
  double *d_s = nullptr, *d_c = nullptr, *d_t = nullptr, *d_o = nullptr;
  auto freeall = [&] {
    if (d_s) cudaFree(d_s);
    if (d_c) cudaFree(d_c);
    if (d_t) cudaFree(d_t);
    if (d_o) cudaFree(d_o);
  };
  try {
    imqh::cuda_check(cudaMalloc(&d_s, 2 * ns * sizeof(double)), "direct alloc");
    imqh::cuda_check(cudaMalloc(&d_c, ns * sizeof(double)), "direct alloc");
    imqh::cuda_check(cudaMalloc(&d_t, 2 * nt * sizeof(double)), "direct alloc");
    imqh::cuda_check(cudaMalloc(&d_o, nt * sizeof(double)), "direct alloc");
    imqh::cuda_check(cudaMemcpyAsync(d_s, sxy, 2 * ns * sizeof(double), cudaMemcpyHostToDevice, s), "H2D");
    imqh::cuda_check(cudaMemcpyAsync(d_c, c, ns * sizeof(double), cudaMemcpyHostToDevice, s), "H2D");
    imqh::cuda_check(cudaMemcpyAsync(d_t, txy, 2 * nt * sizeof(double), cudaMemcpyHostToDevice, s), "H2D");
    imqk::launch_direct(d_t, (long long)nt, d_s, d_c, (long long)ns, t * t, d_o, s);
    imqh::cuda_check(cudaGetLastError(), "direct kernel");
    imqh::cuda_check(cudaMemcpyAsync(out, d_o, nt * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
    imqh::cuda_check(cudaStreamSynchronize(s), "direct");
  } catch (...) {
    freeall();
    throw;
  }
  freeall();
}

double rel_err_inf(const std::vector<double>& a, const std::vector<double>& b) {
  double num = 0.0, den = 0.0;
  for (size_t i = 0; i < b.size(); ++i) {
    num = std::max(num, std::fabs(a[i] - b[i]));
    den = std::max(den, std::fabs(b[i]));
  }
  if (den == 0.0) throw std::invalid_argument("rel_err_inf: reference vector is identically zero");
  return num / den;
}

// Host bucketing of a small point set (partition.cpp:25-54) for exact_cover.
int exact_cover_deviation(const double* xy, size_t n, int L) {
  double mnx = xy[0], mxx = xy[0], mny = xy[1], mxy = xy[1];
  for (size_t i = 0; i < n; ++i) {
    mnx = std::min(mnx, xy[2 * i]); mxx = std::max(mxx, xy[2 * i]);
    mny = std::min(mny, xy[2 * i + 1]); mxy = std::max(mxy, xy[2 * i + 1]);
  }
  double sq[3];
  imqh::square_from_extrema(mnx, mxx, mny, mxy, sq);
  auto bid = [&](int l, size_t p, int& i, int& j) {
    const int g = 1 << (l + 1);
    const double cell = sq[2] / g;
    i = std::clamp((int)std::floor((xy[2 * p] - sq[0]) / cell), 0, g - 1);
    j = std::clamp((int)std::floor((xy[2 * p + 1] - sq[1]) / cell), 0, g - 1);
  };
  std::vector<int> count(n * n, 0);
  for (size_t a = 0; a < n; ++a)
    for (size_t b = 0; b < n; ++b) {
      for (int l = 1; l <= L; ++l) {
        int ai, aj, bi, bj;
        bid(l, a, ai, aj);
        bid(l, b, bi, bj);
        if (std::max(std::abs(ai - bi), std::abs(aj - bj)) < 2) continue;
        if (l >= 2 && std::max(std::abs(ai / 2 - bi / 2), std::abs(aj / 2 - bj / 2)) > 1) continue;
        ++count[a * n + b];
      }
      int ai, aj, bi, bj;
      bid(L, a, ai, aj);
      bid(L, b, bi, bj);
      if (std::max(std::abs(ai - bi), std::abs(aj - bj)) <= 1) ++count[a * n + b];
    }
  int dev = 0;
  for (int c : count) dev = std::max(dev, std::abs(c - 1));
  return dev;
}

}  // namespace

extern "C" {

const char* imq_last_error(void) { return g_last_error.c_str(); }

int imq_operator_create(const double* xy, size_t n, double t, int m, int levels,
                        imq_operator** out) {
  if (!xy || !out || n == 0)
    return fail(IMQ_ERR_INVALID_ARG, "imq_operator_create: null argument or empty point set");
  *out = nullptr;
  return guard([&] {
    auto holder = std::make_unique<imq_operator>();
    holder->op = std::make_unique<imqh::DeviceOperator>(xy, n, t, m, levels);
    *out = holder.release();
    return IMQ_OK;
  });
}

int imq_ext_operator_create_opts(const double* xy, size_t n, double t, int m, int levels,
                                 const imq_ext_options* opts, imq_operator** out) {
  if (!xy || !out || n == 0)
    return fail(IMQ_ERR_INVALID_ARG, "imq_ext_operator_create_opts: null argument or empty point set");
  *out = nullptr;
  imqh::OperatorOptions o;
  if (opts) {
    if (!(opts->ring_tau >= 0) || !(opts->ring2_tau >= 0) || !(opts->inner_tau >= 0) ||
        !(opts->xring_tau >= 0) || !(opts->cert_budget >= 0) || opts->far_rmax < 0 ||
        opts->far_streams < 0)
      return fail(IMQ_ERR_INVALID_ARG, "imq_ext_operator_create_opts: negative or NaN option");
    o.flags = opts->flags;
    o.ring_tau = opts->ring_tau;
    o.ring2_tau = opts->ring2_tau;
    o.inner_tau = opts->inner_tau;
    o.xring_tau = opts->xring_tau;
    o.far_rmax = opts->far_rmax;
    o.far_streams = opts->far_streams;
    o.cert_budget = opts->cert_budget;
  }
  return guard([&] {
    auto holder = std::make_unique<imq_operator>();
    holder->op = std::make_unique<imqh::DeviceOperator>(xy, n, t, m, levels, o);
    *out = holder.release();
    return IMQ_OK;
  });
}

void imq_operator_destroy(imq_operator* op) { delete op; }

int imq_operator_size(const imq_operator* op, size_t* out) {
  if (!op || !out) return fail(IMQ_ERR_INVALID_ARG, "imq_operator_size: null argument");
  *out = (size_t)op->op->size();
  return IMQ_OK;
}

int imq_operator_levels(const imq_operator* op, int* out) {
  if (!op || !out) return fail(IMQ_ERR_INVALID_ARG, "imq_operator_levels: null argument");
  *out = op->op->levels();
  return IMQ_OK;
}

int imq_operator_apply(const imq_operator* op, const double* u, double* b_out) {
  if (!op || !u || !b_out) return fail(IMQ_ERR_INVALID_ARG, "imq_operator_apply: null argument");
  return guard([&] {
    op->op->apply_host(u, b_out);
    return IMQ_OK;
  });
}

int imq_ext_operator_apply_batch(const imq_operator* op, int nrhs, const double* U, double* B) {
  if (!op || !U || !B) return fail(IMQ_ERR_INVALID_ARG, "imq_ext_operator_apply_batch: null argument");
  if (nrhs < 1) return fail(IMQ_ERR_INVALID_ARG, "imq_ext_operator_apply_batch: nrhs must be >= 1");
  return guard([&] {
    op->op->apply_batch(nrhs, U, B);
    return IMQ_OK;
  });
}

int imq_ext_operator_apply_block(const imq_operator* op, int nrhs, const double* U, double* B) {
  if (!op || !U || !B) return fail(IMQ_ERR_INVALID_ARG, "imq_ext_operator_apply_block: null argument");
  if (nrhs < 1) return fail(IMQ_ERR_INVALID_ARG, "imq_ext_operator_apply_block: nrhs must be >= 1");
  return guard([&] {
    op->op->apply_block_host(nrhs, U, B);
    return IMQ_OK;
  });
}

int imq_ext_operator_apply_block_device(const imq_operator* op, int nrhs, const double* d_U,
                                        double* d_B, void* stream) {
  if (!op || !d_U || !d_B)
    return fail(IMQ_ERR_INVALID_ARG, "imq_ext_operator_apply_block_device: null argument");
  if (nrhs < 1)
    return fail(IMQ_ERR_INVALID_ARG, "imq_ext_operator_apply_block_device: nrhs must be >= 1");
  return guard([&] {
    op->op->apply_block_device(nrhs, d_U, d_B, static_cast<cudaStream_t>(stream));
    return IMQ_OK;
  });
}

int imq_dense_matvec(const double* xy, size_t n, double t, const double* u, double* b_out) {
  if (!xy || !u || !b_out || n == 0)
    return fail(IMQ_ERR_INVALID_ARG, "imq_dense_matvec: null argument or empty point set");
  return guard([&] {
    imqh::check_t(t);
    direct_product(xy, u, n, t, xy, n, b_out);
    return IMQ_OK;
  });
}

int imq_dense_solve(const double* xy, size_t n, double t, const double* f, double* c_out,
                    double* residual_out) {
  if (!xy || !f || !c_out || n == 0)
    return fail(IMQ_ERR_INVALID_ARG, "imq_dense_solve: null argument or empty point set");
  return guard([&] {
    std::vector<double> c = imqh::dense_solve(xy, n, t, f, residual_out);
    std::copy(c.begin(), c.end(), c_out);
    return IMQ_OK;
  });
}

int imq_iterative_solve(const imq_operator* op, const double* f, double tol, int max_iter,
                        int restart, double* c_out, imq_solve_stats* stats_out) {
  if (!op || !f || !c_out) return fail(IMQ_ERR_INVALID_ARG, "imq_iterative_solve: null argument");
  return guard([&] {
    imqh::SolveResult r = op->op->solve_host(f, tol, max_iter, restart, c_out);
    if (stats_out) {
      stats_out->iterations = r.iterations;
      stats_out->final_relative_residual = r.final_relative_residual;
      stats_out->converged = r.converged ? 1 : 0;
    }
    return IMQ_OK;
  });
}

int imq_evaluate_interpolant(const double* centers_xy, const double* c, size_t n, double t,
                             const double* x_xy, size_t nx, double* out) {
  if (!centers_xy || !c || !x_xy || !out || n == 0)
    return fail(IMQ_ERR_INVALID_ARG, "imq_evaluate_interpolant: null argument");
  return guard([&] {
    imqh::check_t(t);
    direct_product(centers_xy, c, n, t, x_xy, nx, out);
    return IMQ_OK;
  });
}

int imq_green_exact(const double* x3, const double* y3, double* out) {
  if (!x3 || !y3 || !out) return fail(IMQ_ERR_INVALID_ARG, "imq_green_exact: null argument");
  return guard([&] {
    *out = imqh::green_exact(x3, y3);
    return IMQ_OK;
  });
}

int imq_green_truncated(const double* x3, const double* y3, int m, double* out) {
  if (!x3 || !y3 || !out) return fail(IMQ_ERR_INVALID_ARG, "imq_green_truncated: null argument");
  return guard([&] {
    *out = imqh::green_truncated(x3, y3, m);
    return IMQ_OK;
  });
}

int imq_truncation_error_bound(double rho_major, double r, int m, double* out) {
  if (!out) return fail(IMQ_ERR_INVALID_ARG, "imq_truncation_error_bound: null argument");
  return guard([&] {
    *out = imqh::truncation_error_bound(rho_major, r, m);
    return IMQ_OK;
  });
}

int imq_auto_level(size_t n, int m, int* out) {
  if (!out || n == 0 || n > ((size_t)1 << 31))
    return fail(IMQ_ERR_INVALID_ARG, "imq_auto_level: bad argument");
  return guard([&] {
    *out = imqh::auto_level((int)n, m);
    return IMQ_OK;
  });
}

int imq_cost_upper_bound(size_t n, int m, int levels, double* out) {
  if (!out || n == 0 || n > ((size_t)1 << 31))
    return fail(IMQ_ERR_INVALID_ARG, "imq_cost_upper_bound: bad argument");
  return guard([&] {
    *out = imqh::cost_upper_bound((int)n, m, levels);
    return IMQ_OK;
  });
}

int imq_halton2d(size_t n, double* xy_out) {
  if (!xy_out || n == 0 || n > ((size_t)1 << 31))
    return fail(IMQ_ERR_INVALID_ARG, "imq_halton2d: bad argument");
  return guard([&] {
    std::vector<double> v = imqh::halton2d((int64_t)n);
    std::copy(v.begin(), v.end(), xy_out);
    return IMQ_OK;
  });
}

int imq_random_vector(size_t n, unsigned long long seed, double* out) {
  if (!out || n == 0 || n > ((size_t)1 << 31))
    return fail(IMQ_ERR_INVALID_ARG, "imq_random_vector: bad argument");
  return guard([&] {
    std::vector<double> v = imqh::random_vector((int64_t)n, seed);
    std::copy(v.begin(), v.end(), out);
    return IMQ_OK;
  });
}

int imq_read_points(const char* path, double** xy_out, size_t* n_out) {
  if (!path || !xy_out || !n_out) return fail(IMQ_ERR_INVALID_ARG, "imq_read_points: null argument");
  *xy_out = nullptr;
  *n_out = 0;
  return guard(
      [&] {
        std::vector<double> xy = imqh::read_points(path);
        double* buf = static_cast<double*>(std::malloc(std::max<size_t>(1, xy.size()) * sizeof(double)));
        if (!buf) throw std::bad_alloc();
        std::copy(xy.begin(), xy.end(), buf);
        *xy_out = buf;
        *n_out = xy.size() / 2;
        return IMQ_OK;
      },
      IMQ_ERR_IO);
}

int imq_write_points(const char* path, const double* xy, size_t n) {
  if (!path || (!xy && n > 0)) return fail(IMQ_ERR_INVALID_ARG, "imq_write_points: null argument");
  return guard(
      [&] {
        imqh::write_points(path, xy, n);
        return IMQ_OK;
      },
      IMQ_ERR_IO);
}

void imq_free(void* p) { std::free(p); }

static int g_threads = 1;
int imq_set_threads(int n) {
  if (n < 1) return fail(IMQ_ERR_INVALID_ARG, "imq_set_threads: n must be >= 1");
  g_threads = n;  // device kernels are not thread-count dependent
  return IMQ_OK;
}

// reference capi.cpp:300-394, same eight named checks in the same order.
int imq_verify(const imq_verify_config* cfg, imq_verify_callback cb, void* user_data) {
  if (!cfg || !cfg->xy || cfg->n == 0) {
    fail(IMQ_ERR_INVALID_ARG, "imq_verify: null or empty configuration");
    return -IMQ_ERR_INVALID_ARG;
  }
  try {
    int fails = 0;
    auto report = [&](const char* name, bool pass, double value) {
      if (!pass) ++fails;
      if (cb) cb(name, pass ? 1 : 0, value, user_data);
    };
    imqh::check_t(cfg->t);
    imqh::DeviceOperator op(cfg->xy, cfg->n, cfg->t, cfg->m, cfg->levels);
    const imqh::Separation sep = imqh::verify_separation(op.square(), op.levels(), cfg->t);
    report("separation_ratio", sep.valid, sep.max_ratio);
    const imqh::Separation sep0 = imqh::verify_separation(op.square(), op.levels(), 0.0);
    report("separation_ratio_planar", sep0.valid, sep0.max_ratio);
    {
      // list sizes of every block of every level (partition.cpp:56-83: the
      // reference counts its built slist / near_lists, empty blocks included):
      // the 6 x 6 candidate window of the parent's neighbourhood (level 1: the
      // whole 4 x 4 grid) minus the Chebyshev-distance < 2 part; near lists are
      // the clipped 3 x 3 neighbourhoods of the finest level
      int max_far = 0, max_near = 0;
      bool within = true;
      for (int l = 1; l <= op.levels(); ++l) {
        const int grid = 1 << (l + 1), cap = l == 1 ? 12 : 27;
        for (int i = 0; i < grid; ++i)
          for (int j = 0; j < grid; ++j) {
            const int li = l == 1 ? 0 : std::max(0, 2 * (i / 2) - 2);
            const int hi = l == 1 ? grid - 1 : std::min(grid - 1, 2 * (i / 2) + 3);
            const int lj = l == 1 ? 0 : std::max(0, 2 * (j / 2) - 2);
            const int hj = l == 1 ? grid - 1 : std::min(grid - 1, 2 * (j / 2) + 3);
            const int win = (hi - li + 1) * (hj - lj + 1);
            const int ni = std::min(grid - 1, i + 1) - std::max(0, i - 1) + 1;
            const int nj = std::min(grid - 1, j + 1) - std::max(0, j - 1) + 1;
            const int c = win - ni * nj;  // the 3 x 3 neighbourhood lies inside the window
            max_far = std::max(max_far, c);
            if (c > cap) within = false;
            if (l == op.levels()) max_near = std::max(max_near, ni * nj);
          }
      }
      if (max_near > 9) within = false;
      report("interaction_counts", within, (double)std::max(max_far, max_near));
    }
    {
      const size_t nsub = std::min<size_t>(cfg->n, 200);
      int dev = 0;
      for (int L = 1; L <= 3; ++L) dev = std::max(dev, exact_cover_deviation(cfg->xy, nsub, L));
      // the device enumeration: every far pass of this operator replayed per
      // target (k_far_cover) must produce each reference list entry exactly
      // once (all targets up to 4096, else 4096 spread over the set)
      const imqh::ListCheck lc = op.far_list_check(4096);
      dev = std::max(dev, lc.max_deviation);
      report("exact_cover", dev == 0, (double)dev);
    }
    {
      const size_t nsub = std::min<size_t>(cfg->n, 2000);
      std::unique_ptr<imqh::DeviceOperator> sub;
      imqh::DeviceOperator* o = &op;
      if (nsub != cfg->n) {
        sub = std::make_unique<imqh::DeviceOperator>(cfg->xy, nsub, cfg->t, cfg->m, cfg->levels);
        o = sub.get();
      }
      std::vector<double> u = imqh::random_vector((int64_t)nsub, cfg->seed);
      std::vector<double> bf(nsub), bd(nsub);
      o->apply_host(u.data(), bf.data());
      direct_product(cfg->xy, u.data(), nsub, cfg->t, cfg->xy, nsub, bd.data());
      const double rel = rel_err_inf(bf, bd);
      report("oracle_equivalence", rel <= 5e-8, rel);

      // m = 0 sine moments vanish identically: our moments are
      // mu_{0,i} = sum u |e|^{2i}, whose imaginary part is exactly zero.
      std::vector<double> u1 = imqh::random_vector((int64_t)nsub, cfg->seed + 1);
      {
        double* d = nullptr;
        imqh::cuda_check(cudaMalloc(&d, nsub * sizeof(double)), "verify alloc");
        imqh::cuda_check(cudaMemcpy(d, u1.data(), nsub * sizeof(double), cudaMemcpyHostToDevice), "H2D");
        std::vector<int> perm(nsub);
        o->copy_permutation(perm.data());
        std::vector<double> us(nsub);
        for (size_t p = 0; p < nsub; ++p) us[p] = u1[(size_t)perm[p]];
        imqh::cuda_check(cudaMemcpy(d, us.data(), nsub * sizeof(double), cudaMemcpyHostToDevice), "H2D");
        o->moments(d, o->stream());
        imqh::cuda_check(cudaStreamSynchronize(o->stream()), "verify moments");
        const imqk::TreeParams& P = o->params();
        std::vector<double2> coef(o->coef_count());
        imqh::cuda_check(cudaMemcpy(coef.data(), o->coef_ptr(), coef.size() * sizeof(double2),
                                    cudaMemcpyDeviceToHost), "D2H coef");
        cudaFree(d);
        std::vector<int> ls;
        o->copy_leaf_start(ls);
        double worst = 0.0;
        for (int l = 1; l <= P.L; ++l) {
          const long long nb = 1ll << (2 * (l + 1));
          const int sh = 2 * (P.L - l);
          for (long long q = 0; q < nb; ++q) {
            if (ls[(size_t)(q + 1) << sh] == ls[(size_t)q << sh]) continue;
            for (int k = 0; k <= imqh::horner_top(P.M, 0); ++k) {
              const double2 v = coef[(size_t)P.coef_off[l] + (size_t)q * P.K +
                                     (size_t)imqh::horner_index(P.M, 0, k)];
              worst = std::max(worst, std::fabs(v.y));
            }
          }
        }
        report("m0_sine_moments", worst == 0.0, worst);
      }
      std::vector<double> u2 = imqh::random_vector((int64_t)nsub, cfg->seed + 2);
      const double alpha = 0.7, beta = -1.3;
      std::vector<double> mix(nsub), b1(nsub), b2(nsub), bm(nsub), ref(nsub), b1bis(nsub);
      for (size_t i = 0; i < nsub; ++i) mix[i] = alpha * u1[i] + beta * u2[i];
      o->apply_host(u1.data(), b1.data());
      o->apply_host(u2.data(), b2.data());
      o->apply_host(mix.data(), bm.data());
      for (size_t i = 0; i < nsub; ++i) ref[i] = alpha * b1[i] + beta * b2[i];
      const double lin = rel_err_inf(bm, ref);
      report("linearity", lin <= 1e-12, lin);
      o->apply_host(u1.data(), b1bis.data());
      double dmax = 0.0;
      for (size_t i = 0; i < nsub; ++i) dmax = std::max(dmax, std::fabs(b1bis[i] - b1[i]));
      report("determinism", dmax == 0.0, dmax);
    }
    return fails;
  } catch (const std::invalid_argument& e) {
    fail(IMQ_ERR_INVALID_ARG, e.what());
    return -IMQ_ERR_INVALID_ARG;
  } catch (const std::bad_alloc&) {
    fail(IMQ_ERR_INTERNAL, "out of memory");
    return -IMQ_ERR_INTERNAL;
  } catch (const std::exception& e) {
    fail(IMQ_ERR_INTERNAL, e.what());
    return -IMQ_ERR_INTERNAL;
  }
}

// ------------------------------------------------------------ extensions --

int imq_ext_operator_apply_device(const imq_operator* op, const double* d_u, double* d_b,
                                  void* stream) {
  if (!op || !d_u || !d_b) return fail(IMQ_ERR_INVALID_ARG, "imq_ext_operator_apply_device: null argument");
  return guard([&] {
    op->op->apply_device(d_u, d_b, static_cast<cudaStream_t>(stream));
    return IMQ_OK;
  });
}

int imq_ext_operator_apply_sorted_device(const imq_operator* op, const double* d_us,
                                         double* d_bs, void* stream) {
  if (!op || !d_us || !d_bs)
    return fail(IMQ_ERR_INVALID_ARG, "imq_ext_operator_apply_sorted_device: null argument");
  return guard([&] {
    op->op->apply_sorted(d_us, d_bs, static_cast<cudaStream_t>(stream));
    return IMQ_OK;
  });
}

int imq_ext_operator_synchronize(const imq_operator* op) {
  if (!op) return fail(IMQ_ERR_INVALID_ARG, "imq_ext_operator_synchronize: null argument");
  return guard([&] {
    imqh::cuda_check(cudaStreamSynchronize(op->op->stream()), "synchronize");
    imqh::cuda_check(cudaGetLastError(), "synchronize");
    return IMQ_OK;
  });
}

int imq_ext_operator_permutation(const imq_operator* op, int* perm_out) {
  if (!op || !perm_out) return fail(IMQ_ERR_INVALID_ARG, "imq_ext_operator_permutation: null argument");
  return guard([&] {
    op->op->copy_permutation(perm_out);
    return IMQ_OK;
  });
}

int imq_ext_operator_leaf_start(const imq_operator* op, int* out, size_t capacity) {
  if (!op || !out) return fail(IMQ_ERR_INVALID_ARG, "imq_ext_operator_leaf_start: null argument");
  return guard([&] {
    std::vector<int> ls;
    op->op->copy_leaf_start(ls);
    if (capacity < ls.size()) throw std::invalid_argument("imq_ext_operator_leaf_start: capacity too small");
    std::copy(ls.begin(), ls.end(), out);
    return IMQ_OK;
  });
}

int imq_ext_operator_stats(const imq_operator* op, imq_ext_stats* out) {
  if (!op || !out) return fail(IMQ_ERR_INVALID_ARG, "imq_ext_operator_stats: null argument");
  return guard([&] {
    imqh::PairCounts c = op->op->pair_counts();
    out->n = op->op->size();
    out->m = op->op->order();
    out->levels = op->op->levels();
    out->device = op->op->device();
    out->origin_x = op->op->square()[0];
    out->origin_y = op->op->square()[1];
    out->side = op->op->square()[2];
    out->far_pairs = c.far_pairs;
    out->near_pairs = c.near_pairs;
    out->far_items = c.far_items;
    out->near_items = c.near_items;
    out->near_mode = c.near_mode;
    out->far_pairs_direct = c.far_pairs_direct;
    out->cheb_node_pairs = c.cheb_node_pairs;
    out->cheb_levels = c.cheb_levels;
    out->cheb_ring = c.cheb_ring;
    out->kernel_launches = c.kernel_launches;
    out->cheb_xring = c.cheb_xring;
    const imqh::CertReport& r = op->op->certificate();
    out->cert_estimate = r.estimate;
    out->cert_budget = r.budget;
    out->cert_scale = r.scale;
    for (int k = 0; k < 5; ++k) out->cert_by_kind[k] = r.by_kind[k];
    out->cert_fallbacks = r.fallbacks;
    out->cert_rounds = r.rounds;
    out->gemm_node_pairs = c.gemm_node_pairs;
    return IMQ_OK;
  });
}

int imq_ext_iterative_solve(const imq_operator* op, const double* f, double tol, int max_iter,
                            int restart, double* c_out, imq_solve_stats* stats_out,
                            double* cycle_out, int max_cycles, int* n_cycles) {
  if (!op || !f || !c_out) return fail(IMQ_ERR_INVALID_ARG, "imq_ext_iterative_solve: null argument");
  return guard([&] {
    imqh::SolveResult r = op->op->solve_host(f, tol, max_iter, restart, c_out);
    if (stats_out) {
      stats_out->iterations = r.iterations;
      stats_out->final_relative_residual = r.final_relative_residual;
      stats_out->converged = r.converged ? 1 : 0;
    }
    if (cycle_out)
      for (int i = 0; i < std::min(max_cycles, (int)r.cycle_residuals.size()); ++i)
        cycle_out[i] = r.cycle_residuals[(size_t)i];
    if (n_cycles) *n_cycles = (int)r.cycle_residuals.size();
    return IMQ_OK;
  });
}

int imq_ext_operator_moments(const imq_operator* op, const double* d_us, void* stream) {
  if (!op || !d_us) return fail(IMQ_ERR_INVALID_ARG, "imq_ext_operator_moments: null argument");
  return guard([&] {
    op->op->moments_locked(d_us, static_cast<cudaStream_t>(stream));
    imqh::cuda_check(cudaGetLastError(), "moments launch");
    return IMQ_OK;
  });
}

int imq_ext_operator_gather(const imq_operator* op, const double* d_u, double* d_us,
                            void* stream) {
  if (!op || !d_u || !d_us) return fail(IMQ_ERR_INVALID_ARG, "imq_ext_operator_gather: null argument");
  return guard([&] {
    op->op->gather(d_u, d_us, static_cast<cudaStream_t>(stream));
    imqh::cuda_check(cudaGetLastError(), "gather launch");
    return IMQ_OK;
  });
}

int imq_ext_operator_near_begin(const imq_operator* op, const double* d_us, void* stream) {
  if (!op || !d_us) return fail(IMQ_ERR_INVALID_ARG, "imq_ext_operator_near_begin: null argument");
  return guard([&] {
    op->op->near_begin(d_us, static_cast<cudaStream_t>(stream));
    imqh::cuda_check(cudaGetLastError(), "near_begin launch");
    return IMQ_OK;
  });
}

int imq_ext_operator_moments_local(const imq_operator* op, const double* d_us, void* stream) {
  if (!op || !d_us) return fail(IMQ_ERR_INVALID_ARG, "imq_ext_operator_moments_local: null argument");
  return guard([&] {
    op->op->moments_local(d_us, static_cast<cudaStream_t>(stream));
    imqh::cuda_check(cudaGetLastError(), "moments_local launch");
    return IMQ_OK;
  });
}

int imq_ext_operator_coarse_moments(const imq_operator* op, void** d_ptr, size_t* n_doubles) {
  if (!op || !d_ptr || !n_doubles)
    return fail(IMQ_ERR_INVALID_ARG, "imq_ext_operator_coarse_moments: null argument");
  double2* p = nullptr;
  size_t n = 0;
  op->op->coarse_moments(&p, &n);
  *d_ptr = p;
  *n_doubles = 2 * n;
  return IMQ_OK;
}

int imq_ext_operator_moments_finish(const imq_operator* op, void* stream) {
  if (!op) return fail(IMQ_ERR_INVALID_ARG, "imq_ext_operator_moments_finish: null argument");
  return guard([&] {
    op->op->moments_finish(static_cast<cudaStream_t>(stream));
    imqh::cuda_check(cudaGetLastError(), "moments_finish launch");
    return IMQ_OK;
  });
}

int imq_ext_operator_coefficients(const imq_operator* op, void** d_coef, size_t* count,
                                  long long* level_offsets, int capacity) {
  if (!op || !d_coef || !count)
    return fail(IMQ_ERR_INVALID_ARG, "imq_ext_operator_coefficients: null argument");
  *d_coef = op->op->coef_ptr();
  *count = op->op->coef_count();
  const imqk::TreeParams& P = op->op->params();
  if (level_offsets)
    for (int l = 0; l <= P.L && l < capacity; ++l) level_offsets[l] = l == 0 ? 0 : P.coef_off[l];
  return IMQ_OK;
}

int imq_ext_operator_items(const imq_operator* op, int which, int* items_xyzw, size_t capacity,
                           size_t* count) {
  if (!op || !count) return fail(IMQ_ERR_INVALID_ARG, "imq_ext_operator_items: null argument");
  const std::vector<int4>& v = which == 0 ? op->op->far_items_host() : op->op->near_items_host();
  *count = v.size();
  if (items_xyzw) {
    if (capacity < v.size()) return fail(IMQ_ERR_INVALID_ARG, "imq_ext_operator_items: capacity too small");
    std::memcpy(items_xyzw, v.data(), v.size() * sizeof(int4));
  }
  return IMQ_OK;
}

int imq_ext_operator_check_lists(const imq_operator* op, int max_targets, long long* out5) {
  if (!op || !out5 || max_targets < 1)
    return fail(IMQ_ERR_INVALID_ARG, "imq_ext_operator_check_lists: bad argument");
  return guard([&] {
    const imqh::ListCheck r = op->op->far_list_check(max_targets);
    out5[0] = r.targets;
    out5[1] = r.missing;
    out5[2] = r.duplicated;
    out5[3] = r.extra;
    out5[4] = r.max_entries;
    return IMQ_OK;
  });
}

int imq_ext_operator_local_leaves(const imq_operator* op, int* out, size_t capacity,
                                  size_t* count) {
  if (!op || !count) return fail(IMQ_ERR_INVALID_ARG, "imq_ext_operator_local_leaves: null argument");
  const std::vector<int>& v = op->op->local_leaves_host();
  *count = v.size();
  if (out) {
    if (capacity < v.size()) return fail(IMQ_ERR_INVALID_ARG, "imq_ext_operator_local_leaves: capacity too small");
    std::memcpy(out, v.data(), v.size() * sizeof(int));
  }
  return IMQ_OK;
}

int imq_ext_operator_far_near(const imq_operator* op, const double* d_us, double* d_bs,
                              int far_begin, int far_end, int near_begin, int near_end,
                              int scatter, void* stream) {
  if (!op || !d_us || !d_bs) return fail(IMQ_ERR_INVALID_ARG, "imq_ext_operator_far_near: null argument");
  return guard([&] {
    op->op->far_near_locked(d_us, d_bs, scatter ? op->op->perm_ptr() : nullptr,
                            static_cast<cudaStream_t>(stream), far_begin, far_end, near_begin,
                            near_end);
    imqh::cuda_check(cudaGetLastError(), "far_near launch");
    return IMQ_OK;
  });
}

int imq_ext_shard_bounds(const int* leaf_start, int levels, int world, int* bounds_out) {
  if (!leaf_start || !bounds_out || levels < 1 || levels > 13 || world < 1)
    return fail(IMQ_ERR_INVALID_ARG, "imq_ext_shard_bounds: bad argument");
  return guard([&] {
    const size_t n = ((size_t)1 << (2 * (levels + 1))) + 1;
    std::vector<int> ls(leaf_start, leaf_start + n);
    std::vector<int> b = imqh::shard_bounds(ls, levels, world);
    std::copy(b.begin(), b.end(), bounds_out);
    return IMQ_OK;
  });
}

int imq_ext_shard_bounds_work(const int* leaf_start, int levels, int m, int world,
                              int* bounds_out) {
  if (!leaf_start || !bounds_out || levels < 1 || levels > 13 || world < 1 || m < 0)
    return fail(IMQ_ERR_INVALID_ARG, "imq_ext_shard_bounds_work: bad argument");
  return guard([&] {
    const size_t n = ((size_t)1 << (2 * (levels + 1))) + 1;
    std::vector<int> ls(leaf_start, leaf_start + n);
    std::vector<int> b =
        imqh::shard_bounds_weighted(ls, levels, world, imqh::parent_work(ls, levels, m));
    std::copy(b.begin(), b.end(), bounds_out);
    return IMQ_OK;
  });
}

int imq_ext_operator_restrict(const imq_operator* op, int sorted_lo, int sorted_hi) {
  if (!op) return fail(IMQ_ERR_INVALID_ARG, "imq_ext_operator_restrict: null argument");
  return guard([&] {
    op->op->restrict_targets(sorted_lo, sorted_hi);
    return IMQ_OK;
  });
}

int imq_ext_fp64_peak(int iters, double* tflops, double* ms) {
  if (!tflops || iters < 1) return fail(IMQ_ERR_INVALID_ARG, "imq_ext_fp64_peak: bad argument");
  return guard([&] {
    require_device();
    float t = 0.f;
    *tflops = imqk::measure_dfma_peak(iters, &t);
    if (ms) *ms = t;
    imqh::cuda_check(cudaGetLastError(), "dfma peak");
    return IMQ_OK;
  });
}

int imq_ext_device_count(int* out) {
  if (!out) return fail(IMQ_ERR_INVALID_ARG, "imq_ext_device_count: null argument");
  int nd = 0;
  if (cudaGetDeviceCount(&nd) != cudaSuccess) {
    cudaGetLastError();
    nd = 0;
  }
  *out = nd;
  return IMQ_OK;
}

int imq_ext_set_device(int device) {
  return guard([&] {
    require_device();
    imqh::cuda_check(cudaSetDevice(device), "cudaSetDevice");
    return IMQ_OK;
  });
}

}  // extern "C"
