// operator.cu -- build / apply / solve of the device-resident fast operator.
//
// Build (reference fastmv.cpp:32-77, partition.cpp:9-85), all on the GPU
// except O(#leaves) bookkeeping:
//   H2D points -> min/max + finiteness reduction -> bounding square (host,
//   reference arithmetic) -> bit-exact finest-level binning to Morton keys ->
//   stable radix sort (key, index) -> gathered SoA coordinates -> leaf offsets
//   -> work lists for the far (<= 64 targets of one level-(L-1) block per warp)
//   and near (<= 32 targets of one leaf per warp) kernels.
// Interaction lists are never materialised: kernels enumerate them on the fly
// (the reference's O(grid^4) list build, partition.cpp:56-72, is 151 s at L=8).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <climits>
#include <cmath>
#include <cstring>
#include <new>
#include <stdexcept>
#include <thread>

#include "host_math.hpp"
#include "imq_device.cuh"
#include "operator.hpp"

#ifndef IMQ_GEMM_MIN_TILES
#define IMQ_GEMM_MIN_TILES 256  // node / ring passes with fewer 32-box tiles stay Horner items
#endif

namespace imqh {

constexpr size_t kM2tMaxSmem = 220 * 1024;  // fused M2M + transform: M <= ~22

void cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    throw std::bad_alloc();
  }
  throw cuda_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

namespace {

template <typename T>
T* dalloc(size_t count, const char* what) {
  T* p = nullptr;
  if (count == 0) count = 1;
  cuda_check(cudaMalloc(&p, count * sizeof(T)), what);
  return p;
}
template <typename T>
void dfree(T*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace

DeviceOperator::DeviceOperator(const double* xy_host, size_t n, double t, int M, int levels,
                               const OperatorOptions& opt)
    : opt_(opt) {
  opt_.ring_tau = std::max(opt_.ring_tau, kRingTau);  // stricter only
  opt_.ring2_tau = std::max(opt_.ring2_tau, kRing2Tau);
  opt_.inner_tau = std::max(opt_.inner_tau, kInnerTau);
  opt_.xring_tau = std::max(opt_.xring_tau, kXringTau);
  if (n == 0) throw std::invalid_argument("build_operator: empty point set");
  check_t(t);  // KernelParams(t) precedes build_operator (capi.cpp:110)
  if (n > (size_t)INT_MAX) throw std::invalid_argument("build_operator: too many points");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    throw cuda_error("no CUDA device available: the B200 build has no CPU fallback");
  }
  cuda_check(cudaGetDevice(&device_), "cudaGetDevice");
  N_ = (int)n;
  M_ = M;
  t_ = t;
  cuda_check(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "stream create");
  int prio_lo = 0, prio_hi = 0;
  cuda_check(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi), "priority range");
  cuda_check(cudaStreamCreateWithPriority(&hp_stream_, cudaStreamNonBlocking, prio_hi),
             "stream create");
  cuda_check(cudaEventCreateWithFlags(&ev_hp_done_, cudaEventDisableTiming), "event create");
  for (int k = 0; k < kAuxStreams; ++k) {
    cuda_check(cudaStreamCreateWithPriority(&aux_[k], cudaStreamNonBlocking, prio_hi),
               "stream create");
    cuda_check(cudaEventCreateWithFlags(&ev_join_[k], cudaEventDisableTiming), "event create");
  }
  cuda_check(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming), "event create");
  cuda_check(cudaEventCreateWithFlags(&ev_last_, cudaEventDisableTiming), "event create");
  if (opt_.far_streams > 0)  // scheduling: far groups on 1..4 streams
    far_streams_ = std::max(1, std::min(1 + kAuxStreams, opt_.far_streams));
  cuda_check(cudaStreamCreateWithFlags(&near_stream_, cudaStreamNonBlocking), "stream create");
  cuda_check(cudaEventCreateWithFlags(&ev_near_fork_, cudaEventDisableTiming), "event create");
  cuda_check(cudaEventCreateWithFlags(&ev_near_done_, cudaEventDisableTiming), "event create");
  pending_levels_ = levels;
  try {
    build(xy_host);
  } catch (...) {
    release();
    throw;
  }
}

DeviceOperator::~DeviceOperator() { release(); }

void DeviceOperator::release() {
  DeviceGuard g(device_);
  if (stream_) cudaStreamSynchronize(stream_);
  if (ev_last_) cudaEventSynchronize(ev_last_);
  dfree(d_xs_); dfree(d_ys_); dfree(d_leaf_); dfree(d_perm_); dfree(d_leaf_start_);
  dfree(d_far_items_); dfree(d_near_items_);
  dfree(d_tr_off_); dfree(d_tr_idx_); dfree(d_tr_val_); dfree(d_binom_); dfree(d_m2t_);
  dfree(d_mu_); dfree(d_coef_); dfree(d_u_); dfree(d_us_); dfree(d_far_); dfree(d_b_);
  dfree(d_part_);
  dfree(d_need_par_); dfree(d_local_leaves_); dfree(d_own_lvl_);
  dfree(d_pair_items_); dfree(d_pair_part_); dfree(d_chunks_); dfree(d_contrib_off_);
  dfree(d_contrib_); dfree(d_near_s_); dfree(d_farc_); dfree(d_pull_items_);
  dfree(d_cheb_items_); dfree(d_cboxes_); dfree(d_ceval_items_);
  dfree(d_cnx_); dfree(d_cny_); dfree(d_cnleaf_); dfree(d_cval_); dfree(d_ccoef_);
  dfree(d_rnx_); dfree(d_rny_); dfree(d_rnleaf_); dfree(d_rval_); dfree(d_rcoef_);
  dfree(d_ring_items_); dfree(d_lpart_items_);
  dfree(d_xnx_); dfree(d_xny_); dfree(d_xnleaf_); dfree(d_xval_); dfree(d_xring_items_);
  free_gemm_pass(gx_);
  for (GemmPass& g : gnode_) free_gemm_pass(g);
  for (GemmPass& g : gring_) free_gemm_pass(g);
  dfree(d_xboxes_);
  dfree(solve_ws_);
  solve_ws_bytes_ = 0;
  dfree(d_u2_);
  dfree(d_b2_);
  dfree(d_blk_us_);
  dfree(d_blk_part_);
  blk_cap_ = 0;
  for (int sl = 0; sl < 2; ++sl) {
    dfree(d_blk_u_[sl]);
    dfree(d_blk_b_[sl]);
  }
  blk_io_cap_ = 0;
  for (int sl = 0; sl < 2; ++sl) {
    if (pin_in_[sl]) cudaFreeHost(pin_in_[sl]);
    if (pin_out_[sl]) cudaFreeHost(pin_out_[sl]);
    pin_in_[sl] = pin_out_[sl] = nullptr;
    for (cudaEvent_t e : ev_chunk_[sl]) cudaEventDestroy(e);
    ev_chunk_[sl].clear();
  }
  pool_.reset();
  if (cin_) {
    cudaStreamSynchronize(cin_);
    cudaStreamSynchronize(cout_);
    cudaStreamDestroy(cin_);
    cudaStreamDestroy(cout_);
    for (cudaEvent_t e : {ev_io_start_, ev_in_[0], ev_in_[1], ev_gath_[0], ev_gath_[1], ev_done_[0],
                          ev_done_[1], ev_out_[0], ev_out_[1]})
      if (e) cudaEventDestroy(e);
    cin_ = cout_ = nullptr;
  }
  if (solve_pin_) cudaFreeHost(solve_pin_);
  solve_pin_ = nullptr;
  solve_pin_bytes_ = 0;
  if (stream_) cudaStreamDestroy(stream_);
  stream_ = nullptr;
  for (int k = 0; k < kAuxStreams; ++k) {
    if (aux_[k]) cudaStreamDestroy(aux_[k]);
    if (ev_join_[k]) cudaEventDestroy(ev_join_[k]);
    aux_[k] = nullptr;
    ev_join_[k] = nullptr;
  }
  if (ev_fork_) cudaEventDestroy(ev_fork_);
  ev_fork_ = nullptr;
  if (ev_last_) cudaEventDestroy(ev_last_);
  ev_last_ = nullptr;
  if (near_stream_) cudaStreamDestroy(near_stream_);
  if (hp_stream_) cudaStreamDestroy(hp_stream_);
  if (ev_hp_done_) cudaEventDestroy(ev_hp_done_);
  hp_stream_ = nullptr;
  ev_hp_done_ = nullptr;
  if (ev_near_fork_) cudaEventDestroy(ev_near_fork_);
  if (ev_near_done_) cudaEventDestroy(ev_near_done_);
  near_stream_ = nullptr;
  ev_near_fork_ = ev_near_done_ = nullptr;
}

void DeviceOperator::build(const double* xy_host) {
  cudaStream_t s = stream_;
  const long long n = N_;
  double* d_xy = dalloc<double>(2 * (size_t)n, "points");
  uint32_t* d_keys = nullptr;
  int* d_idx = nullptr;
  void* d_tmp = nullptr;
  double* d_part = nullptr;
  try {
    cuda_check(cudaMemcpyAsync(d_xy, xy_host, 2 * (size_t)n * sizeof(double),
                               cudaMemcpyHostToDevice, s),
               "H2D points");
    const int nparts = imqk::minmax_parts(n);
    d_part = dalloc<double>(5 * (size_t)nparts + 5, "minmax");
    imqk::launch_minmax(d_xy, n, d_part, nparts, d_part + 5 * (size_t)nparts, s);
    double ext[5];
    cuda_check(cudaMemcpyAsync(ext, d_part + 5 * (size_t)nparts, sizeof ext,
                               cudaMemcpyDeviceToHost, s),
               "D2H extrema");
    cuda_check(cudaStreamSynchronize(s), "minmax");
    if (ext[4] > 0.0) throw std::invalid_argument("build_operator: non-finite coordinate");
    check_M(M_);
    K_ = horner_count(M_);  // stored far coefficients per block (zero slots dropped)
    Ke_ = order_Ke(M_);
    square_from_extrema(ext[0], ext[1], ext[2], ext[3], sq_);
    if (L_ <= 0) L_ = pending_levels_ > 0 ? pending_levels_ : auto_level(N_, M_);
    if (L_ > imqk::kMaxLevels - 1)
      throw std::invalid_argument("build_operator: levels must be <= 13 on this build");

    // ---- tree parameters
    P_.N = N_; P_.M = M_; P_.K = K_; P_.Ke = Ke_; P_.L = L_;
    P_.t = t_; P_.t2 = t_ * t_;
    P_.ox = sq_[0]; P_.oy = sq_[1];
    long long mo = 0, co = 0;
    for (int l = 1; l <= L_; ++l) {
      const int grid = 1 << (l + 1);
      P_.cell[l] = sq_[2] / grid;  // partition.cpp:46 (double / int)
      P_.mu_off[l] = mo;
      P_.coef_off[l] = co;
      mo += (long long)grid * grid * Ke_;
      co += (long long)grid * grid * K_;
    }
    coef_count_ = (size_t)co;

    // ---- bin + stable Morton sort
    const int gridL = 1 << (L_ + 1);
    const int bits = 2 * (L_ + 1);
    d_keys = dalloc<uint32_t>((size_t)n, "keys");
    d_idx = dalloc<int>((size_t)n, "idx");
    d_leaf_ = dalloc<uint32_t>((size_t)n, "leaf");
    d_perm_ = dalloc<int>((size_t)n, "perm");
    imqk::launch_bin(d_xy, n, sq_[0], sq_[1], P_.cell[L_], gridL, d_keys, d_idx, s);
    const size_t tb = imqk::sort_temp_bytes(n, bits);
    d_tmp = dalloc<unsigned char>(tb, "sort temp");
    imqk::launch_sort(d_tmp, tb, d_keys, d_leaf_, d_idx, d_perm_, n, bits, s);
    d_xs_ = dalloc<double>((size_t)n, "xs");
    d_ys_ = dalloc<double>((size_t)n, "ys");
    imqk::launch_gather_points(d_xy, d_perm_, n, d_xs_, d_ys_, s);
    const long long n_leaves = 1ll << (2 * (L_ + 1));
    d_leaf_start_ = dalloc<int>((size_t)n_leaves + 1, "leaf_start");
    imqk::launch_leaf_start(d_leaf_, n, n_leaves, d_leaf_start_, s);
    std::vector<int> ls((size_t)n_leaves + 1);
    cuda_check(cudaMemcpyAsync(ls.data(), d_leaf_start_, ls.size() * sizeof(int),
                               cudaMemcpyDeviceToHost, s),
               "D2H leaf_start");
    cuda_check(cudaStreamSynchronize(s), "tree build");
    cuda_check(cudaGetLastError(), "tree kernels");

    // leaf P2M parallelism: ~64 points per warp on average over non-empty leaves
    {
      long long ne = 0;
      for (long long q = 0; q < n_leaves; ++q) ne += ls[(size_t)q + 1] > ls[(size_t)q];
      const double mean = ne ? (double)N_ / (double)ne : 1.0;
      int w = 1;
      while (w < 8 && mean > 64.0 * w * 1.5) w *= 2;
      P_.p2m_wpl = w;
    }
    P_.xs = d_xs_;
    P_.ys = d_ys_;
    P_.leaf = d_leaf_;
    P_.leaf_start = d_leaf_start_;
    // ---- work lists (all targets)
    leaf_start_h_ = std::move(ls);
    build_items(0, N_);

    // ---- tables
    const Transform tr = build_transform(M_, t_);
    const std::vector<double> bn = binomials(M_);
    d_tr_off_ = dalloc<int>(tr.off.size(), "transform");
    d_tr_idx_ = dalloc<int>(tr.idx.size(), "transform");
    d_tr_val_ = dalloc<double>(tr.val.size(), "transform");
    d_binom_ = dalloc<double>(bn.size(), "binomials");
    cuda_check(cudaMemcpyAsync(d_tr_off_, tr.off.data(), tr.off.size() * sizeof(int),
                               cudaMemcpyHostToDevice, s), "H2D transform");
    cuda_check(cudaMemcpyAsync(d_tr_idx_, tr.idx.data(), tr.idx.size() * sizeof(int),
                               cudaMemcpyHostToDevice, s), "H2D transform");
    cuda_check(cudaMemcpyAsync(d_tr_val_, tr.val.data(), tr.val.size() * sizeof(double),
                               cudaMemcpyHostToDevice, s), "H2D transform");
    cuda_check(cudaMemcpyAsync(d_binom_, bn.data(), bn.size() * sizeof(double),
                               cudaMemcpyHostToDevice, s), "H2D binomials");
    if (L_ >= 2 &&
        imqk::m2m_tr_smem(M_, Ke_, K_, (int)tr.val.size()) <= kM2tMaxSmem) {
      // fused M2M + transform tables, one set per parent level (exact child
      // offsets +-cell_{l+1}/2), k_m2m_tr
      const size_t H1 = (size_t)M_ / 2 + 1, M1 = (size_t)M_ + 1;
      m2t_stride_ = 4 * (M1 * M1 + H1 * H1);
      d_m2t_ = dalloc<double2>(m2t_stride_ * (size_t)(L_ - 1), "m2m tables");
      for (int l = 1; l <= L_ - 1; ++l) {
        const std::vector<double> T = m2m_tables(M_, 0.5 * P_.cell[l + 1]);
        cuda_check(cudaMemcpy(d_m2t_ + m2t_stride_ * (size_t)(l - 1), T.data(),
                              T.size() * sizeof(double), cudaMemcpyHostToDevice), "H2D m2m");
      }
    }
    T_.off = d_tr_off_;
    T_.idx = d_tr_idx_;
    T_.val = d_tr_val_;
    T_.nnz = (int)tr.val.size();

    // ---- expansion storage + workspace
    d_mu_ = dalloc<double2>((size_t)mo, "moments");
    // empty blocks keep zero moments forever (P2M never writes them)
    cuda_check(cudaMemsetAsync(d_mu_, 0, (size_t)mo * sizeof(double2), s), "memset mu");
    d_coef_ = dalloc<double2>((size_t)co, "coefficients");
    d_u_ = dalloc<double>((size_t)n, "u");
    d_us_ = dalloc<double>((size_t)n, "u sorted");
    d_far_ = dalloc<double>((size_t)n, "far");
    d_b_ = dalloc<double>((size_t)n, "b");

    cuda_check(cudaStreamSynchronize(s), "operator build");
    certify();
  } catch (...) {
    dfree(d_xy); dfree(d_keys); dfree(d_idx); dfree(d_tmp); dfree(d_part);
    throw;
  }
  dfree(d_xy); dfree(d_keys); dfree(d_idx); dfree(d_tmp); dfree(d_part);
}

// Far items: <= 32 Rmax targets of one level-(L-1) block; near items: <= 32 Rn
// targets of one leaf.  Both are grouped by R = ceil(count / 32) so each group
// runs the kernel specialised for it.  Only targets in [p_lo, p_hi) (aligned
// to level-(L-1) block boundaries by the caller) get items.
void DeviceOperator::build_items(int p_lo, int p_hi) {
  const std::vector<int>& ls = leaf_start_h_;
  const long long n_par = 1ll << (2 * L_);  // level L-1 (level 0 = 2x2 for L = 1)
  const long long n_leaves = 1ll << (2 * (L_ + 1));
  far_items_h_.clear();
  near_items_h_.clear();
  auto grouped = [](std::vector<std::vector<int4>>& g, std::vector<int4>& out,
                    std::vector<int>& off) {
    off.assign(16, 0);
    for (size_t r = 0; r < g.size(); ++r) {
      out.insert(out.end(), g[r].begin(), g[r].end());
      off[r + 1] = (int)out.size();
    }
    for (size_t r = g.size() + 1; r < 16; ++r) off[r] = (int)out.size();
  };
  // Points per lane: as large as the kernels allow (register blocking), but
  // small enough that the GPU still gets >= ~8 waves of warps (kWarpsWanted).
  constexpr double kWarpsWanted = 148.0 * 64;
  const double nt = (double)(p_hi - p_lo);
  const int rfit = (int)std::max(1.0, std::floor(nt / (32.0 * kWarpsWanted)));
  int rmax = imqk::m2p_specialised(M_) ? std::min(rfit, imqk::far_max_points_per_lane()) : 2;
  if (opt_.far_rmax > 0)  // scheduling only
    rmax = std::max(1, std::min(imqk::far_max_points_per_lane(), opt_.far_rmax));
  // Level split (L >= 4): the lists of levels 1..L-2 are shared by every
  // target of a level-(L-2) block, so those levels run as a separate "coarse"
  // pass whose items span whole grandparents (fewer idle lanes), and the
  // per-parent "fine" pass covers levels L-1..L and adds the coarse partial.
  far_split_ = L_ >= 4 && !opt(kOptNoSplit);
  auto chunked = [&](long long blocks, int span, std::vector<std::vector<int4>>& g) {
    for (long long p = 0; p < blocks; ++p) {
      const int a = std::max(p_lo, ls[(size_t)(span * p)]);
      const int b = std::min(p_hi, ls[(size_t)(span * p + span)]);
      if (b <= a) continue;
      // balanced chunks: fewest items of <= 32 rmax targets, sizes multiple of 32
      const int nchunk = (b - a + 32 * rmax - 1) / (32 * rmax);
      const int size = 32 * ((b - a + 32 * nchunk - 1) / (32 * nchunk));
      for (int c = a; c < b; c += size) {
        const int cnt = std::min(size, b - c);
        // item.x: a level-(L-1) block containing the targets' ancestors
        g[(size_t)((cnt + 31) / 32 - 1)].push_back(make_int4((int)(p * (span / 4)), c, cnt, 0));
      }
    }
  };
  std::vector<std::vector<int4>> groups((size_t)rmax);
  chunked(n_par, 4, groups);
  grouped(groups, far_items_h_, far_group_off_);
  n_far_fine_ = (int)far_items_h_.size();
  far_cgroup_off_.assign(16, n_far_fine_);
  if (far_split_) {
    std::vector<std::vector<int4>> cg((size_t)rmax);
    chunked(n_par / 4, 16, cg);
    std::vector<int4> citems;
    grouped(cg, citems, far_cgroup_off_);
    for (int& o : far_cgroup_off_) o += n_far_fine_;
    far_items_h_.insert(far_items_h_.end(), citems.begin(), citems.end());
    dfree(d_farc_);
    d_farc_ = dalloc<double>((size_t)N_, "coarse far");
  }
  // Partial pass (L >= 4): the fine items keep only the outer ring of X at
  // level L (needed by all four leaves of X), and per-leaf items evaluate the
  // rest of each leaf's level-L list (7 of X's 12 inner-ring leaves), adding
  // into the coarse partial before the fine pass (build_far_list lsplit).
  dfree(d_lpart_items_);
  n_lpart_items_ = 0;
  lpart_group_off_.assign(16, 0);
  lpart_leaf2_ = imqk::m2p_specialised(M_);
  if (far_split_ && !opt(kOptNoLsplit)) {
    // specialised orders: two leaves per warp (k_m2p_leaf2), items of
    // <= 16 R2 targets grouped by R = ceil(count / 16) and paired inside a
    // group (an odd group gets an empty partner); else one leaf chunk of
    // <= 32 rmax targets per warp (k_m2p_far_generic, lsplit 2)
    const int gran = lpart_leaf2_ ? 16 : 32;
    const int rm = lpart_leaf2_ ? std::min(imqk::far_max_points_per_lane(), 2 * rmax) : rmax;
    std::vector<std::vector<int4>> pg((size_t)rm);
    for (long long q = 0; q < n_leaves; ++q) {
      const int a = std::max(p_lo, ls[(size_t)q]), b = std::min(p_hi, ls[(size_t)q + 1]);
      if (b <= a) continue;
      const int nchunk = (b - a + gran * rm - 1) / (gran * rm);
      const int size = gran * ((b - a + gran * nchunk - 1) / (gran * nchunk));
      for (int c = a; c < b; c += size) {
        const int cnt = std::min(size, b - c);
        pg[(size_t)((cnt + gran - 1) / gran - 1)].push_back(
            lpart_leaf2_ ? make_int4((int)q, c, cnt, 0)
                         : make_int4((int)(q >> 2), c, cnt, L_ | (2 << 12)));
      }
    }
    if (lpart_leaf2_)
      for (auto& g : pg)
        if (g.size() & 1) g.push_back(make_int4(0, 0, 0, 0));
    std::vector<int4> pitems;
    grouped(pg, pitems, lpart_group_off_);
    n_lpart_items_ = (int)pitems.size();
    if (n_lpart_items_) {
      d_lpart_items_ = dalloc<int4>(pitems.size(), "partial items");
      cuda_check(cudaMemcpy(d_lpart_items_, pitems.data(), pitems.size() * sizeof(int4),
                            cudaMemcpyHostToDevice), "H2D partial items");
    }
  }
  build_cheb(p_lo, p_hi);
  // near items: one leaf each; R from the mean leaf occupancy (a typical leaf
  // in one item), then the smallest source split (1, 3 or 9 ways) that gives
  // the GPU enough warps
  long long ne = 0;
  for (long long q = 0; q < n_leaves; ++q) ne += std::min(p_hi, ls[(size_t)q + 1]) > std::max(p_lo, ls[(size_t)q]);
  const double occ = ne ? nt / (double)ne : 1.0;
  // (measured: the near kernel wants many warps more than register blocking;
  // split the sources 3 or 9 ways until ~4 x kWarpsWanted items exist, and
  // drop to one target per lane if even the 9-way split is short of that)
  constexpr double kNearWarps = 4 * kWarpsWanted;
  int nrmax = std::max(1, std::min(3, (int)std::ceil(1.25 * occ / 32.0)));
  auto count_items = [&](int r) {
    long long c = 0;
    for (long long q = 0; q < n_leaves; ++q) {
      const int a = std::max(p_lo, ls[(size_t)q]), b = std::min(p_hi, ls[(size_t)q + 1]);
      if (b > a) c += (b - a + 32 * r - 1) / (32 * r);
    }
    return (double)c;
  };
  double nitems = count_items(nrmax);
  near_split_ = nitems >= kNearWarps ? 1 : (3 * nitems >= kNearWarps ? 3 : 9);
  if (near_split_ == 9 && 9 * nitems < kNearWarps && nrmax > 1) {
    nrmax = 1;
    nitems = count_items(1);
  }
  // symmetric near field: whole point set, every leaf within one item
  int max_leaf = 0;
  for (long long q = 0; q < n_leaves; ++q)
    max_leaf = std::max(max_leaf, ls[(size_t)q + 1] - ls[(size_t)q]);
  // unsharded: when the per-leaf items fill the GPU (else the chunk-pair
  // path); sharded ranges: whenever the leaves fit one item (boundary pairs
  // are completed by pull items below)
  const bool full = p_lo == 0 && p_hi == N_;
  near_sym_ = (full ? near_split_ == 1 : true) &&
              max_leaf <= 32 * imqk::near_max_points_per_lane() && !opt(kOptNearNoSym);
  if (near_sym_) near_split_ = 1;
  std::vector<std::vector<int4>> ngroups((size_t)(near_sym_ ? 8 : nrmax));
  if (near_sym_) {
    // symmetric: one leaf per half-warp item, grouped by R = ceil(count / 16)
    // and sorted inside a group by the forward neighbours' point count (the
    // two halves of a warp then stream (nearly) equally long source ranges)
    const int g = 1 << (L_ + 1);
    std::vector<std::vector<std::pair<int, int4>>> keyed(8);
    for (long long q = 0; q < n_leaves; ++q) {
      const int a = std::max(p_lo, ls[(size_t)q]), b = std::min(p_hi, ls[(size_t)q + 1]);
      if (b <= a) continue;
      int li, lj, fwd = 0;
      imqdev::demorton((uint32_t)q, li, lj);
      for (int dir = 0; dir < 4; ++dir) {
        const int bi = li + (dir == 0 ? 0 : 1), bj = lj + (dir == 0 ? 1 : dir - 2);
        if (bi > g - 1 || bj < 0 || bj > g - 1) continue;
        const uint32_t qb = imqdev::morton((uint32_t)bi, (uint32_t)bj);
        fwd += ls[(size_t)qb + 1] - ls[qb];
      }
      keyed[(size_t)((b - a + 15) / 16 - 1)].push_back({fwd, make_int4((int)q, a, b - a, 15)});
    }
    for (size_t r = 0; r < keyed.size(); ++r) {
      std::stable_sort(keyed[r].begin(), keyed[r].end(),
                       [](const std::pair<int, int4>& x, const std::pair<int, int4>& y) {
                         return x.first < y.first;
                       });
      for (const auto& e : keyed[r]) ngroups[r].push_back(e.second);
    }
  } else {
    for (long long q = 0; q < n_leaves; ++q) {
      const int a = std::max(p_lo, ls[(size_t)q]), b = std::min(p_hi, ls[(size_t)q + 1]);
      for (int c = a; c < b; c += 32 * nrmax) {
        const int cnt = std::min(32 * nrmax, b - c);
        for (int r = 0; r < near_split_; ++r)
          ngroups[(size_t)((cnt + 31) / 32 - 1)].push_back(make_int4(
              (int)q, c, cnt, near_split_ == 1 ? 15 : (near_split_ == 3 ? 16 + r : 32 + r)));
      }
    }
  }
  // pull items (sharded symmetric mode): own leaf B, direction d, backward
  // neighbour C (non-empty) outside [p_lo, p_hi)
  std::vector<int4> pull;
  if (near_sym_ && !full) {
    const int g = 1 << (L_ + 1);
    for (long long q = 0; q < n_leaves; ++q) {
      const int a = ls[(size_t)q], b = ls[(size_t)q + 1];
      if (b <= a || a < p_lo || b > p_hi) continue;
      int li, lj;
      imqdev::demorton((uint32_t)q, li, lj);
      for (int dir = 0; dir < 4; ++dir) {
        const int ci = li - (dir == 0 ? 0 : 1), cj = lj - (dir == 0 ? 1 : dir - 2);
        if (ci < 0 || cj < 0 || cj > g - 1) continue;
        const uint32_t qc = imqdev::morton((uint32_t)ci, (uint32_t)cj);
        const int c0 = ls[qc], c1 = ls[(size_t)qc + 1];
        if (c1 <= c0 || (c0 >= p_lo && c1 <= p_hi)) continue;
        pull.push_back(make_int4(a, (b - a) | (dir << 16), c0, c1 - c0));
      }
    }
  }
  dfree(d_pull_items_);
  n_pull_ = (int)pull.size();
  if (n_pull_) {
    d_pull_items_ = dalloc<int4>(pull.size(), "pull items");
    cuda_check(cudaMemcpy(d_pull_items_, pull.data(), pull.size() * sizeof(int4),
                          cudaMemcpyHostToDevice), "H2D pull items");
  }
  build_pair_items(p_lo, p_hi);
  const int nslots = near_sym_ ? 5 : (near_pair_ ? 1 : near_split_);
  if (nslots > 1) {
    dfree(d_part_);
    d_part_ = dalloc<double>((size_t)nslots * (size_t)N_, "near partials");
  }
  grouped(ngroups, near_items_h_, near_group_off_);
  n_far_ = (int)far_items_h_.size();
  n_near_ = (int)near_items_h_.size();
  dfree(d_far_items_);
  dfree(d_near_items_);
  d_far_items_ = dalloc<int4>(far_items_h_.size(), "far items");
  d_near_items_ = dalloc<int4>(near_items_h_.size(), "near items");
  cuda_check(cudaMemcpy(d_far_items_, far_items_h_.data(), far_items_h_.size() * sizeof(int4),
                        cudaMemcpyHostToDevice), "H2D far items");
  cuda_check(cudaMemcpy(d_near_items_, near_items_h_.data(), near_items_h_.size() * sizeof(int4),
                        cudaMemcpyHostToDevice), "H2D near items");
  target_lo_ = p_lo;
  target_hi_ = p_hi;
}

// Chunk-pair symmetric near field for the whole point set when leaves are too
// large for k_p2p_near_sym (see direct.cu).  Sets near_pair_.
void DeviceOperator::build_pair_items(int p_lo, int p_hi) {
  dfree(d_pair_items_); dfree(d_pair_part_); dfree(d_chunks_); dfree(d_contrib_off_);
  dfree(d_contrib_); dfree(d_near_s_);
  near_pair_ = false;
  n_pair_items_ = n_chunks_ = 0;
  if (near_sym_ || p_lo != 0 || p_hi != N_ || opt(kOptNearNoPair)) return;
  const std::vector<int>& ls = leaf_start_h_;
  const int g = 1 << (L_ + 1);
  const long long n_leaves = (long long)g * g;
  constexpr int CS = imqk::kNearChunk;
  // chunks of every leaf
  std::vector<int> leaf_chunk0((size_t)n_leaves + 1, 0);
  std::vector<int2> chunks;
  for (long long q = 0; q < n_leaves; ++q) {
    leaf_chunk0[(size_t)q] = (int)chunks.size();
    for (int c = ls[(size_t)q]; c < ls[(size_t)q + 1]; c += CS)
      chunks.push_back(make_int2(c, std::min(CS, ls[(size_t)q + 1] - c)));
  }
  leaf_chunk0[(size_t)n_leaves] = (int)chunks.size();
  std::vector<int2> pairs;  // (target chunk a, source chunk b)
  auto add = [&](int a, int b) { pairs.push_back(make_int2(a, b)); };
  for (long long q = 0; q < n_leaves; ++q) {
    int li, lj;
    imqdev::demorton((uint32_t)q, li, lj);
    for (int a = leaf_chunk0[(size_t)q]; a < leaf_chunk0[(size_t)q + 1]; ++a) {
      for (int b = a; b < leaf_chunk0[(size_t)q + 1]; ++b) add(a, b);
      for (int dir = 0; dir < 4; ++dir) {
        const int bi = li + (dir == 0 ? 0 : 1), bj = lj + (dir == 0 ? 1 : dir - 2);
        if (bi > g - 1 || bj < 0 || bj > g - 1) continue;
        const uint32_t qb = imqdev::morton((uint32_t)bi, (uint32_t)bj);
        for (int b = leaf_chunk0[qb]; b < leaf_chunk0[(size_t)qb + 1]; ++b) add(a, b);
      }
    }
    if ((double)pairs.size() * 2 * CS * sizeof(double) > 2.0e9) return;  // too large: plain path
  }
  // group by targets per lane R = ceil(|a| / 32) (one kernel specialisation
  // per group, so small chunks do not idle 3/4 of an R = 4 item); the order
  // inside a group, and with it every chunk's contribution order, is fixed
  auto rof = [&](const int2& pr) { return (chunks[(size_t)pr.x].y + 31) / 32; };
  std::stable_sort(pairs.begin(), pairs.end(),
                   [&](const int2& x, const int2& y) { return rof(x) < rof(y); });
  pair_group_off_.assign(imqk::kPairR + 1, 0);
  for (const int2& pr : pairs) ++pair_group_off_[(size_t)rof(pr)];
  for (int r = 1; r <= imqk::kPairR; ++r) pair_group_off_[(size_t)r] += pair_group_off_[(size_t)r - 1];
  std::vector<int4> items;
  std::vector<std::vector<int>> contrib(chunks.size());
  for (const int2& pr : pairs) {
    const int i = (int)items.size(), a = pr.x, b = pr.y;
    items.push_back(make_int4(chunks[(size_t)a].x, chunks[(size_t)a].y, chunks[(size_t)b].x,
                              chunks[(size_t)b].y));
    contrib[(size_t)a].push_back(i * 2 * CS);
    if (a != b) contrib[(size_t)b].push_back(i * 2 * CS + CS);
  }
  std::vector<int> off(chunks.size() + 1, 0), flat;
  for (size_t c = 0; c < chunks.size(); ++c) {
    off[c + 1] = off[c] + (int)contrib[c].size();
    flat.insert(flat.end(), contrib[c].begin(), contrib[c].end());
  }
  if (flat.empty()) flat.push_back(0);
  n_pair_items_ = (int)items.size();
  n_chunks_ = (int)chunks.size();
  d_pair_items_ = dalloc<int4>(items.size(), "pair items");
  d_pair_part_ = dalloc<double>(items.size() * 2 * CS, "pair partials");
  d_chunks_ = dalloc<int2>(chunks.size(), "chunks");
  d_contrib_off_ = dalloc<int>(off.size(), "contrib off");
  d_contrib_ = dalloc<int>(flat.size(), "contrib");
  d_near_s_ = dalloc<double>((size_t)N_, "near");
  cuda_check(cudaMemcpy(d_pair_items_, items.data(), items.size() * sizeof(int4),
                        cudaMemcpyHostToDevice), "H2D pair items");
  cuda_check(cudaMemcpy(d_chunks_, chunks.data(), chunks.size() * sizeof(int2),
                        cudaMemcpyHostToDevice), "H2D chunks");
  cuda_check(cudaMemcpy(d_contrib_off_, off.data(), off.size() * sizeof(int),
                        cudaMemcpyHostToDevice), "H2D contrib off");
  cuda_check(cudaMemcpy(d_contrib_, flat.data(), flat.size() * sizeof(int),
                        cudaMemcpyHostToDevice), "H2D contrib");
  near_pair_ = true;
}

// Coarse far field by Chebyshev interpolation (cheb.cu): for the levels
// 1..lc = L-2 of the coarse pass, each non-empty box evaluates its list at
// kChebN^2 nodes instead of at all of its points; used when the boxes of
// level lc hold on average >= 1.5x as many targets as nodes.
void DeviceOperator::build_cheb(int p_lo, int p_hi) {
  constexpr int NC = imqk::kChebN, NN = NC * NC;
  cheb_ = false;
  ring_ = false;
  dfree(d_cheb_items_); dfree(d_cboxes_); dfree(d_ceval_items_);
  dfree(d_ring_items_);
  dfree(d_xring_items_); dfree(d_xboxes_);
  xring_ = false;
  xgemm_ = false;
  free_gemm_pass(gx_);
  n_cheb_items_ = n_ceval_ = n_ring_items_ = n_xring_items_ = n_xboxes_ = 0;
  if (!far_split_ || opt(kOptNoCheb) || !imqk::m2p_specialised(M_)) return;
  const int lc = L_ - 2;
  const std::vector<int>& ls = leaf_start_h_;
  auto own = [&](int l, long long q) {  // targets of block q at level l inside [p_lo, p_hi)
    const int sh = 2 * (L_ - l);
    const int a = std::max(p_lo, ls[(size_t)(q << sh)]);
    const int b = std::min(p_hi, ls[(size_t)((q + 1) << sh)]);
    return std::max(0, b - a);
  };
  long long nonempty = 0, tot = 0;
  for (long long q = 0; q < (1ll << (2 * (lc + 1))); ++q) {
    const int c = own(lc, q);
    if (c > 0) ++nonempty, tot += c;
  }
  if (!nonempty || (double)tot < 1.5 * NN * (double)nonempty) return;
  // The rings (build_far_list mode 2): the level-l ring of a level-(l-1) box
  // A, l = 2..L-1, through NR x NR nodes of A, when the level-lc boxes hold on
  // average >= 1.25x as many targets as ring nodes (coarser levels always
  // gain: A's four children would evaluate the ring at 4 NC^2 nodes).
  constexpr int NR = imqk::kChebNR, NRR = NR * NR;
  ring_ = !opt(kOptNoRing) && (double)tot >= 1.25 * NRR * (double)nonempty;
  // Rings of levels ring_l0_..L-1 only: the level-l ring is interpolated on a
  // level-(l-1) box A of half-width h only where t >= tau h, i.e. where the
  // lifted singularities of the ring's expansions sit >= tau h off the real
  // plane (coarse boxes with t << h need more nodes at high orders).
  {
    const double tau = opt_.ring_tau;
    ring_l0_ = L_;
    for (int l = L_ - 1; l >= 2 && P_.t >= tau * 0.5 * P_.cell[l - 1]; --l) ring_l0_ = l;
    if (ring_l0_ > L_ - 1) ring_ = false;
  }
  // node geometry (all boxes of levels 1..lc), tables.  The levels whose own
  // inner lists (rings on) sit where t >= 2.5 h use NI x NI nodes (a suffix
  // of the levels: h shrinks with the level).
  cheb_base_.assign((size_t)lc + 1, 0);
  inner_v_.assign((size_t)lc + 1, 0);
  cnode_base_.assign((size_t)lc + 2, 0);
  long long nb = 0;
  {
    const double taui = opt_.inner_tau;
    for (int l = 1; l <= lc; ++l) {
      cheb_base_[(size_t)l] = nb;
      nb += 1ll << (2 * (l + 1));
      inner_v_[(size_t)l] = ring_ && l >= std::max(2, ring_l0_) && !opt(kOptNoInner) &&
                            P_.t >= taui * 0.5 * P_.cell[l];
      const long long npl = inner_v_[(size_t)l] ? (long long)imqk::kChebNI * imqk::kChebNI : NN;
      cnode_base_[(size_t)l + 1] = cnode_base_[(size_t)l] + (1ll << (2 * (l + 1))) * npl;
    }
  }
  const size_t want_nodes = (size_t)cnode_base_[(size_t)lc + 1];
  if (cheb_nodes_ != want_nodes || cheb_coefs_ != (size_t)nb * NN) {
    dfree(d_cnx_); dfree(d_cny_); dfree(d_cnleaf_); dfree(d_cval_); dfree(d_ccoef_);
    cheb_nodes_ = want_nodes;
    cheb_coefs_ = (size_t)nb * NN;
    d_cnx_ = dalloc<double>(cheb_nodes_, "cheb nodes");
    d_cny_ = dalloc<double>(cheb_nodes_, "cheb nodes");
    d_cnleaf_ = dalloc<uint32_t>(cheb_nodes_, "cheb node keys");
    d_cval_ = dalloc<double>(cheb_nodes_, "cheb values");
    d_ccoef_ = dalloc<double>(cheb_coefs_, "cheb coefficients");
    cuda_check(cudaMemset(d_cnleaf_, 0, cheb_nodes_ * sizeof(uint32_t)), "cheb keys");
    std::vector<double> T(NN), SL(NN), SR(NN);
    const long double pi = 3.141592653589793238462643383279502884L;
    for (int k = 0; k < NC; ++k)
      for (int i = 0; i < NC; ++i) T[(size_t)k * NC + i] = (double)cosl(k * pi * (i + 0.5L) / NC);
    for (int kp = 0; kp < NC; ++kp)
      for (int k = 0; k < NC; ++k) {
        long double sl = 0, sr = 0;
        for (int i = 0; i < NC; ++i) {
          const long double u = cosl(pi * (i + 0.5L) / NC), w = cosl(kp * pi * (i + 0.5L) / NC);
          sl += w * cosl(k * acosl((u - 1) / 2));
          sr += w * cosl(k * acosl((u + 1) / 2));
        }
        const long double f = (2.0L / NC) * (kp == 0 ? 0.5L : 1.0L);
        SL[(size_t)kp * NC + k] = (double)(f * sl);
        SR[(size_t)kp * NC + k] = (double)(f * sr);
      }
    imqk::cheb_set_tables(T.data(), SL.data(), SR.data());
    {
      constexpr int NI = imqk::kChebNI;
      std::vector<double> TI((size_t)NI * NI);
      for (int k = 0; k < NI; ++k)
        for (int i = 0; i < NI; ++i) TI[(size_t)k * NI + i] = (double)cosl(k * pi * (i + 0.5L) / NI);
      imqk::cheb_set_inner_tables(TI.data());
    }
    for (int l = 1; l <= lc; ++l) {
      if (inner_v_[(size_t)l])
        imqk::launch_cheb_nodes_inner(P_, l, cnode_base_[(size_t)l], d_cnx_, d_cny_, stream_);
      else  // (the NC-node levels come first: their offsets are cheb_base_ * NN)
        imqk::launch_cheb_nodes(P_, l, cheb_base_[(size_t)l], d_cnx_, d_cny_, stream_);
    }
    cuda_check(cudaStreamSynchronize(stream_), "cheb nodes");
  }
  Pn_ = P_;
  Pn_.xs = d_cnx_;
  Pn_.ys = d_cny_;
  Pn_.leaf = d_cnleaf_;
  Pn_.N = (int)cheb_nodes_;
  if (ring_) {  // ring nodes of every box of levels 1..lc (rings of levels 2..L-1)
    // per parent level a: ring variant (fewer nodes where t >= 2.5 h_a, the
    // singularities sitting further off the real plane) and node offset
    const double tau2 = opt_.ring2_tau;
    ring_v_.assign((size_t)lc + 1, 0);
    ring_nbase_.assign((size_t)lc + 2, 0);
    for (int a = 1; a <= lc; ++a) {
      ring_v_[(size_t)a] = P_.t >= tau2 * 0.5 * P_.cell[a] ? 1 : 0;
      const long long nr = imqk::kRingNr[ring_v_[(size_t)a]];
      ring_nbase_[(size_t)a + 1] = ring_nbase_[(size_t)a] + (1ll << (2 * (a + 1))) * nr * nr;
    }
    const size_t want = (size_t)ring_nbase_[(size_t)lc + 1];
    if (ring_nodes_ != want) {
      dfree(d_rnx_); dfree(d_rny_); dfree(d_rnleaf_); dfree(d_rval_); dfree(d_rcoef_);
      ring_nodes_ = want;
      d_rnx_ = dalloc<double>(ring_nodes_, "ring nodes");
      d_rny_ = dalloc<double>(ring_nodes_, "ring nodes");
      d_rnleaf_ = dalloc<uint32_t>(ring_nodes_, "ring node keys");
      d_rval_ = dalloc<double>(ring_nodes_, "ring values");
      d_rcoef_ = dalloc<double>((size_t)(1ll << (2 * (lc + 2))) * NN, "ring child coefficients");
      cuda_check(cudaMemset(d_rnleaf_, 0, ring_nodes_ * sizeof(uint32_t)), "ring keys");
      const long double pi = 3.141592653589793238462643383279502884L;
      for (int v = 0; v < 2; ++v) {
        const int nr = imqk::kRingNr[v];
        std::vector<double> TR((size_t)nr * nr), B[2];
        for (int k = 0; k < nr; ++k)
          for (int i = 0; i < nr; ++i) TR[(size_t)k * nr + i] = (double)cosl(k * pi * (i + 0.5L) / nr);
        // B[h][k'][i] = (2/NC) w_k' sum_i' T_k'(u_i') l_i((u_i' -/+ 1) / 2), l_i the
        // Lagrange basis of the nr parent nodes, l_i(y) = (2/nr) sum_k w_k T_k(x_i) T_k(y)
        for (int h = 0; h < 2; ++h) {
          B[h].assign((size_t)NC * nr, 0.0);
          for (int kp = 0; kp < NC; ++kp)
            for (int i = 0; i < nr; ++i) {
              const long double xi = cosl(pi * (i + 0.5L) / nr);
              long double acc = 0;
              for (int ip = 0; ip < NC; ++ip) {
                const long double u = cosl(pi * (ip + 0.5L) / NC);
                const long double y = h == 0 ? (u - 1) / 2 : (u + 1) / 2;
                long double li = 0;
                for (int k = 0; k < nr; ++k)
                  li += (k == 0 ? 0.5L : 1.0L) * cosl(k * acosl(xi)) * cosl(k * acosl(y));
                acc += cosl(kp * pi * (ip + 0.5L) / NC) * (2.0L / nr) * li;
              }
              B[h][(size_t)kp * nr + i] = (double)((2.0L / NC) * (kp == 0 ? 0.5L : 1.0L) * acc);
            }
        }
        imqk::cheb_set_ring_tables(v, TR.data(), B[0].data(), B[1].data());
      }
      for (int l = 1; l <= lc; ++l)
        imqk::launch_cheb_nodes_ring(P_, l, ring_v_[(size_t)l], ring_nbase_[(size_t)l], d_rnx_,
                                     d_rny_, stream_);
      cuda_check(cudaStreamSynchronize(stream_), "ring nodes");
    }
    Pr_ = P_;
    Pr_.xs = d_rnx_;
    Pr_.ys = d_rny_;
    Pr_.leaf = d_rnleaf_;
    Pr_.N = (int)ring_nodes_;
  }
  // node items (level | list mode << 8 in item.w), coefficient box lists
  // (own non-empty boxes per level), evaluation items
  std::vector<std::vector<int4>> g((size_t)imqk::far_max_points_per_lane());
  std::vector<std::vector<int4>> rg((size_t)imqk::far_max_points_per_lane());
  std::vector<int> boxes;
  cbox_off_.assign((size_t)lc + 2, 0);
  // node chunks of <= 32 * kFarMaxR, balanced (324 -> 192 + 132, 676 -> 256 + 256 + 164)
  auto chunks = [](std::vector<std::vector<int4>>& grp, int par, long long start, int nn, int w) {
    const int nch = (nn + 255) / 256, ch = ((nn + nch - 1) / nch + 31) / 32 * 32;
    for (int c = 0; c < nn; c += ch) {
      const int cnt = std::min(ch, nn - c);
      grp[(size_t)((cnt + 31) / 32 - 1)].push_back(make_int4(par, (int)(start + c), cnt, w));
    }
  };
  // node / ring passes of the levels with enough boxes run as tensor-core
  // GEMMs (make_gemm_pass below): no work items for them
  const int gtile = imqk::node_gemm_tile();
  std::vector<char> gn((size_t)lc + 1, 0), gr((size_t)lc + 1, 0);
  for (int l = 2; l <= lc; ++l) {
    long long nb_own = 0;
    for (long long q = 0; q < (1ll << (2 * (l + 1))); ++q) nb_own += own(l, q) > 0;
    // where the GEMM wins (measured at config 4, k_node_gemm vs k_m2p_far): node
    // counts that leave idle target slots in the Horner kernel's 32-lane x R
    // items (not a multiple of 256), and levels with enough boxes to fill the
    // GPU (>= 256 tiles); the 16 x 16 passes run at 77 % of the pipe as Horner
    // items of R = 8 and at 63 % as GEMMs
    const int npd = inner_v_[(size_t)l] ? imqk::kChebNI : imqk::kChebN;
    const bool big = imqk::m2p_specialised(M_) && nb_own >= IMQ_GEMM_MIN_TILES * (long long)gtile;
    auto wins = [&](int nn) { return imqk::node_gemm_mt(nn) > 0; };
    gn[(size_t)l] = big && wins(npd * npd);
    if (ring_ && l + 1 >= ring_l0_) {
      const int nr = imqk::kRingNr[ring_v_[(size_t)l]];
      gr[(size_t)l] = big && wins(nr * nr);
    }
  }
  for (int l = 1; l <= lc; ++l) {
    cbox_off_[(size_t)l] = (int)boxes.size();
    for (long long q = 0; q < (1ll << (2 * (l + 1))); ++q) {
      if (!own(l, q)) continue;
      boxes.push_back((int)q);
      // own list of q at level l (without the ring of its parent when rings are on)
      if (!gn[(size_t)l]) {
        const long long npl =
            inner_v_[(size_t)l] ? (long long)imqk::kChebNI * imqk::kChebNI : (long long)NN;
        chunks(g, (int)(q << (2 * (L_ - 1 - l))), cnode_base_[(size_t)l] + q * npl, (int)npl,
               l | ((ring_ && l >= ring_l0_ ? 1 : 0) << 8));
      }
      // the level-(l+1) ring of q at q's ring nodes
      if (ring_ && l + 1 >= ring_l0_ && !gr[(size_t)l])
        chunks(rg, (int)((4 * q) << (2 * (L_ - 2 - l))),
               ring_nbase_[(size_t)l] + q * imqk::kRingNr[ring_v_[(size_t)l]] *
                                            imqk::kRingNr[ring_v_[(size_t)l]],
               imqk::kRingNr[ring_v_[(size_t)l]] * imqk::kRingNr[ring_v_[(size_t)l]],
               (l + 1) | (2 << 8));
    }
  }
  cbox_off_[(size_t)lc + 1] = (int)boxes.size();
  {
    const long double pi = 3.141592653589793238462643383279502884L;
    auto rel = [&](int l, int n) {  // node offsets h cos(pi (i + 1/2) / n), as the node kernels
      std::vector<double> r((size_t)n);
      for (int i = 0; i < n; ++i) r[(size_t)i] = 0.5 * P_.cell[l] * (double)cosl(pi * (i + 0.5L) / n);
      return r;
    };
    for (GemmPass& g : gnode_) free_gemm_pass(g);
    for (GemmPass& g : gring_) free_gemm_pass(g);
    gnode_.resize((size_t)lc + 1);
    gring_.resize((size_t)lc + 1);
    for (int l = 2; l <= lc; ++l) {
      const std::vector<int> bl(boxes.begin() + cbox_off_[(size_t)l], boxes.begin() + cbox_off_[(size_t)l + 1]);
      if (gn[(size_t)l]) {
        const bool inner = ring_ && l >= ring_l0_;
        const int npd = inner_v_[(size_t)l] ? imqk::kChebNI : imqk::kChebN;
        const long long npl = (long long)npd * npd;
        make_gemm_pass(gnode_[(size_t)l], l, npd, rel(l, npd), bl, true,
                       [&](int c, std::vector<GemmOff>& o) {
                         const int cx = c >> 1, cy = c & 1, lo = inner ? -1 : -2, hi = inner ? 2 : 3;
                         for (int ri = lo; ri <= hi; ++ri)
                           for (int rj = lo; rj <= hi; ++rj) {
                             const int dx = ri - cx, dy = rj - cy;
                             if (std::max(std::abs(dx), std::abs(dy)) >= 2) o.push_back({l, dx, dy});
                           }
                       },
                       d_cval_ + cnode_base_[(size_t)l]);
        (void)npl;
      }
      if (gr[(size_t)l]) {
        const int nr = imqk::kRingNr[ring_v_[(size_t)l]];
        make_gemm_pass(gring_[(size_t)l], l, nr, rel(l, nr), bl, false,
                       [&](int, std::vector<GemmOff>& o) {
                         for (int ri = -2; ri <= 3; ++ri)
                           for (int rj = -2; rj <= 3; ++rj)
                             if (ri == -2 || ri == 3 || rj == -2 || rj == 3) o.push_back({l + 1, ri, rj});
                       },
                       d_rval_ + ring_nbase_[(size_t)l]);
      }
    }
  }
  std::vector<int4> citems, ritems;
  cheb_group_off_.assign(16, 0);
  ring_group_off_.assign(16, 0);
  for (size_t r = 0; r < g.size(); ++r) {
    citems.insert(citems.end(), g[r].begin(), g[r].end());
    cheb_group_off_[r + 1] = (int)citems.size();
    ritems.insert(ritems.end(), rg[r].begin(), rg[r].end());
    ring_group_off_[r + 1] = (int)ritems.size();
  }
  for (size_t r = g.size() + 1; r < 16; ++r) {
    cheb_group_off_[r] = (int)citems.size();
    ring_group_off_[r] = (int)ritems.size();
  }
  // evaluation items: targets of the level-lc boxes, or with the rings of the
  // level-(L-1) boxes (their series carries the level-(L-1) ring's field)
  std::vector<int4> ev;
  const int per = imqk::cheb_eval_points_per_item();
  const int le = ring_ ? L_ - 1 : lc;
  for (long long q = 0; q < (1ll << (2 * (le + 1))); ++q) {
    const int sh = 2 * (L_ - le);
    const int a = std::max(p_lo, ls[(size_t)(q << sh)]), b = std::min(p_hi, ls[(size_t)((q + 1) << sh)]);
    for (int c = a; c < b; c += per) ev.push_back(make_int4((int)q, c, std::min(per, b - c), 0));
  }
  n_ring_items_ = (int)ritems.size();
  if (ring_ && n_ring_items_) {
    d_ring_items_ = dalloc<int4>(ritems.size(), "ring items");
    cuda_check(cudaMemcpy(d_ring_items_, ritems.data(), ritems.size() * sizeof(int4),
                          cudaMemcpyHostToDevice), "H2D ring items");
  }
  // The level-L outer ring of each level-(L-1) box X (20 leaves needed by all
  // of X's targets) through NX x NX nodes of X, added into X's series, where
  // the lifted singularities sit >= tau_x h_X off the real plane (NX = 14
  // needs t / h_X >= ~5 for ~1e-13) and X holds enough targets.
  if (ring_) {
    constexpr int NX = imqk::kChebNX, NXX = NX * NX;
    const double taux = opt_.xring_tau;
    long long nx_ne = 0, nx_tot = 0;
    for (long long q = 0; q < (1ll << (2 * L_)); ++q) {
      const int c = own(L_ - 1, q);
      if (c > 0) ++nx_ne, nx_tot += c;
    }
    xring_ = !opt(kOptNoXring) && nx_ne > 0 &&
             P_.t >= taux * 0.5 * P_.cell[L_ - 1] &&
             (double)nx_tot >= 1.25 * NXX * (double)nx_ne;
    if (xring_) {
      const long long nbx = 1ll << (2 * L_);
      if (xring_nodes_ != (size_t)nbx * NXX) {
        dfree(d_xnx_); dfree(d_xny_); dfree(d_xnleaf_); dfree(d_xval_);
        xring_nodes_ = (size_t)nbx * NXX;
        d_xnx_ = dalloc<double>(xring_nodes_, "x-ring nodes");
        d_xny_ = dalloc<double>(xring_nodes_, "x-ring nodes");
        d_xnleaf_ = dalloc<uint32_t>(xring_nodes_, "x-ring node keys");
        d_xval_ = dalloc<double>(xring_nodes_, "x-ring values");
        cuda_check(cudaMemset(d_xnleaf_, 0, xring_nodes_ * sizeof(uint32_t)), "x-ring keys");
        const long double pi = 3.141592653589793238462643383279502884L;
        std::vector<double> TX((size_t)NXX);
        for (int k = 0; k < NX; ++k)
          for (int i = 0; i < NX; ++i) TX[(size_t)k * NX + i] = (double)cosl(k * pi * (i + 0.5L) / NX);
        imqk::cheb_set_x_tables(TX.data());
        imqk::launch_cheb_nodes_x(P_, L_ - 1, d_xnx_, d_xny_, stream_);
        cuda_check(cudaStreamSynchronize(stream_), "x-ring nodes");
      }
      Px_ = P_;
      Px_.xs = d_xnx_;
      Px_.ys = d_xny_;
      Px_.leaf = d_xnleaf_;
      Px_.N = (int)xring_nodes_;
      std::vector<std::vector<int4>> xg((size_t)imqk::far_max_points_per_lane());
      std::vector<int> xboxes;
      for (long long q = 0; q < nbx; ++q) {
        if (!own(L_ - 1, q)) continue;
        xboxes.push_back((int)q);
        chunks(xg, (int)q, q * NXX, NXX, 0);  // levels / modes from the launch (far_near)
      }
      std::vector<int4> xitems;
      xring_group_off_.assign(16, 0);
      for (size_t r = 0; r < xg.size(); ++r) {
        xitems.insert(xitems.end(), xg[r].begin(), xg[r].end());
        xring_group_off_[r + 1] = (int)xitems.size();
      }
      for (size_t r = xg.size() + 1; r < 16; ++r) xring_group_off_[r] = (int)xitems.size();
      n_xring_items_ = (int)xitems.size();
      n_xboxes_ = (int)xboxes.size();
      d_xring_items_ = dalloc<int4>(std::max<size_t>(1, xitems.size()), "x-ring items");
      d_xboxes_ = dalloc<int>(std::max<size_t>(1, xboxes.size()), "x-ring boxes");
      if (n_xring_items_)
        cuda_check(cudaMemcpy(d_xring_items_, xitems.data(), xitems.size() * sizeof(int4),
                              cudaMemcpyHostToDevice), "H2D x-ring items");
      if (n_xboxes_)
        cuda_check(cudaMemcpy(d_xboxes_, xboxes.data(), xboxes.size() * sizeof(int),
                              cudaMemcpyHostToDevice), "H2D x-ring boxes");
      {  // the X-node pass as a GEMM: per class the 7 level-(L-1) inner blocks
         // (ring mode 1), then the 20 level-L outer-ring leaves (lsplit 4)
        const long double pi = 3.141592653589793238462643383279502884L;
        std::vector<double> rx((size_t)NX);
        for (int i = 0; i < NX; ++i)
          rx[(size_t)i] = 0.5 * P_.cell[L_ - 1] * (double)cosl(pi * (i + 0.5L) / NX);
        const int Lx = L_ - 1;
        make_gemm_pass(gx_, Lx, NX, rx, xboxes, true,
                       [&](int c, std::vector<GemmOff>& o) {
                         const int cx = c >> 1, cy = c & 1;
                         for (int ri = -1; ri <= 2; ++ri)
                           for (int rj = -1; rj <= 2; ++rj) {
                             const int dx = ri - cx, dy = rj - cy;
                             if (std::max(std::abs(dx), std::abs(dy)) >= 2) o.push_back({Lx, dx, dy});
                           }
                         for (int ri = -2; ri <= 3; ++ri)
                           for (int rj = -2; rj <= 3; ++rj)
                             if (ri == -2 || ri == 3 || rj == -2 || rj == 3) o.push_back({L_, ri, rj});
                       },
                       d_xval_);
        xgemm_ = gx_.on;
      }
    }
  }
  n_cheb_items_ = (int)citems.size();
  n_ceval_ = (int)ev.size();
  d_cheb_items_ = dalloc<int4>(citems.size(), "cheb items");
  d_cboxes_ = dalloc<int>(boxes.size(), "cheb boxes");
  d_ceval_items_ = dalloc<int4>(ev.size(), "cheb eval items");
  cuda_check(cudaMemcpy(d_cheb_items_, citems.data(), citems.size() * sizeof(int4),
                        cudaMemcpyHostToDevice), "H2D cheb items");
  cuda_check(cudaMemcpy(d_cboxes_, boxes.data(), boxes.size() * sizeof(int),
                        cudaMemcpyHostToDevice), "H2D cheb boxes");
  cuda_check(cudaMemcpy(d_ceval_items_, ev.data(), ev.size() * sizeof(int4),
                        cudaMemcpyHostToDevice), "H2D cheb eval");
  cheb_lc_ = lc;
  cheb_ = true;
}

// ------------------------------------------------------------ certificate --
// Build-time certificate of the interpolated far field (DESIGN.md §3,
// "Safety").  The gates of build_cheb() (t / h thresholds, node counts) come
// from sweeps; this check measures, on the operator's own geometry, how well
// each interpolant resolves its field: one probe product (u = random_vector(N,
// kProbeSeed), sorted order) fills every node-value array, k_cheb_tail forms
// each box's tensor Chebyshev coefficients and estimates the interpolation
// error from their decay (cheb.cu), and the error of a product is estimated as
//     est = sum over interpolation kinds of max_box estimate  /  max_i |b_i|.
// While est > budget (kCertBudget = 1e-12, or the stricter option), the kind
// with the largest contribution is switched off -- a level's inner list back
// to kChebN nodes, a ring variant back to kChebNR nodes, a ring level (and
// the coarser ones) back to per-child evaluation, the X-ring off, and as a
// last resort the whole Chebyshev path (all pairs direct, exact) -- and the
// work lists are rebuilt.  Sharded ranks inherit the decisions (they are
// stored in opt_ before restrict_targets rebuilds the lists), so every rank
// interpolates the same way.
void DeviceOperator::certify() {
  cert_ = CertReport{};
  if (!cheb_) return;
  constexpr unsigned long long kProbeSeed = 0x1D0C5EEDull;
  const double budget = opt_.cert_budget > 0 ? std::min(opt_.cert_budget, kCertBudget) : kCertBudget;
  cert_.budget = budget;
  double* d_max = dalloc<double>(1, "certificate");
  double2* d_tail = nullptr;
  size_t tail_cap = 0;
  try {
    for (int round = 0; round < 16 && cheb_; ++round) {
      cert_.rounds = round + 1;
      imqk::launch_random_vector(d_us_, N_, kProbeSeed, stream_);
      apply_sorted_locked(d_us_, d_b_, nullptr, stream_);
      imqk::launch_absmax(d_b_, N_, d_max, stream_);
      // kinds: {kind, level, box list offset / count (device), values, n}
      struct Kind { int kind, level; const int* boxes; int nb; const double* vals; int n; };
      std::vector<Kind> kinds;
      const int lc = cheb_lc_;
      for (int l = 1; l <= lc; ++l) {
        const int nb = cbox_off_[(size_t)l + 1] - cbox_off_[(size_t)l];
        if (!nb) continue;
        const int* bx = d_cboxes_ + cbox_off_[(size_t)l];
        const int n = inner_v_[(size_t)l] ? imqk::kChebNI : imqk::kChebN;
        kinds.push_back({inner_v_[(size_t)l] ? 1 : 0, l, bx, nb, d_cval_ + cnode_base_[(size_t)l], n});
        if (ring_ && l + 1 >= ring_l0_) {
          const int nr = imqk::kRingNr[ring_v_[(size_t)l]];
          kinds.push_back({ring_v_[(size_t)l] ? 3 : 2, l, bx, nb, d_rval_ + ring_nbase_[(size_t)l], nr});
        }
      }
      if (xring_ && n_xboxes_) kinds.push_back({4, L_ - 1, d_xboxes_, n_xboxes_, d_xval_, imqk::kChebNX});
      size_t total = 0;
      for (const Kind& k : kinds) total += (size_t)k.nb;
      if (total > tail_cap) {
        dfree(d_tail);
        d_tail = dalloc<double2>(total, "certificate tails");
        tail_cap = total;
      }
      size_t off = 0;
      for (const Kind& k : kinds) {
        imqk::launch_cheb_tail(k.boxes, k.nb, k.vals, k.n, d_tail + off, stream_);
        off += (size_t)k.nb;
      }
      std::vector<double2> tails(total);
      double bmax = 0.0;
      if (total)
        cuda_check(cudaMemcpyAsync(tails.data(), d_tail, total * sizeof(double2),
                                   cudaMemcpyDeviceToHost, stream_), "D2H certificate");
      cuda_check(cudaMemcpyAsync(&bmax, d_max, sizeof(double), cudaMemcpyDeviceToHost, stream_),
                 "D2H certificate");
      cuda_check(cudaStreamSynchronize(stream_), "certificate");
      cuda_check(cudaGetLastError(), "certificate kernels");
      cert_.scale = bmax;
      if (!(bmax > 0.0)) break;  // nothing to compare against (all-zero field)
      std::vector<double> est(kinds.size(), 0.0);
      double sum = 0.0;
      off = 0;
      for (size_t i = 0; i < kinds.size(); ++i) {
        double m = 0.0;
        for (int b = 0; b < kinds[i].nb; ++b) m = std::max(m, tails[off + (size_t)b].x);
        off += (size_t)kinds[i].nb;
        est[i] = m / bmax;
        sum += est[i];
      }
      for (int k = 0; k < 5; ++k) cert_.by_kind[k] = 0.0;
      for (size_t i = 0; i < kinds.size(); ++i)
        cert_.by_kind[kinds[i].kind] = std::max(cert_.by_kind[kinds[i].kind], est[i]);
      cert_.estimate = sum;
      if (!(sum > budget) || opt(kOptCertReport)) break;  // certified (NaN fails)
      // switch off the largest contributor and rebuild
      size_t w = 0;
      for (size_t i = 1; i < kinds.size(); ++i)
        if (!(est[i] <= est[w])) w = i;
      const Kind& k = kinds[w];
      const double above = 1.0 + 1e-9;  // just above t / h of that level
      switch (k.kind) {
        case 0: opt_.flags |= kOptNoCheb; break;
        case 1: opt_.inner_tau = std::max(opt_.inner_tau, above * t_ / (0.5 * P_.cell[k.level])); break;
        case 2: opt_.ring_tau = std::max(opt_.ring_tau, above * t_ / (0.5 * P_.cell[k.level])); break;
        case 3: opt_.ring2_tau = std::max(opt_.ring2_tau, above * t_ / (0.5 * P_.cell[k.level])); break;
        case 4: opt_.flags |= kOptNoXring; break;
      }
      ++cert_.fallbacks;
      build_items(0, N_);
      have_counts_ = false;
    }
  } catch (...) {
    dfree(d_max);
    dfree(d_tail);
    throw;
  }
  dfree(d_max);
  dfree(d_tail);
}

// Device list check (imq_verify "exact_cover", tests): the far passes'
// enumeration replayed per target (k_far_cover) against the reference lists.
ListCheck DeviceOperator::far_list_check(int max_targets) {
  std::lock_guard<std::mutex> lk(mtx_);
  DeviceGuard g(device_);
  cuda_check(cudaStreamSynchronize(stream_), "list check");
  cuda_check(cudaEventSynchronize(ev_last_), "list check");
  ListCheck r;
  const int lo = target_lo_, hi = target_hi_, n = hi - lo;
  if (n <= 0) return r;
  const int nt = std::max(1, std::min(n, max_targets));
  std::vector<int> tg((size_t)nt);
  for (int i = 0; i < nt; ++i) tg[(size_t)i] = lo + (int)(((long long)i * n) / nt);
  imqk::CoverModes Mo{};
  Mo.split = far_split_ ? 1 : 0;
  Mo.cheb = cheb_ ? 1 : 0;
  Mo.lc = cheb_lc_;
  Mo.ring = cheb_ && ring_ ? 1 : 0;
  Mo.ring_l0 = ring_l0_;
  Mo.lsplit = n_lpart_items_ > 0 ? 1 : 0;
  Mo.leaf2 = lpart_leaf2_ ? 1 : 0;
  Mo.xring = cheb_ && ring_ && xring_ && n_lpart_items_ > 0 ? 1 : 0;
  int* d_t = dalloc<int>((size_t)nt, "list check");
  int4* d_o = dalloc<int4>((size_t)nt, "list check");
  std::vector<int4> o((size_t)nt);
  try {
    cuda_check(cudaMemcpy(d_t, tg.data(), tg.size() * sizeof(int), cudaMemcpyHostToDevice), "H2D");
    imqk::CoverGemm Gm{};
    for (size_t l = 0; l < gnode_.size() && l <= (size_t)imqk::kMaxLevels; ++l)
      if (gnode_[l].on) {
        Gm.node[l] = gnode_[l].d_D;
        Gm.node_nd[l] = gnode_[l].n_deltas;
      }
    for (size_t l = 0; l < gring_.size() && l <= (size_t)imqk::kMaxLevels; ++l)
      if (gring_[l].on) {
        Gm.ring[l] = gring_[l].d_D;
        Gm.ring_nd[l] = gring_[l].n_deltas;
      }
    if (xgemm_ && gx_.on) {
      Gm.x = gx_.d_D;
      Gm.x_nd = gx_.n_deltas;
    }
    imqk::launch_far_cover(P_, d_t, nt, Mo, Gm, d_o, stream_);
    cuda_check(cudaStreamSynchronize(stream_), "list check");
    cuda_check(cudaGetLastError(), "list check kernel");
    cuda_check(cudaMemcpy(o.data(), d_o, o.size() * sizeof(int4), cudaMemcpyDeviceToHost), "D2H");
  } catch (...) {
    dfree(d_t);
    dfree(d_o);
    throw;
  }
  dfree(d_t);
  dfree(d_o);
  r.targets = nt;
  for (const int4& v : o) {
    r.missing += v.x;
    r.duplicated += v.y;
    r.extra += v.z;
    r.max_deviation = std::max(r.max_deviation, v.x + v.y + v.z);
    r.max_entries = std::max(r.max_entries, v.w);
  }
  return r;
}

// Node passes as tensor-core GEMMs (nodegemm.cu).  The nodes of every box of
// a level sit at the same positions relative to the box, and a box's list is
// a fixed set of source offsets (per class = the box's position in its parent
// where the list depends on it), so the basis A_delta[k][n] of every (node,
// offset) pair is formed once here (k_gemm_basis: the reference's truncated
// expansion in the monomial form) and each pass is one GEMM
// launch.  The offsets are exactly those build_far_list enumerates for the
// pass (the device list check replays both, k_far_cover).
void DeviceOperator::free_gemm_pass(GemmPass& g) {
  dfree(g.d_A);
  dfree(g.d_D);
  dfree(g.d_boxes);
  dfree(g.d_order);
  g = GemmPass{};
}

void DeviceOperator::make_gemm_pass(GemmPass& g, int box_level, int n_per_dim,
                                    const std::vector<double>& rel, const std::vector<int>& boxes,
                                    bool by_class,
                                    const std::function<void(int, std::vector<GemmOff>&)>& offsets,
                                    double* out) {
  free_gemm_pass(g);
  const int n_nodes = n_per_dim * n_per_dim, mt = imqk::node_gemm_mt(n_nodes);
  if (!imqk::m2p_specialised(M_) || mt == 0 || boxes.empty()) return;
  const int mp = 8 * mt, k2pad = imqk::node_gemm_k2pad(K_), ncls = by_class ? 4 : 1;
  // offsets per class; unique (level, dx, dy) -> one basis matrix
  std::vector<std::vector<GemmOff>> per((size_t)ncls);
  std::vector<GemmOff> uniq;
  std::vector<std::vector<int>> idx((size_t)ncls);
  int nd = 0;
  for (int c = 0; c < ncls; ++c) {
    offsets(c, per[(size_t)c]);
    // Phase order: offsets sorted by the residue of the source's cell index
    // modulo 2^(sh+1) per dimension (sh = source level - box level; a box of
    // class c has index = (c >> 1, c & 1) mod 2).  CTAs working on
    // neighbouring boxes (and the other classes of the same parents, which
    // run beside them) then read the same source coefficients at the same
    // time, so those re-reads hit L2 instead of DRAM (config 4 X-node pass:
    // 4.0 GB -> see profiles/README.md).  Any fixed order is a valid sum.
    const int cx = by_class ? (c >> 1) : 0, cy = by_class ? (c & 1) : 0;
    auto key = [&](const GemmOff& o) {
      const int sh = o.level - box_level, md = (2 << sh) - 1;
      return ((sh & 7) << 16) | ((((cx << sh) + o.dx) & md) << 8) | (((cy << sh) + o.dy) & md);
    };
    std::stable_sort(per[(size_t)c].begin(), per[(size_t)c].end(),
                     [&](const GemmOff& a, const GemmOff& b) { return key(a) > key(b); });
    nd = std::max(nd, (int)per[(size_t)c].size());
    for (const GemmOff& o : per[(size_t)c]) {
      int u = 0;
      while (u < (int)uniq.size() &&
             !(uniq[(size_t)u].level == o.level && uniq[(size_t)u].dx == o.dx && uniq[(size_t)u].dy == o.dy))
        ++u;
      if (u == (int)uniq.size()) uniq.push_back(o);
      idx[(size_t)c].push_back(u);
    }
  }
  if (nd == 0) return;
  // source centres relative to the box centre: level box_level + sh, cell index
  // (b << sh) + d -> (d + 0.5 - 2^sh / 2) cell_src
  std::vector<double> sx(uniq.size()), sy(uniq.size()), nx((size_t)n_nodes), ny((size_t)n_nodes);
  for (size_t u = 0; u < uniq.size(); ++u) {
    const int sh = uniq[u].level - box_level;
    const double cs = P_.cell[uniq[u].level], base = 0.5 - 0.5 * (double)(1 << sh);
    sx[u] = (uniq[u].dx + base) * cs;
    sy[u] = (uniq[u].dy + base) * cs;
  }
  for (int n = 0; n < n_nodes; ++n) {
    nx[(size_t)n] = rel[(size_t)(n / n_per_dim)];
    ny[(size_t)n] = rel[(size_t)(n % n_per_dim)];
  }
  double* d_tmp = dalloc<double>(2 * uniq.size() + 2 * (size_t)n_nodes, "gemm geometry");
  try {
    cuda_check(cudaMemcpy(d_tmp, sx.data(), sx.size() * sizeof(double), cudaMemcpyHostToDevice), "H2D");
    cuda_check(cudaMemcpy(d_tmp + uniq.size(), sy.data(), sy.size() * sizeof(double),
                          cudaMemcpyHostToDevice), "H2D");
    cuda_check(cudaMemcpy(d_tmp + 2 * uniq.size(), nx.data(), nx.size() * sizeof(double),
                          cudaMemcpyHostToDevice), "H2D");
    cuda_check(cudaMemcpy(d_tmp + 2 * uniq.size() + n_nodes, ny.data(), ny.size() * sizeof(double),
                          cudaMemcpyHostToDevice), "H2D");
    g.d_A = dalloc<double>(uniq.size() * (size_t)k2pad * mp, "gemm basis");
    imqk::launch_gemm_basis(g.d_A, d_tmp, d_tmp + uniq.size(), (int)uniq.size(),
                            d_tmp + 2 * uniq.size(), d_tmp + 2 * uniq.size() + n_nodes, n_nodes, mp,
                            k2pad, M_, P_.t2, stream_);
    cuda_check(cudaStreamSynchronize(stream_), "gemm basis");
    cuda_check(cudaGetLastError(), "gemm basis");
  } catch (...) {
    dfree(d_tmp);
    throw;
  }
  dfree(d_tmp);
  std::vector<imqk::GemmDelta> D((size_t)ncls * nd);
  for (int c = 0; c < ncls; ++c)
    for (int d = 0; d < nd; ++d) {
      if (d < (int)idx[(size_t)c].size()) {
        const GemmOff& o = uniq[(size_t)idx[(size_t)c][(size_t)d]];
        D[(size_t)c * nd + d] = {o.level, o.dx, o.dy, 0,
                                 g.d_A + (size_t)idx[(size_t)c][(size_t)d] * k2pad * mp};
      } else {  // padding: a source outside every grid (no contribution)
        D[(size_t)c * nd + d] = {box_level, 1 << 28, 0, 0, g.d_A};
      }
    }
  g.d_D = dalloc<imqk::GemmDelta>(D.size(), "gemm offsets");
  cuda_check(cudaMemcpy(g.d_D, D.data(), D.size() * sizeof(imqk::GemmDelta), cudaMemcpyHostToDevice),
             "H2D offsets");
  std::vector<int> bx;
  const int tile = imqk::node_gemm_tile();
  g.cls.n = ncls;
  g.cls.box_off[0] = 0;
  g.cls.tile_off[0] = 0;
  for (int c = 0; c < ncls; ++c) {
    for (int q : boxes)
      if (!by_class || (q & 3) == c) bx.push_back(q);
    g.cls.box_off[c + 1] = (int)bx.size();
    g.cls.tile_off[c + 1] = g.cls.tile_off[c] + (g.cls.box_off[c + 1] - g.cls.box_off[c] + tile - 1) / tile;
  }
  g.d_boxes = dalloc<int>(bx.size(), "gemm boxes");
  cuda_check(cudaMemcpy(g.d_boxes, bx.data(), bx.size() * sizeof(int), cudaMemcpyHostToDevice),
             "H2D boxes");
  g.cls.order = nullptr;
  if (ncls > 1) {  // tile j of every class before tile j + 1 of any
    std::vector<int2> ord;
    int most = 0;
    for (int c = 0; c < ncls; ++c) most = std::max(most, g.cls.tile_off[c + 1] - g.cls.tile_off[c]);
    for (int j = 0; j < most; ++j)
      for (int c = 0; c < ncls; ++c)
        if (j < g.cls.tile_off[c + 1] - g.cls.tile_off[c]) ord.push_back(make_int2(c, j));
    g.d_order = dalloc<int2>(ord.size(), "gemm tile order");
    cuda_check(cudaMemcpy(g.d_order, ord.data(), ord.size() * sizeof(int2), cudaMemcpyHostToDevice),
               "H2D tile order");
    g.cls.order = g.d_order;
  }
  g.box_level = box_level;
  g.n_nodes = n_nodes;
  g.n_deltas = nd;
  g.k2pad = k2pad;
  g.out = out;
  g.on = true;
}

void DeviceOperator::launch_gemm_pass(const GemmPass& g, cudaStream_t s) {
  if (g.on)
    imqk::launch_node_gemm(P_, g.box_level, g.d_boxes, g.cls, g.d_D, g.n_deltas, g.k2pad, d_coef_,
                           g.out, g.n_nodes, s);
}

void DeviceOperator::restrict_targets(int p_lo, int p_hi) {
  std::lock_guard<std::mutex> lk(mtx_);
  DeviceGuard g(device_);
  if (p_lo < 0 || p_hi > N_ || p_lo > p_hi)
    throw std::invalid_argument("restrict_targets: bad sorted-position range");
  // Both ends must be level-(L-1) block boundaries (a value leaf_start[4p]):
  // setup_sharded_moments() counts a parent as owned only when it lies fully
  // inside the range, so a parent straddling a cut would add its points to
  // the coarse moments on no rank.
  auto boundary = [&](int v) {
    const long long np = 1ll << (2 * L_);
    long long lo = 0, hi = np;  // smallest p with leaf_start[4p] >= v
    while (lo < hi) {
      const long long mid = (lo + hi) / 2;
      if (leaf_start_h_[(size_t)(4 * mid)] < v) lo = mid + 1; else hi = mid;
    }
    return leaf_start_h_[(size_t)(4 * lo)] == v;
  };
  if (!boundary(p_lo) || !boundary(p_hi))
    throw std::invalid_argument("restrict_targets: range ends must be level-(L-1) block boundaries");
  cuda_check(cudaStreamSynchronize(stream_), "restrict");
  cuda_check(cudaEventSynchronize(ev_last_), "restrict");  // work on other streams
  build_items(p_lo, p_hi);
  setup_sharded_moments(p_lo, p_hi);
}

// World+1 sorted-position bounds, cut at level-(L-1) block boundaries, with
// near-equal point counts per rank (far work per target is ~uniform).
std::vector<int> shard_bounds(const std::vector<int>& ls, int L, int world) {
  if (world < 1) throw std::invalid_argument("shard_bounds: world must be >= 1");
  const long long n_par = 1ll << (2 * L);
  const int n = ls.back();
  std::vector<int> b((size_t)world + 1, n);
  b[0] = 0;
  long long p = 0;
  for (int r = 1; r < world; ++r) {
    const double want = (double)n * r / world;
    while (p < n_par && ls[(size_t)(4 * (p + 1))] <= want) ++p;
    // choose the closer of the two parent boundaries around `want`
    int lo = ls[(size_t)(4 * p)], hi = p < n_par ? ls[(size_t)(4 * (p + 1))] : n;
    b[(size_t)r] = (want - lo <= hi - want) ? lo : hi;
    if (b[(size_t)r] < b[(size_t)r - 1]) b[(size_t)r] = b[(size_t)r - 1];
  }
  return b;
}

// Per level-(L-1) block evaluation work, from the tree alone: far (target,
// source block) pairs x (M^2 + 4M + 12) DFMA-equivalents + near pairs x 6
// (symmetric evaluation), the counts exactly as pair_counts() forms them.
// For L >= 4 the levels 1..L-2 go through the Chebyshev nodes (build_cheb):
// a box's list then costs min(1, 400 / its targets) per target, plus the
// series evaluation (~1.4 pairs per target).
std::vector<double> parent_work(const std::vector<int>& ls, int L, int M) {
  auto count = [&](int l, int i, int j) -> long long {
    const uint32_t q = imqdev::morton((uint32_t)i, (uint32_t)j);
    const int sh = 2 * (L - l);
    return (long long)ls[(size_t)(q + 1) << sh] - ls[(size_t)q << sh];
  };
  auto list_count = [&](int l, int i, int j) {
    const int grid = 1 << (l + 1);
    int lo_i = 0, hi_i = grid - 1, lo_j = 0, hi_j = grid - 1;
    if (l >= 2) {
      lo_i = std::max(0, 2 * (i / 2 - 1)); hi_i = std::min(grid - 1, 2 * (i / 2 + 1) + 1);
      lo_j = std::max(0, 2 * (j / 2 - 1)); hi_j = std::min(grid - 1, 2 * (j / 2 + 1) + 1);
    }
    int ns = 0;
    for (int qi = lo_i; qi <= hi_i; ++qi)
      for (int qj = lo_j; qj <= hi_j; ++qj)
        if (std::max(std::abs(qi - i), std::abs(qj - j)) >= 2 && count(l, qi, qj) > 0) ++ns;
    return ns;
  };
  // shared list sizes of levels 1..L-1, per block (Morton order)
  std::vector<std::vector<int>> ns((size_t)L);
  for (int l = 1; l < L; ++l) {
    const int grid = 1 << (l + 1);
    ns[(size_t)l].assign((size_t)grid * grid, 0);
    for (int i = 0; i < grid; ++i)
      for (int j = 0; j < grid; ++j)
        if (count(l, i, j) > 0) ns[(size_t)l][imqdev::morton(i, j)] = list_count(l, i, j);
  }
  const double c_far = (double)M * M + 4.0 * M + 12.0, c_near = 6.0;
  const int gL = 1 << (L + 1);
  const long long n_par = 1ll << (2 * L);
  std::vector<double> w((size_t)n_par, 0.0);
  for (long long p = 0; p < n_par; ++p) {
    const long long np = (long long)ls[(size_t)(4 * p + 4)] - ls[(size_t)(4 * p)];
    if (!np) continue;
    double shared = 0.0;
    for (int l = 1; l < L; ++l) {
      const long long a = p >> (2 * (L - 1 - l));
      double wl = 1.0;
      if (L >= 4 && l <= L - 2) {
        const int sh = 2 * (L - l);
        const double na = (double)ls[(size_t)((a + 1) << sh)] - ls[(size_t)(a << sh)];
        wl = std::min(1.0, (double)(imqk::kChebN * imqk::kChebN) / na);
      }
      double nl = wl * ns[(size_t)l][(size_t)a];
      if (L >= 4 && l >= 2) {  // the level-l ring goes through the level-(l-1) box's nodes
        const long long pa = a >> 2;
        int ai, aj;
        imqdev::demorton((uint32_t)pa, ai, aj);
        const int g1 = 1 << (l + 1);
        double nr = 0;
        for (int qi = std::max(0, 2 * ai - 2); qi <= std::min(g1 - 1, 2 * ai + 3); ++qi)
          for (int qj = std::max(0, 2 * aj - 2); qj <= std::min(g1 - 1, 2 * aj + 3); ++qj) {
            const int ri = qi - 2 * ai, rj = qj - 2 * aj;
            if ((ri == -2 || ri == 3 || rj == -2 || rj == 3) && count(l, qi, qj) > 0) nr += 1;
          }
        const int sh = 2 * (L - l + 1);
        const double na = (double)ls[(size_t)(pa + 1) << sh] - ls[(size_t)pa << sh];
        nl += nr * (std::min(1.0, (double)(imqk::kChebNR * imqk::kChebNR) / na) - wl);
      }
      shared += nl;
    }
    if (L >= 4) shared += 1.4;
    double far = shared * (double)np, near = 0.0;
    for (int c = 0; c < 4; ++c) {
      const uint32_t q = (uint32_t)(4 * p + c);
      const long long nc = (long long)ls[(size_t)q + 1] - ls[q];
      if (!nc) continue;
      int i, j;
      imqdev::demorton(q, i, j);
      far += (double)nc * list_count(L, i, j);
      long long nn = 0;
      for (int qi = std::max(0, i - 1); qi <= std::min(gL - 1, i + 1); ++qi)
        for (int qj = std::max(0, j - 1); qj <= std::min(gL - 1, j + 1); ++qj)
          nn += count(L, qi, qj);
      near += (double)nc * (double)nn;
    }
    w[(size_t)p] = c_far * far + c_near * near;
  }
  return w;
}

// Bounds balanced by a per-parent weight (cuts at level-(L-1) boundaries).
std::vector<int> shard_bounds_weighted(const std::vector<int>& ls, int L, int world,
                                       const std::vector<double>& w) {
  if (world < 1) throw std::invalid_argument("shard_bounds: world must be >= 1");
  const long long n_par = 1ll << (2 * L);
  std::vector<double> cum((size_t)n_par + 1, 0.0);
  for (long long p = 0; p < n_par; ++p) cum[(size_t)p + 1] = cum[(size_t)p] + w[(size_t)p];
  const int n = ls.back();
  std::vector<int> b((size_t)world + 1, n);
  b[0] = 0;
  long long p = 0;
  for (int r = 1; r < world; ++r) {
    const double want = cum[(size_t)n_par] * r / world;
    while (p < n_par && cum[(size_t)p + 1] <= want) ++p;
    const long long cut = (want - cum[(size_t)p] <= cum[(size_t)std::min(p + 1, n_par)] - want)
                              ? p : std::min(p + 1, n_par);
    b[(size_t)r] = ls[(size_t)(4 * cut)];
    if (b[(size_t)r] < b[(size_t)r - 1]) b[(size_t)r] = b[(size_t)r - 1];
  }
  return b;
}

void DeviceOperator::moments(const double* d_us, cudaStream_t s) {
  imqk::launch_p2m_leaf(P_, d_us, d_mu_, nullptr, 0, s);
  if (d_m2t_) {
    // level l's kernel translates its children (level l + 1) up and writes
    // their coefficients; level 1 also transforms itself
    for (int l = L_ - 1; l >= 1; --l)
      imqk::launch_m2m_tr(P_, l, nullptr, 0, 1ll << (2 * (l + 1)), d_mu_ + P_.mu_off[l + 1],
                          d_mu_ + P_.mu_off[l], d_coef_ + P_.coef_off[l + 1],
                          l == 1 ? d_coef_ + P_.coef_off[1] : nullptr, m2t_V(l), m2t_W(l), T_, s);
    if (L_ == 1) imqk::launch_transform(P_, d_mu_, d_coef_, T_, s);
    return;
  }
  // orders beyond the fused kernel's shared memory: separate passes
  for (int l = L_ - 1; l >= 1; --l) imqk::launch_m2m(P_, l, d_mu_, d_binom_, s);
  imqk::launch_transform(P_, d_mu_, d_coef_, T_, s);
}

// ---------------------------------------------------------------------------
// Sharded moments (one rank of a multi-GPU application).  The rank owns the
// level-(L-1) blocks [par_lo, par_hi) (its targets).  Its far field needs, at
// levels L-1 and L, only blocks inside the children of the 3x3 neighbourhoods
// of its blocks' parents ("local" = own + halo), which it forms itself from
// its copy of u; at levels <= L-2 it contributes the moments of its OWN points
// (M2M of its own level-(L-1) blocks) and the caller sums those coarse levels
// over ranks (one all-reduce of mu[levels 1..L-2]) before moments_finish().
// ---------------------------------------------------------------------------
bool DeviceOperator::sharded() const { return !need_par_h_.empty(); }

void DeviceOperator::gather(const double* d_u, double* d_us, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(mtx_);
  DeviceGuard g(device_);
  Ordered o(*this, s);
  if (sharded())
    imqk::launch_gather_leaves(d_u, d_perm_, d_leaf_start_, d_local_leaves_,
                               (int)local_leaves_h_.size(), d_us, s);
  else
    imqk::launch_gather(d_u, d_perm_, N_, d_us, s);
}

void DeviceOperator::setup_sharded_moments(int p_lo, int p_hi) {
  dfree(d_need_par_); dfree(d_local_leaves_); dfree(d_own_lvl_);
  need_par_h_.clear();
  local_leaves_h_.clear();
  if ((p_lo == 0 && p_hi == N_) || L_ < 3 || !d_m2t_) return;
  const std::vector<int>& ls = leaf_start_h_;
  const int G = 1 << L_;  // level L-1 grid
  const long long npar = (long long)G * G;
  par_lo_ = (int)npar;
  par_hi_ = 0;
  for (long long p = 0; p < npar; ++p)
    if (ls[(size_t)(4 * p)] >= p_lo && ls[(size_t)(4 * p + 4)] <= p_hi && ls[(size_t)(4 * p)] < p_hi) {
      par_lo_ = std::min<long long>(par_lo_, p);
      par_hi_ = std::max<long long>(par_hi_, p + 1);
    }
  if (par_hi_ <= par_lo_) {
    par_lo_ = par_hi_ = 0;
  }
  std::vector<char> need((size_t)npar, 0);
  for (int p = par_lo_; p < par_hi_; ++p) {
    int pi, pj;
    imqdev::demorton((uint32_t)p, pi, pj);
    const int gi = pi >> 1, gj = pj >> 1;  // grandparent block (level L-2)
    for (int a = std::max(0, 2 * gi - 2); a <= std::min(G - 1, 2 * gi + 3); ++a)
      for (int b = std::max(0, 2 * gj - 2); b <= std::min(G - 1, 2 * gj + 3); ++b)
        need[imqdev::morton((uint32_t)a, (uint32_t)b)] = 1;
  }
  for (long long p = 0; p < npar; ++p) {
    if (!need[(size_t)p] || ls[(size_t)(4 * p)] == ls[(size_t)(4 * p + 4)]) continue;
    need_par_h_.push_back((int)p);
    for (int c = 0; c < 4; ++c)
      if (ls[(size_t)(4 * p + c)] < ls[(size_t)(4 * p + c + 1)]) local_leaves_h_.push_back((int)(4 * p + c));
  }
  if (need_par_h_.empty()) need_par_h_.push_back(0);  // keeps "sharded" set; zero-work lists
  d_need_par_ = dalloc<int>(need_par_h_.size(), "need par");
  d_local_leaves_ = dalloc<int>(std::max<size_t>(1, local_leaves_h_.size()), "local leaves");
  cuda_check(cudaMemcpy(d_need_par_, need_par_h_.data(), need_par_h_.size() * sizeof(int),
                        cudaMemcpyHostToDevice), "H2D need par");
  if (!local_leaves_h_.empty())
    cuda_check(cudaMemcpy(d_local_leaves_, local_leaves_h_.data(),
                          local_leaves_h_.size() * sizeof(int), cudaMemcpyHostToDevice),
               "H2D local leaves");
  d_own_lvl_ = dalloc<double2>((size_t)npar * Ke_, "own level moments");
}

void DeviceOperator::moments_local(const double* d_us, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(mtx_);
  DeviceGuard g(device_);
  Ordered order(*this, s);
  if (!sharded()) {  // unsharded: the full moments, nothing to reduce
    moments(d_us, s);
    return;
  }
  const int G = 1 << L_;
  const long long npar = (long long)G * G;
  const int nneed = (int)need_par_h_.size();
  imqk::launch_p2m_leaf(P_, d_us, d_mu_, d_local_leaves_, (int)local_leaves_h_.size(), s);
  // level L-1 for own + halo blocks (the needed parents), with the level-L
  // coefficients of their children (= the local leaves)
  imqk::launch_m2m_tr(P_, L_ - 1, d_need_par_, 0, nneed, d_mu_ + P_.mu_off[L_],
                      d_mu_ + P_.mu_off[L_ - 1], d_coef_ + P_.coef_off[L_], nullptr, m2t_V(L_ - 1),
                      m2t_W(L_ - 1), T_, s);
  // own-only level L-1 -> coarse levels (partial sums, reduced by the caller).
  // The coarse region is zeroed and only the parents above the own range are
  // translated (a contiguous Morton range per level): the all-reduce then
  // sums exactly the own-only partials.
  (void)npar;
  cuda_check(cudaMemsetAsync(d_mu_ + P_.mu_off[1], 0,
                             (size_t)(P_.mu_off[L_ - 1] - P_.mu_off[1]) * sizeof(double2), s),
             "coarse memset");
  if (par_hi_ <= par_lo_) return;
  long long a0 = par_lo_ >> 2, a1 = ((long long)par_hi_ + 3) >> 2;  // level-(L-2) parents
  // level L-1 input rows of those parents: own blocks, zero for the others
  cuda_check(cudaMemsetAsync(d_own_lvl_ + (size_t)(4 * a0) * Ke_, 0,
                             (size_t)(4 * (a1 - a0)) * Ke_ * sizeof(double2), s),
             "memset");
  cuda_check(cudaMemcpyAsync(d_own_lvl_ + (size_t)par_lo_ * Ke_,
                             d_mu_ + P_.mu_off[L_ - 1] + (size_t)par_lo_ * Ke_,
                             (size_t)(par_hi_ - par_lo_) * Ke_ * sizeof(double2),
                             cudaMemcpyDeviceToDevice, s),
             "own level copy");
  for (int l = L_ - 2; l >= 1; --l) {
    const double2* in = l == L_ - 2 ? d_own_lvl_ : d_mu_ + P_.mu_off[l + 1];
    imqk::launch_m2m_tr(P_, l, nullptr, a0, a1 - a0, in, d_mu_ + P_.mu_off[l], nullptr, nullptr,
                        m2t_V(l), m2t_W(l), T_, s);
    a0 >>= 2;
    a1 = (a1 + 3) >> 2;
  }
}

void DeviceOperator::coarse_moments(double2** ptr, size_t* count) const {
  *ptr = d_mu_ + P_.mu_off[1];
  *count = sharded() ? (size_t)(P_.mu_off[L_ - 1] - P_.mu_off[1]) : 0;
}

void DeviceOperator::moments_finish(cudaStream_t s) {
  std::lock_guard<std::mutex> lk(mtx_);
  DeviceGuard g(device_);
  Ordered order(*this, s);
  if (!sharded()) return;  // moments_local already transformed everything
  imqk::launch_transform(P_, d_mu_, d_coef_, T_, s, 1, L_ - 2);
  imqk::launch_transform(P_, d_mu_, d_coef_, T_, s, L_ - 1, L_ - 1, d_need_par_,
                         (int)need_par_h_.size());
  // (the local leaves' level-L coefficients came with moments_local's M2M)
}

void DeviceOperator::far_near(const double* d_us, double* d_out, const int* perm,
                              cudaStream_t s, int far_begin, int far_end, int near_begin,
                              int near_end, bool near_launched) {
  far_begin = std::max(0, far_begin);
  far_end = std::min(far_end, n_far_);
  near_begin = std::max(0, near_begin);
  near_end = std::min(near_end, n_near_);
  const bool sym = (near_sym_ || near_pair_) && near_end > near_begin;
  if (sym && near_sym_ && !near_launched) {  // symmetric near field first; the far epilogue combines
    imqk::launch_p2p_near_sym(P_, d_near_items_, near_group_off_.data(), near_begin, near_end,
                              d_us, d_part_, s);
    imqk::launch_p2p_pull(P_, d_pull_items_, n_pull_, d_us, d_part_, s);
  }
  if (sym && near_pair_) {
    imqk::launch_p2p_pair(P_, d_pair_items_, pair_group_off_.data(), d_us, d_pair_part_, s);
    imqk::launch_pair_reduce(d_chunks_, n_chunks_, d_contrib_off_, d_contrib_, d_pair_part_,
                             d_near_s_, nullptr, nullptr, s);
  }
  // fork: group launches on s + the aux streams, joined back into s
  auto far_pass = [&](int b, int e, const int* goff, const double* near_part, int nslots,
                      double* out, const int* pm, double* far_s, const double* far_add, int lmin,
                      int lmax, const imqk::TreeParams* Pp = nullptr,
                      const int4* its = nullptr, int ring = 0, int lsplit = 0,
                      bool leaf2 = false) {
    if (e <= b) return;
    cudaStream_t ss[1 + kAuxStreams] = {s};
    cuda_check(cudaEventRecord(ev_fork_, s), "fork");
    for (int k = 0; k < kAuxStreams; ++k) {
      ss[k + 1] = aux_[k];
      cuda_check(cudaStreamWaitEvent(aux_[k], ev_fork_, 0), "fork wait");
    }
    imqk::launch_m2p_far(Pp ? *Pp : P_, its ? its : d_far_items_, goff, b, e, d_coef_, far_s, ss,
                         far_streams_, near_part, nslots, out, pm, far_add, lmin, lmax, ring,
                         lsplit, leaf2);
    for (int k = 0; k < kAuxStreams; ++k) {
      cuda_check(cudaEventRecord(ev_join_[k], aux_[k]), "join");
      cuda_check(cudaStreamWaitEvent(s, ev_join_[k], 0), "join wait");
    }
  };
  const double* near_part = sym ? (near_pair_ ? d_near_s_ : d_part_) : nullptr;
  const int nslots = near_pair_ ? 1 : 5;
  if (far_split_) {
    // coarse pass (levels 1..L-2) into d_farc_, then the fine pass (L-1..L)
    const bool cheb_run = cheb_ && far_end > n_far_fine_;
    // the partial pass (whole fine range only) and, with it, the X-ring
    const bool lsplit = n_lpart_items_ > 0 && far_begin == 0 && far_end >= n_far_fine_;
    const bool xr = cheb_run && xring_ && lsplit;
    if (cheb_run) {
      // list fields at the Chebyshev nodes of every box, series per level
      // (parent restricted + own), summed at the targets of the level-lc boxes
      // The node, ring and X-node passes are independent of one another
      // (each reads the coefficients and writes its own node values): ONE
      // fork over s + the aux streams, the GEMMs first (one stream each), the
      // Horner item groups round-robin behind them, one join -- every
      // kernel's tail is filled by whatever is ready on another stream.
      {
        cudaStream_t ss[1 + kAuxStreams] = {s};
        cuda_check(cudaEventRecord(ev_fork_, s), "fork");
        for (int k = 0; k < kAuxStreams; ++k) {
          ss[k + 1] = aux_[k];
          cuda_check(cudaStreamWaitEvent(aux_[k], ev_fork_, 0), "fork wait");
        }
        int gi = 0;
        auto gstream = [&]() { return ss[1 + (gi++ % kAuxStreams)]; };
        if (xr && xgemm_)  // at the NX x NX nodes of each level-(L-1) box X: its level-(L-1)
                           // inner blocks and its level-L outer ring, as GEMMs
          launch_gemm_pass(gx_, gstream());
        if (ring_)
          for (const GemmPass& g : gring_)
            if (g.on) launch_gemm_pass(g, gstream());
        for (const GemmPass& g : gnode_)  // the GEMM levels
          if (g.on) launch_gemm_pass(g, gstream());
        auto items_pass = [&](int n_it, const int* goff, double* far_s, int lmin, int lmax,
                              const imqk::TreeParams& Pp, const int4* its, int ring, int lsp) {
          if (n_it > 0)
            imqk::launch_m2p_far(Pp, its, goff, 0, n_it, d_coef_, far_s, ss, far_streams_, nullptr,
                                 0, nullptr, nullptr, nullptr, lmin, lmax, ring, lsp, false);
        };
        // list fields at the Chebyshev nodes of every box
        items_pass(n_cheb_items_, cheb_group_off_.data(), d_cval_, 1, cheb_lc_, Pn_, d_cheb_items_,
                   0, 0);
        if (ring_)  // the level-(l+1) rings at the NR x NR nodes of the level-l boxes
          items_pass(n_ring_items_, ring_group_off_.data(), d_rval_, 2, L_ - 1, Pr_,
                     d_ring_items_, 0, 0);
        if (xr && !xgemm_)  // X nodes through k_m2p_far (ring mode 1 at level L-1, lsplit 4 at L)
          items_pass(n_xring_items_, xring_group_off_.data(), d_xval_, L_ - 1, L_, Px_,
                     d_xring_items_, 1, 4);
        for (int k = 0; k < kAuxStreams; ++k) {
          cuda_check(cudaEventRecord(ev_join_[k], aux_[k]), "join");
          cuda_check(cudaStreamWaitEvent(s, ev_join_[k], 0), "join wait");
        }
      }
      constexpr long long NN = imqk::kChebN * imqk::kChebN, NRR = imqk::kChebNR * imqk::kChebNR;
      for (int l = 1; l <= cheb_lc_; ++l) {
        const int* bx = d_cboxes_ + cbox_off_[(size_t)l];
        const int nbx = cbox_off_[(size_t)l + 1] - cbox_off_[(size_t)l];
        if (ring_ && l >= ring_l0_) {
          // parent series restricted + parent's level-l ring -> this level; then + own list
          const int* pbx = d_cboxes_ + cbox_off_[(size_t)l - 1];
          const int npb = cbox_off_[(size_t)l] - cbox_off_[(size_t)l - 1];
          imqk::launch_cheb_ring_coef(ring_v_[(size_t)l - 1], pbx, npb, cheb_base_[(size_t)l - 1],
                                      d_ccoef_, d_rval_ + ring_nbase_[(size_t)l - 1],
                                      d_ccoef_ + cheb_base_[(size_t)l] * NN, s);
          if (inner_v_[(size_t)l])  // own inner lists at NI x NI nodes, added
            imqk::launch_cheb_inner_coef(bx, nbx, d_cval_ + cnode_base_[(size_t)l],
                                         d_ccoef_ + cheb_base_[(size_t)l] * NN, s);
          else
            imqk::launch_cheb_coef(l, bx, nbx, cheb_base_[(size_t)l], -1, d_cval_, d_ccoef_, s);
        } else {
          imqk::launch_cheb_coef(l, bx, nbx, cheb_base_[(size_t)l],
                                 l > 1 ? cheb_base_[(size_t)l - 1] : 0, d_cval_, d_ccoef_, s);
        }
      }
      if (ring_) {
        const int lc = cheb_lc_;
        imqk::launch_cheb_ring_coef(ring_v_[(size_t)lc], d_cboxes_ + cbox_off_[(size_t)lc],
                                    cbox_off_[(size_t)lc + 1] - cbox_off_[(size_t)lc],
                                    cheb_base_[(size_t)lc], d_ccoef_,
                                    d_rval_ + ring_nbase_[(size_t)lc], d_rcoef_, s);
        if (xr) imqk::launch_cheb_xring_coef(d_xboxes_, n_xboxes_, d_xval_, d_rcoef_, s);
        imqk::launch_cheb_eval(P_, L_ - 1, d_ceval_items_, n_ceval_, 0, d_rcoef_, d_farc_, s);
      } else {
        imqk::launch_cheb_eval(P_, cheb_lc_, d_ceval_items_, n_ceval_,
                               cheb_base_[(size_t)cheb_lc_], d_ccoef_, d_farc_, s);
      }
    } else {
      far_pass(std::max(far_begin, n_far_fine_), far_end, far_cgroup_off_.data(), nullptr, 0,
               nullptr, nullptr, d_farc_, nullptr, 1, L_ - 2);
    }
    if (xr) {
      // everything but the level-L inner ring went through the series: the
      // per-leaf partial pass is the last far pass and combines far + near
      if (near_launched && sym) cuda_check(cudaStreamWaitEvent(s, ev_near_done_, 0), "near join");
      far_pass(0, n_lpart_items_, lpart_group_off_.data(), near_part, nslots, d_out, perm, d_far_,
               d_farc_, L_, L_, nullptr, d_lpart_items_, 0, 0, lpart_leaf2_);
    } else {
      // the partial pass: inner-ring leaves of level L per leaf, accumulated
      // into the coarse partial
      if (lsplit)
        far_pass(0, n_lpart_items_, lpart_group_off_.data(), nullptr, 0, nullptr, nullptr, d_farc_,
                 d_farc_, L_, L_, nullptr, d_lpart_items_, 0, 0, lpart_leaf2_);
      if (near_launched && sym) cuda_check(cudaStreamWaitEvent(s, ev_near_done_, 0), "near join");
      far_pass(far_begin, std::min(far_end, n_far_fine_), far_group_off_.data(), near_part, nslots,
               d_out, perm, d_far_, d_farc_, L_ - 1, L_, nullptr, nullptr,
               cheb_run && ring_ ? 1 : 0, lsplit ? 1 : 0);
    }
  } else {
    if (near_launched && sym) cuda_check(cudaStreamWaitEvent(s, ev_near_done_, 0), "near join");
    far_pass(far_begin, far_end, far_group_off_.data(), near_part, nslots, d_out, perm, d_far_,
             nullptr, 1, L_);
  }
  if (near_sym_ || near_pair_) return;
  if (near_end > near_begin)
    imqk::launch_p2p_near(P_, d_near_items_, near_group_off_.data(), near_begin, near_end, d_us,
                          d_far_, d_out, perm, d_part_, s);
  if (near_split_ > 1 && near_end > near_begin)
    imqk::launch_near_combine(target_lo_, target_hi_, N_, near_split_, d_far_, d_part_, d_out,
                              perm, s);
}

void DeviceOperator::apply_sorted_locked(const double* d_us, double* d_out, const int* perm,
                                         cudaStream_t s) {
  if (near_pair_ && n_far_ > 0) {
    // chunk-pair near field on its own stream, concurrent with the moments
    // and the far field; the pair reduction adds far + near and unsorts
    cuda_check(cudaEventRecord(ev_near_fork_, s), "near fork");
    cuda_check(cudaStreamWaitEvent(near_stream_, ev_near_fork_, 0), "near fork wait");
    imqk::launch_p2p_pair(P_, d_pair_items_, pair_group_off_.data(), d_us, d_pair_part_,
                          near_stream_);
    cuda_check(cudaEventRecord(ev_near_done_, near_stream_), "near done");
    moments(d_us, s);
    far_near(d_us, d_out, perm, s, 0, n_far_, 0, 0);  // far field only -> d_far_
    cuda_check(cudaStreamWaitEvent(s, ev_near_done_, 0), "near join");
    imqk::launch_pair_reduce(d_chunks_, n_chunks_, d_contrib_off_, d_contrib_, d_pair_part_, d_out,
                             d_far_, perm, s);
    return;
  }
  if (near_sym_ && n_near_ > 0 && n_far_ > 0 && !sharded()) {
    // symmetric near field on its own stream, concurrent with the moments and
    // the coarse / node passes (which leave FP64 issue slots free); the fine
    // pass, whose epilogue adds the near slots, waits for it
    cuda_check(cudaEventRecord(ev_near_fork_, s), "near fork");
    cuda_check(cudaStreamWaitEvent(near_stream_, ev_near_fork_, 0), "near fork wait");
    imqk::launch_p2p_near_sym(P_, d_near_items_, near_group_off_.data(), 0, n_near_, d_us,
                              d_part_, near_stream_);
    imqk::launch_p2p_pull(P_, d_pull_items_, n_pull_, d_us, d_part_, near_stream_);
    cuda_check(cudaEventRecord(ev_near_done_, near_stream_), "near done");
    // the critical path (moments -> node passes -> fine pass) on a
    // high-priority stream, so its blocks are scheduled ahead of pending near
    // blocks; the near field fills the SMs it leaves idle
    cuda_check(cudaStreamWaitEvent(hp_stream_, ev_near_fork_, 0), "hp fork wait");
    moments(d_us, hp_stream_);
    far_near(d_us, d_out, perm, hp_stream_, 0, n_far_, 0, n_near_, true);
    cuda_check(cudaEventRecord(ev_hp_done_, hp_stream_), "hp done");
    cuda_check(cudaStreamWaitEvent(s, ev_hp_done_, 0), "hp join");
    return;
  }
  moments(d_us, s);
  far_near(d_us, d_out, perm, s, 0, n_far_, 0, n_near_);
}

void DeviceOperator::near_begin(const double* d_us, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(mtx_);
  DeviceGuard g(device_);
  Ordered o(*this, s);
  if (!near_sym_ || n_near_ == 0) return;
  cuda_check(cudaEventRecord(ev_near_fork_, s), "near fork");
  cuda_check(cudaStreamWaitEvent(near_stream_, ev_near_fork_, 0), "near fork wait");
  imqk::launch_p2p_near_sym(P_, d_near_items_, near_group_off_.data(), 0, n_near_, d_us, d_part_,
                            near_stream_);
  imqk::launch_p2p_pull(P_, d_pull_items_, n_pull_, d_us, d_part_, near_stream_);
  cuda_check(cudaEventRecord(ev_near_done_, near_stream_), "near done");
  near_pending_ = true;
}

void DeviceOperator::apply_sorted(const double* d_us, double* d_bs, cudaStream_t stream) {
  std::lock_guard<std::mutex> lk(mtx_);
  DeviceGuard g(device_);
  Ordered o(*this, stream);
  apply_sorted_locked(d_us, d_bs, nullptr, stream);
  cuda_check(cudaGetLastError(), "apply_sorted launch");
}

void DeviceOperator::apply_device(const double* d_u, double* d_b, cudaStream_t stream) {
  std::lock_guard<std::mutex> lk(mtx_);
  DeviceGuard g(device_);
  Ordered o(*this, stream);
  imqk::launch_gather(d_u, d_perm_, N_, d_us_, stream);
  apply_sorted_locked(d_us_, d_b, d_perm_, stream);
  cuda_check(cudaGetLastError(), "apply_device launch");
}

void DeviceOperator::apply_host(const double* u, double* b) { apply_batch(1, u, b); }

// Host vectors (imq_operator_apply semantics), nrhs products in a pipeline:
// the copy-in of u_{k+1} (copy engine 1) and the copy-out of b_{k-1} (copy
// engine 2) overlap the product of u_k (SMs).  Device input / output
// buffers are double-buffered.  Pageable host buffers (what a reference
// caller passes: std::vector memory, capi.cpp:130-138) are staged through
// pinned buffers in kIoChunk pieces by a thread pool, each piece's DMA
// overlapping the CPU copy of the next.  Results are identical to
// apply_device's (the same kernels on the same data).
void DeviceOperator::io_setup(bool pin_in, bool pin_out, bool two_slots) {
  if (!cin_) {
    cuda_check(cudaStreamCreateWithFlags(&cin_, cudaStreamNonBlocking), "stream create");
    cuda_check(cudaStreamCreateWithFlags(&cout_, cudaStreamNonBlocking), "stream create");
    for (cudaEvent_t* e : {&ev_io_start_, &ev_in_[0], &ev_in_[1], &ev_gath_[0], &ev_gath_[1],
                           &ev_done_[0], &ev_done_[1], &ev_out_[0], &ev_out_[1]})
      cuda_check(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event create");
  }
  const size_t bytes = (size_t)N_ * sizeof(double);
  const int slots = two_slots ? 2 : 1;
  if (two_slots && !d_u2_) {
    d_u2_ = dalloc<double>((size_t)N_, "u (second slot)");
    d_b2_ = dalloc<double>((size_t)N_, "b (second slot)");
  }
  auto pinned = [&](double*& p) {
    if (!p) {
      void* q = nullptr;
      cuda_check(cudaHostAlloc(&q, bytes, cudaHostAllocDefault), "pinned staging");
      p = static_cast<double*>(q);
    }
  };
  for (int sl = 0; sl < slots; ++sl) {
    if (pin_in) pinned(pin_in_[sl]);
    if (pin_out) {
      pinned(pin_out_[sl]);
      const size_t nch = (bytes + kIoChunk - 1) / kIoChunk;
      while (ev_chunk_[sl].size() < nch) {
        cudaEvent_t e;
        cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event create");
        ev_chunk_[sl].push_back(e);
      }
    }
  }
  if ((pin_in || pin_out) && !pool_) {
    const unsigned hw = std::thread::hardware_concurrency();
    pool_ = std::make_unique<CopyPool>((int)std::max(1u, std::min(16u, hw ? hw : 1u)));
  }
}

void DeviceOperator::apply_batch(int nrhs, const double* U, double* B) {
  if (nrhs < 1) throw std::invalid_argument("apply_batch: nrhs must be >= 1");
  std::lock_guard<std::mutex> lk(mtx_);
  DeviceGuard g(device_);
  cudaStream_t s = stream_;
  Ordered o(*this, s);
  const size_t n = (size_t)N_, bytes = n * sizeof(double);
  const bool pu = host_pinned(U), pb = host_pinned(B);
  io_setup(!pu, !pb, nrhs > 1);
  double* du[2] = {d_u_, nrhs > 1 ? d_u2_ : d_u_};
  double* db[2] = {d_b_, nrhs > 1 ? d_b2_ : d_b_};
  const size_t nch = (bytes + kIoChunk - 1) / kIoChunk;
  auto piece = [&](size_t c, size_t& off, size_t& len) {
    off = c * kIoChunk;
    len = std::min(kIoChunk, bytes - off);
  };
  // everything queued on s before this call precedes the copies
  cuda_check(cudaEventRecord(ev_io_start_, s), "io start");
  cuda_check(cudaStreamWaitEvent(cin_, ev_io_start_, 0), "io wait");
  cuda_check(cudaStreamWaitEvent(cout_, ev_io_start_, 0), "io wait");
  auto drain = [&](int j) {  // pageable output of product j
    const int sj = j & 1;
    char* dst = reinterpret_cast<char*>(B + (size_t)j * n);
    const char* src = reinterpret_cast<const char*>(pin_out_[sj]);
    if (pool_->threads() < 2) {
      for (size_t c = 0; c < nch; ++c) {
        size_t off, len;
        piece(c, off, len);
        cuda_check(cudaEventSynchronize(ev_chunk_[sj][c]), "D2H chunk");
        std::memcpy(dst + off, src + off, len);
      }
      return;
    }
    // the workers copy piece c as soon as its DMA has landed
    pool_->stream_begin(dst, src, bytes, kIoChunk, false);
    cudaError_t err = cudaSuccess;
    for (size_t c = 0; c < nch; ++c) {
      if (err == cudaSuccess) err = cudaEventSynchronize(ev_chunk_[sj][c]);
      pool_->stream_release(c + 1);  // (on an error too: the workers must finish the job)
    }
    pool_->stream_end();
    cuda_check(err, "D2H chunk");
  };
  for (int k = 0; k < nrhs; ++k) {
    const int sl = k & 1;
    const double* src = U + (size_t)k * n;
    // d_u[sl] was last read by the gather of product k - 2
    cuda_check(cudaStreamWaitEvent(cin_, ev_gath_[sl], 0), "slot wait");
    if (pu) {
      cuda_check(cudaMemcpyAsync(du[sl], src, bytes, cudaMemcpyHostToDevice, cin_), "H2D u");
    } else {
      cuda_check(cudaEventSynchronize(ev_in_[sl]), "staging wait");  // pin_in[sl] free
      const char* hs = reinterpret_cast<const char*>(src);
      char* ps = reinterpret_cast<char*>(pin_in_[sl]);
      char* ds = reinterpret_cast<char*>(du[sl]);
      if (pool_->threads() < 2) {
        for (size_t c = 0; c < nch; ++c) {
          size_t off, len;
          piece(c, off, len);
          std::memcpy(ps + off, hs + off, len);
          cuda_check(cudaMemcpyAsync(ds + off, ps + off, len, cudaMemcpyHostToDevice, cin_), "H2D u");
        }
      } else {
        // the workers stage piece after piece; each piece's DMA is queued as
        // soon as it is staged
        pool_->stream_begin(ps, hs, bytes, kIoChunk, true);
        cudaError_t err = cudaSuccess;
        for (size_t c = 0; c < nch; ++c) {
          size_t off, len;
          piece(c, off, len);
          pool_->stream_wait(c);
          if (err == cudaSuccess)
            err = cudaMemcpyAsync(ds + off, ps + off, len, cudaMemcpyHostToDevice, cin_);
        }
        pool_->stream_end();
        cuda_check(err, "H2D u");
      }
    }
    cuda_check(cudaEventRecord(ev_in_[sl], cin_), "event");
    cuda_check(cudaStreamWaitEvent(s, ev_in_[sl], 0), "event");
    imqk::launch_gather(du[sl], d_perm_, N_, d_us_, s);
    cuda_check(cudaEventRecord(ev_gath_[sl], s), "event");
    cuda_check(cudaStreamWaitEvent(s, ev_out_[sl], 0), "event");  // d_b[sl] copied out
    apply_sorted_locked(d_us_, db[sl], d_perm_, s);
    cuda_check(cudaEventRecord(ev_done_[sl], s), "event");
    cuda_check(cudaStreamWaitEvent(cout_, ev_done_[sl], 0), "event");
    if (pb) {
      cuda_check(cudaMemcpyAsync(B + (size_t)k * n, db[sl], bytes, cudaMemcpyDeviceToHost, cout_),
                 "D2H b");
    } else {
      char* ps = reinterpret_cast<char*>(pin_out_[sl]);
      const char* ds = reinterpret_cast<const char*>(db[sl]);
      for (size_t c = 0; c < nch; ++c) {
        size_t off, len;
        piece(c, off, len);
        cuda_check(cudaMemcpyAsync(ps + off, ds + off, len, cudaMemcpyDeviceToHost, cout_), "D2H b");
        cuda_check(cudaEventRecord(ev_chunk_[sl][c], cout_), "event");
      }
    }
    cuda_check(cudaEventRecord(ev_out_[sl], cout_), "event");
    cuda_check(cudaGetLastError(), "apply kernels");
    if (!pb && k >= 1) drain(k - 1);
  }
  if (!pb) drain(nrhs - 1);
  cuda_check(cudaStreamSynchronize(cout_), "apply");
  cuda_check(cudaStreamSynchronize(cin_), "apply");
  cuda_check(cudaStreamSynchronize(s), "apply");
  cuda_check(cudaGetLastError(), "apply kernels");
}

// ------------------------------------------------------ block product (f4) --
// The per-leaf symmetric near field is the one stage where several
// right-hand sides share arithmetic: a pair's kernel value costs ~10 FP64
// instructions and each vector only adds two DFMAs to it.  (The far field in
// its GEMM form -- basis x coefficient matrix, fastmv.cpp:125-135 -- needs as
// many DFMA-pipe slots per vector as the Horner form, and the FP64 tensor
// cores share that pipe on B200, so the far passes run per vector.)
bool DeviceOperator::block_near_ok() const {
  return near_sym_ && !near_pair_ && n_near_ > 0 && n_far_ > 0 && !sharded() && n_pull_ == 0;
}

void DeviceOperator::apply_block_locked(int nv, const double* d_U, size_t ldu, double* d_B,
                                        size_t ldb, cudaStream_t s) {
  const size_t n = (size_t)N_;
  if (nv < 2 || !block_near_ok()) {  // other near-field modes: vector by vector
    for (int v = 0; v < nv; ++v) {
      imqk::launch_gather(d_U + v * ldu, d_perm_, N_, d_us_, s);
      apply_sorted_locked(d_us_, d_B + v * ldb, d_perm_, s);
    }
    return;
  }
  if (nv > imqk::near_block_max()) throw std::invalid_argument("apply_block: group too large");
  if (blk_cap_ < nv) {
    cuda_check(cudaStreamSynchronize(s), "block workspace");
    cuda_check(cudaEventSynchronize(ev_last_), "block workspace");
    dfree(d_blk_us_);
    dfree(d_blk_part_);
    blk_cap_ = 0;
    d_blk_us_ = dalloc<double>((size_t)nv * n, "block vectors");
    d_blk_part_ = dalloc<double>((size_t)nv * 5 * n, "block near partials");
    blk_cap_ = nv;
  }
  for (int v = 0; v < nv; ++v)
    imqk::launch_gather(d_U + v * ldu, d_perm_, N_, d_blk_us_ + v * n, s);
  // one near-field launch sequence for the whole group, on the near stream
  cuda_check(cudaEventRecord(ev_near_fork_, s), "near fork");
  cuda_check(cudaStreamWaitEvent(near_stream_, ev_near_fork_, 0), "near fork wait");
  imqk::launch_p2p_near_sym_block(P_, d_near_items_, near_group_off_.data(), 0, n_near_, nv,
                                  d_blk_us_, n, d_blk_part_, 5 * n, near_stream_);
  cuda_check(cudaEventRecord(ev_near_done_, near_stream_), "near done");
  // moments + far field per vector on the high-priority stream; each final
  // pass adds its vector's near slots
  cuda_check(cudaStreamWaitEvent(hp_stream_, ev_near_fork_, 0), "hp fork wait");
  double* const part_single = d_part_;
  try {
    for (int v = 0; v < nv; ++v) {
      d_part_ = d_blk_part_ + (size_t)v * 5 * n;
      moments(d_blk_us_ + v * n, hp_stream_);
      far_near(d_blk_us_ + v * n, d_B + v * ldb, d_perm_, hp_stream_, 0, n_far_, 0, n_near_, true);
    }
  } catch (...) {
    d_part_ = part_single;
    throw;
  }
  d_part_ = part_single;
  cuda_check(cudaEventRecord(ev_hp_done_, hp_stream_), "hp done");
  cuda_check(cudaStreamWaitEvent(s, ev_hp_done_, 0), "hp join");
}

void DeviceOperator::apply_block_device(int nrhs, const double* d_U, double* d_B,
                                        cudaStream_t stream) {
  if (nrhs < 1) throw std::invalid_argument("apply_block: nrhs must be >= 1");
  std::lock_guard<std::mutex> lk(mtx_);
  DeviceGuard g(device_);
  Ordered o(*this, stream);
  const size_t n = (size_t)N_;
  const int G = imqk::near_block_max();
  for (int k = 0; k < nrhs; k += G)
    apply_block_locked(std::min(G, nrhs - k), d_U + (size_t)k * n, n, d_B + (size_t)k * n, n,
                       stream);
  cuda_check(cudaGetLastError(), "apply_block launch");
}

void DeviceOperator::apply_block_host(int nrhs, const double* U, double* B) {
  if (nrhs < 1) throw std::invalid_argument("apply_block: nrhs must be >= 1");
  std::lock_guard<std::mutex> lk(mtx_);
  DeviceGuard g(device_);
  cudaStream_t s = stream_;
  Ordered o(*this, s);
  const size_t n = (size_t)N_, bytes = n * sizeof(double);
  const int G = std::min(nrhs, imqk::near_block_max());
  io_setup(false, false, false);  // copy streams and events
  const int slots = nrhs > G ? 2 : 1;
  if (blk_io_cap_ < G || (slots == 2 && !d_blk_u_[1])) {
    cuda_check(cudaStreamSynchronize(s), "block slots");
    for (int sl = 0; sl < 2; ++sl) {
      dfree(d_blk_u_[sl]);
      dfree(d_blk_b_[sl]);
    }
    blk_io_cap_ = 0;
    for (int sl = 0; sl < slots; ++sl) {
      d_blk_u_[sl] = dalloc<double>((size_t)G * n, "block input slot");
      d_blk_b_[sl] = dalloc<double>((size_t)G * n, "block output slot");
    }
    blk_io_cap_ = G;
  }
  cuda_check(cudaEventRecord(ev_io_start_, s), "io start");
  cuda_check(cudaStreamWaitEvent(cin_, ev_io_start_, 0), "io wait");
  cuda_check(cudaStreamWaitEvent(cout_, ev_io_start_, 0), "io wait");
  for (int k = 0, gi = 0; k < nrhs; k += G, ++gi) {
    const int sl = slots == 2 ? (gi & 1) : 0, nv = std::min(G, nrhs - k);
    // the slot's previous group (gi - 2) has been gathered / copied out
    if (gi >= slots) cuda_check(cudaStreamWaitEvent(cin_, ev_gath_[sl], 0), "slot wait");
    cuda_check(cudaMemcpyAsync(d_blk_u_[sl], U + (size_t)k * n, (size_t)nv * bytes,
                               cudaMemcpyHostToDevice, cin_), "H2D U");
    cuda_check(cudaEventRecord(ev_in_[sl], cin_), "event");
    cuda_check(cudaStreamWaitEvent(s, ev_in_[sl], 0), "event");
    if (gi >= slots) cuda_check(cudaStreamWaitEvent(s, ev_out_[sl], 0), "event");
    apply_block_locked(nv, d_blk_u_[sl], n, d_blk_b_[sl], n, s);
    cuda_check(cudaEventRecord(ev_gath_[sl], s), "event");
    cuda_check(cudaEventRecord(ev_done_[sl], s), "event");
    cuda_check(cudaStreamWaitEvent(cout_, ev_done_[sl], 0), "event");
    cuda_check(cudaMemcpyAsync(B + (size_t)k * n, d_blk_b_[sl], (size_t)nv * bytes,
                               cudaMemcpyDeviceToHost, cout_), "D2H B");
    cuda_check(cudaEventRecord(ev_out_[sl], cout_), "event");
    cuda_check(cudaGetLastError(), "apply_block kernels");
  }
  cuda_check(cudaStreamSynchronize(cout_), "apply_block");
  cuda_check(cudaStreamSynchronize(cin_), "apply_block");
  cuda_check(cudaStreamSynchronize(s), "apply_block");
  cuda_check(cudaGetLastError(), "apply_block kernels");
}

void DeviceOperator::copy_permutation(int* perm_host) const {
  DeviceGuard g(device_);
  cuda_check(cudaMemcpy(perm_host, d_perm_, (size_t)N_ * sizeof(int), cudaMemcpyDeviceToHost),
             "D2H perm");
}
void DeviceOperator::copy_leaf_start(std::vector<int>& out) const {
  DeviceGuard g(device_);
  const long long n_leaves = 1ll << (2 * (L_ + 1));
  out.resize((size_t)n_leaves + 1);
  cuda_check(cudaMemcpy(out.data(), d_leaf_start_, out.size() * sizeof(int),
                        cudaMemcpyDeviceToHost),
             "D2H leaf_start");
}

// Exact far / near pair counts of this tree (the flop model's P_far, P_near).
PairCounts DeviceOperator::pair_counts() {
  std::lock_guard<std::mutex> lk(mtx_);
  if (have_counts_) {  // pair counts are fixed; the work lists follow restrict_targets
    counts_.far_items = n_far_;
    counts_.near_items = n_near_;
    counts_.near_mode = near_pair_ ? 2 : (near_sym_ ? 1 : 0);
    fill_eval_counts();
    return counts_;
  }
  std::vector<int> ls;
  copy_leaf_start(ls);
  const int L = L_;
  auto count = [&](int l, int i, int j) -> long long {
    const uint32_t q = imqdev::morton((uint32_t)i, (uint32_t)j);
    const int sh = 2 * (L - l);
    return (long long)ls[(size_t)(q + 1) << sh] - ls[(size_t)q << sh];
  };
  double far = 0, near = 0;
  far_by_level_.assign((size_t)L + 1, 0.0);
  ring_direct_ = 0;
  ring_child_by_level_.assign((size_t)L + 1, 0.0);
  ring_par_by_level_.assign((size_t)L + 1, 0.0);
  // number of non-empty level-l ring blocks of the level-(l-1) box (ai, aj)
  auto ring_count = [&](int l, int ai, int aj) {
    const int g1 = 1 << (l + 1);
    long long nr = 0;
    for (int qi = std::max(0, 2 * ai - 2); qi <= std::min(g1 - 1, 2 * ai + 3); ++qi)
      for (int qj = std::max(0, 2 * aj - 2); qj <= std::min(g1 - 1, 2 * aj + 3); ++qj) {
        const int ri = qi - 2 * ai, rj = qj - 2 * aj;
        if ((ri == -2 || ri == 3 || rj == -2 || rj == 3) && count(l, qi, qj) > 0) ++nr;
      }
    return nr;
  };
  for (int l = 2; l < L; ++l) {
    const int ga = 1 << l;
    for (int ai = 0; ai < ga; ++ai)
      for (int aj = 0; aj < ga; ++aj)
        if (count(l - 1, ai, aj)) ring_par_by_level_[(size_t)l] += (double)ring_count(l, ai, aj);
  }
  xring_direct_ = xring_lists_ = 0;
  if (L >= 3) {  // level-L outer rings of the level-(L-1) boxes
    const int ga = 1 << L;
    for (int ai = 0; ai < ga; ++ai)
      for (int aj = 0; aj < ga; ++aj)
        if (count(L - 1, ai, aj)) xring_lists_ += (double)ring_count(L, ai, aj);
  }
  lists_by_level_.assign((size_t)L + 1, 0.0);
  for (int l = 1; l <= L; ++l) {
    const int grid = 1 << (l + 1);
    for (int i = 0; i < grid; ++i)
      for (int j = 0; j < grid; ++j) {
        const long long nt = count(l, i, j);
        if (!nt) continue;
        int lo_i = 0, hi_i = grid - 1, lo_j = 0, hi_j = grid - 1;
        if (l >= 2) {
          lo_i = std::max(0, 2 * (i / 2 - 1)); hi_i = std::min(grid - 1, 2 * (i / 2 + 1) + 1);
          lo_j = std::max(0, 2 * (j / 2 - 1)); hi_j = std::min(grid - 1, 2 * (j / 2 + 1) + 1);
        }
        long long ns = 0;
        for (int qi = lo_i; qi <= hi_i; ++qi)
          for (int qj = lo_j; qj <= hi_j; ++qj)
            if (std::max(std::abs(qi - i), std::abs(qj - j)) >= 2 && count(l, qi, qj) > 0) ++ns;
        far += (double)nt * (double)ns;
        far_by_level_[(size_t)l] += (double)nt * (double)ns;
        lists_by_level_[(size_t)l] += (double)ns;
        if (l >= 2 && l < L) {  // the level-l ring of the parent
          const long long nr = ring_count(l, i >> 1, j >> 1);
          ring_child_by_level_[(size_t)l] += (double)nr;
          if (l == L - 1) ring_direct_ += (double)nt * (double)nr;
        }
        if (l == L && L >= 3) xring_direct_ += (double)nt * (double)ring_count(L, i >> 1, j >> 1);
        if (l == L) {
          long long nn = 0;
          for (int qi = std::max(0, i - 1); qi <= std::min(grid - 1, i + 1); ++qi)
            for (int qj = std::max(0, j - 1); qj <= std::min(grid - 1, j + 1); ++qj)
              nn += count(l, qi, qj);
          near += (double)nt * (double)nn;
        }
      }
  }
  counts_.far_pairs = far;
  counts_.near_pairs = near;
  have_counts_ = true;
  counts_.far_items = n_far_;
  counts_.near_items = n_near_;
  counts_.near_mode = near_pair_ ? 2 : (near_sym_ ? 1 : 0);
  fill_eval_counts();
  return counts_;
}

// Pairs the kernels actually evaluate: direct (target, block) pairs of the
// levels not covered by the Chebyshev pass, and (node, block) pairs.
// This library's kernel launches in one apply_device (every kernel of a product is its own).
int DeviceOperator::kernel_launches_per_apply() const {
  auto groups = [](const std::vector<int>& off) {
    int g = 0;
    for (size_t r = 1; r < off.size(); ++r) g += off[r] > off[r - 1];
    return g;
  };
  // gather, leaf P2M, then the fused M2M + transform per parent level (or,
  // beyond its shared memory, a M2M per parent level and a transform per level)
  int n = 1 + 1 + (d_m2t_ ? std::max(1, L_ - 1) : (L_ - 1) + L_);
  if (near_sym_) n += groups(near_group_off_) + (n_pull_ > 0);
  else if (near_pair_) n += groups(pair_group_off_) + 1;
  else n += groups(near_group_off_) + (near_split_ > 1);
  if (far_split_) {
    std::vector<int> fine(far_group_off_);
    for (int& o : fine) o = std::min(o, n_far_fine_);
    n += (cheb_ && ring_ && xring_ && n_lpart_items_ > 0 ? 0 : groups(fine)) +
         groups(lpart_group_off_);
    if (cheb_) {
      n += groups(cheb_group_off_) + cheb_lc_ + 1;  // node groups, coefficients, evaluation
      for (const GemmPass& g : gnode_) n += g.on ? 1 : 0;
      if (ring_) {
        n += groups(ring_group_off_) + 1;  // ring node groups, level-(L-1) ring coefficients
        if (xring_) n += (xgemm_ ? 1 : groups(xring_group_off_)) + 1;  // X-node pass, coefficients
        for (const GemmPass& g : gring_) n += g.on ? 1 : 0;
        for (int l = std::max(2, ring_l0_); l <= cheb_lc_; ++l) ++n;  // coarse ring coefficients
      }
    } else {
      n += groups(far_cgroup_off_);
    }
  } else {
    n += groups(far_group_off_);
  }
  return n;
}

void DeviceOperator::fill_eval_counts() {
  const int lc = cheb_ ? cheb_lc_ : 0;
  const bool rings = cheb_ && ring_ && ring_par_by_level_.size() == far_by_level_.size();
  constexpr double NN = imqk::kChebN * imqk::kChebN, NRR = imqk::kChebNR * imqk::kChebNR;
  double direct = 0, nodes = 0, gemm = 0;
  for (int l = 1; l <= L_ && l < (int)far_by_level_.size(); ++l) {
    if (l <= lc) {
      const double npl = (size_t)l < inner_v_.size() && inner_v_[(size_t)l]
                             ? (double)imqk::kChebNI * imqk::kChebNI : NN;
      const double p = (lists_by_level_[(size_t)l] -
                        (rings && l >= ring_l0_ ? ring_child_by_level_[(size_t)l] : 0.0)) * npl;
      nodes += p;
      if ((size_t)l < gnode_.size() && gnode_[(size_t)l].on) gemm += p;
    }
    else
      direct += far_by_level_[(size_t)l];
    if (rings && l >= ring_l0_ && l < L_ && (size_t)l - 1 < ring_v_.size()) {
      const double nr = imqk::kRingNr[ring_v_[(size_t)l - 1]];
      const double p = ring_par_by_level_[(size_t)l] * nr * nr;
      nodes += p;
      if ((size_t)l - 1 < gring_.size() && gring_[(size_t)l - 1].on) gemm += p;
    }
  }
  if (rings) direct -= ring_direct_;
  if (rings && xring_ && n_lpart_items_ > 0) {
    // X nodes: level-L outer rings and the level-(L-1) inner lists
    const double inner_lm1 = lists_by_level_[(size_t)L_ - 1] - ring_child_by_level_[(size_t)L_ - 1];
    direct -= xring_direct_ + (far_by_level_[(size_t)L_ - 1] - ring_direct_);
    nodes += (xring_lists_ + inner_lm1) * imqk::kChebNX * imqk::kChebNX;
    if (xgemm_) gemm += (xring_lists_ + inner_lm1) * imqk::kChebNX * imqk::kChebNX;
  }
  counts_.gemm_node_pairs = gemm;
  counts_.far_pairs_direct = direct;
  counts_.cheb_node_pairs = nodes;
  counts_.cheb_levels = lc;
  counts_.cheb_ring = cheb_ && ring_ ? 1 : 0;
  counts_.kernel_launches = kernel_launches_per_apply();
  counts_.cheb_xring = cheb_ && ring_ && xring_ && n_lpart_items_ > 0 ? 1 : 0;
}

// ------------------------------------------------------------------ GMRES --
// solver.cpp:41-159 with every N-vector resident on the device in Morton
// order.  MGS coefficients are produced and consumed on the device; the host
// sees only the (j+2)-entry Hessenberg column per Arnoldi step.
SolveResult DeviceOperator::solve_host(const double* f, double tol, int max_iter, int restart,
                                       double* c) {
  if (!(tol > 0.0) || !std::isfinite(tol))
    throw std::invalid_argument("iterative_solve: tol must be positive");
  if (max_iter < 0) throw std::invalid_argument("iterative_solve: max_iter must be >= 0");
  if (restart < 1) throw std::invalid_argument("iterative_solve: restart must be >= 1");
  const size_t n = (size_t)N_;
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(f[i]))
      throw std::runtime_error("iterative_solve: non-finite value at iteration 0");

  std::lock_guard<std::mutex> lk(mtx_);
  DeviceGuard g(device_);
  cudaStream_t s = stream_;
  Ordered order(*this, s);
  SolveResult rep;
  const auto t_enter = std::chrono::steady_clock::now();
  std::fill(c, c + n, 0.0);

  const int mcap = std::max(1, std::min(restart, max_iter));
  const int nparts = imqk::dot_parts(N_);
  const int mgs_parts = imqk::mgs_grid(N_);
  const size_t hld = (size_t)mcap + 2;  // one Hessenberg column slot per Arnoldi step
  // Arnoldi steps are enqueued kLookahead ahead of the host's Givens
  // processing (the basis and the Hessenberg columns never depend on the
  // rotations), so the GPU does not idle on the per-step host round trip.
  // A step enqueued past convergence is discarded and never counted.
  constexpr int kLookahead = 1, kRing = kLookahead + 2;
  double *d_f = nullptr, *d_x = nullptr, *d_r = nullptr, *d_w = nullptr, *d_V = nullptr;
  double *d_h = nullptr, *d_part = nullptr, *d_mgs = nullptr, *h_pin = nullptr;
  int *d_flag = nullptr, *flag_pin = nullptr;
  void* ws = nullptr;
  cudaEvent_t ev[kRing] = {}, tev[kRing][3] = {};
  const bool trace = opt(kOptTrace);
  auto cleanup = [&]() {
    ws = nullptr;  // solve_ws_ stays cached on the operator
    for (int i = 0; i < kRing; ++i) {
      if (ev[i]) cudaEventDestroy(ev[i]);
      for (auto& e : tev[i])
        if (e) cudaEventDestroy(e);
    }
  };
  try {
    {  // one stream-ordered workspace from the device pool (kept cached by the
       // pool between solves, so repeated solves do not pay cudaMalloc)
      size_t off = 0;
      auto carve = [&](size_t bytes) {
        const size_t o = off;
        off += (bytes + 255) & ~(size_t)255;
        return o;
      };
      const size_t o_f = carve(n * 8), o_x = carve(n * 8), o_r = carve(n * 8), o_w = carve(n * 8);
      const size_t o_V = carve(n * (size_t)(mcap + 1) * 8), o_h = carve(hld * (size_t)(mcap + 1) * 8);
      const size_t o_p = carve((size_t)nparts * 8), o_m = carve(2 * (size_t)mgs_parts * 8);
      const size_t o_fl = carve((size_t)mcap * sizeof(int));
      // The operator's own cached workspace (grown on demand, freed with the
      // operator): the process-wide default pool is left untouched.
      if (solve_ws_bytes_ < off) {
        cuda_check(cudaStreamSynchronize(s), "gmres workspace");
        dfree(solve_ws_);
        solve_ws_bytes_ = 0;
        const cudaError_t e = cudaMalloc(&solve_ws_, off);
        if (e == cudaErrorMemoryAllocation) {
          cudaGetLastError();
          solve_ws_ = nullptr;
          throw std::bad_alloc();
        }
        cuda_check(e, "gmres workspace");
        solve_ws_bytes_ = off;
      }
      ws = solve_ws_;
      char* b = static_cast<char*>(ws);
      d_f = reinterpret_cast<double*>(b + o_f);
      d_x = reinterpret_cast<double*>(b + o_x);
      d_r = reinterpret_cast<double*>(b + o_r);
      d_w = reinterpret_cast<double*>(b + o_w);
      d_V = reinterpret_cast<double*>(b + o_V);
      d_h = reinterpret_cast<double*>(b + o_h);
      d_part = reinterpret_cast<double*>(b + o_p);
      d_mgs = reinterpret_cast<double*>(b + o_m);
      d_flag = reinterpret_cast<int*>(b + o_fl);
    }
    {  // pinned staging for the Hessenberg columns + flags, kept by the operator
      const size_t bytes = hld * (size_t)(mcap + 1) * sizeof(double) + (size_t)mcap * sizeof(int);
      if (bytes > solve_pin_bytes_) {  // (cudaMallocHost costs ms: round up generously)
        if (solve_pin_) cudaFreeHost(solve_pin_);
        solve_pin_ = nullptr;
        solve_pin_bytes_ = 0;
        const size_t cap = std::max(bytes, (size_t)130 * 129 * sizeof(double) + 128 * sizeof(int));
        cuda_check(cudaMallocHost(&solve_pin_, cap), "pinned h");
        solve_pin_bytes_ = cap;
      }
      h_pin = static_cast<double*>(solve_pin_);
      flag_pin = reinterpret_cast<int*>(h_pin + hld * (size_t)(mcap + 1));
    }
    for (int i = 0; i < kRing; ++i) {
      cuda_check(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming), "event");
      if (trace)
        for (auto& e : tev[i]) cuda_check(cudaEventCreate(&e), "event");
    }
    // f in Morton order
    cuda_check(cudaMemcpyAsync(d_u_, f, n * sizeof(double), cudaMemcpyHostToDevice, s), "H2D f");
    imqk::launch_gather(d_u_, d_perm_, N_, d_f, s);
    double* d_scalar = d_h + hld * (size_t)mcap;
    auto nrm2 = [&](const double* v) {
      imqk::launch_dot(v, v, N_, d_part, nparts, d_scalar, 1, s);
      cuda_check(cudaMemcpyAsync(h_pin + hld * (size_t)mcap, d_scalar, sizeof(double),
                                 cudaMemcpyDeviceToHost, s), "D2H norm");
      cuda_check(cudaStreamSynchronize(s), "norm");
      return h_pin[hld * (size_t)mcap];
    };
    auto matvec = [&](const double* in, double* out) { apply_sorted_locked(in, out, nullptr, s); };

    const double bnorm = nrm2(d_f);
    if (bnorm == 0.0) {
      rep.converged = true;
      rep.cycle_residuals.push_back(0.0);
      cleanup();
      return rep;
    }
    double t_mv = 0, t_mgs = 0;
    const auto t_start = std::chrono::steady_clock::now();
    cuda_check(cudaMemsetAsync(d_x, 0, n * sizeof(double), s), "memset x");
    cuda_check(cudaMemcpyAsync(d_r, d_f, n * sizeof(double), cudaMemcpyDeviceToDevice, s), "r=f");
    int total = 0;
    double rel = 1.0;
    std::vector<double> cs((size_t)mcap), sn((size_t)mcap), gv((size_t)mcap + 1), y((size_t)mcap);
    // Arnoldi step jj on the device: w = A v_jj, MGS against v_0..v_jj,
    // h column -> slot jj, v_{jj+1} = w / h_{jj+1,jj}; column + flag -> host.
    auto enqueue = [&](int jj, int m) {
      const int r = jj % kRing;
      if (trace) cudaEventRecord(tev[r][0], s);
      matvec(d_V + (size_t)jj * n, d_w);
      if (trace) cudaEventRecord(tev[r][1], s);
      cuda_check(cudaMemsetAsync(d_flag + jj, 0, sizeof(int), s), "flag");
      cuda_check(imqk::launch_mgs(d_V, d_w, N_, (long long)n, jj, d_mgs, mgs_parts,
                                  d_h + hld * (size_t)jj, d_flag + jj,
                                  jj + 1 < m ? d_V + (size_t)(jj + 1) * n : nullptr, s),
                 "MGS launch");
      if (trace) cudaEventRecord(tev[r][2], s);
      cuda_check(cudaMemcpyAsync(h_pin + hld * (size_t)jj, d_h + hld * (size_t)jj,
                                 (size_t)(jj + 2) * sizeof(double), cudaMemcpyDeviceToHost, s),
                 "D2H h");
      cuda_check(cudaMemcpyAsync(flag_pin + jj, d_flag + jj, sizeof(int), cudaMemcpyDeviceToHost,
                                 s), "D2H flag");
      cuda_check(cudaEventRecord(ev[r], s), "step event");
    };
    while (true) {
      if (total > 0) {
        matvec(d_x, d_w);
        imqk::launch_sub(d_r, d_f, d_w, N_, s);
      }
      rel = nrm2(d_r) / bnorm;
      rep.cycle_residuals.push_back(rel);
      if (!std::isfinite(rel))
        throw std::runtime_error("iterative_solve: non-finite value at iteration " +
                                 std::to_string(total));
      if (rel <= tol || total >= max_iter) break;
      const int m = std::min(restart, max_iter - total);
      const double beta = rel * bnorm;
      imqk::launch_div(d_V, d_r, N_, beta, s);
      std::fill(gv.begin(), gv.end(), 0.0);
      gv[0] = beta;
      int k = 0, enq = 0;
      for (int j = 0; j < m; ++j) {
        while (enq < m && enq <= j + kLookahead) enqueue(enq++, m);
        cuda_check(cudaEventSynchronize(ev[j % kRing]), "arnoldi step");
        ++total;
        if (trace) {
          float a = 0, b2 = 0;
          cudaEventElapsedTime(&a, tev[j % kRing][0], tev[j % kRing][1]);
          cudaEventElapsedTime(&b2, tev[j % kRing][1], tev[j % kRing][2]);
          t_mv += a;
          t_mgs += b2;
        }
        if (flag_pin[j])
          throw std::runtime_error("iterative_solve: non-finite value at iteration " +
                                   std::to_string(total));
        double* h = h_pin + hld * (size_t)j;  // rotated in place (host copy)
        const double hh = h[(size_t)j + 1];
        for (int i = 0; i < j; ++i) {
          const double t0 = cs[(size_t)i] * h[(size_t)i] + sn[(size_t)i] * h[(size_t)i + 1];
          h[(size_t)i + 1] = -sn[(size_t)i] * h[(size_t)i] + cs[(size_t)i] * h[(size_t)i + 1];
          h[(size_t)i] = t0;
        }
        const double denom = std::hypot(h[(size_t)j], hh);
        if (denom == 0.0) {
          k = j;
          break;
        }
        cs[(size_t)j] = h[(size_t)j] / denom;
        sn[(size_t)j] = hh / denom;
        h[(size_t)j] = denom;
        h[(size_t)j + 1] = 0.0;
        gv[(size_t)j + 1] = -sn[(size_t)j] * gv[(size_t)j];
        gv[(size_t)j] = cs[(size_t)j] * gv[(size_t)j];
        k = j + 1;
        const double rel_est = std::fabs(gv[(size_t)j + 1]) / bnorm;
        if (rel_est <= tol || hh == 0.0) break;
      }
      if (k == 0) break;
      for (int i = k - 1; i >= 0; --i) {
        double sacc = gv[(size_t)i];
        for (int l = i + 1; l < k; ++l) sacc -= h_pin[hld * (size_t)l + (size_t)i] * y[(size_t)l];
        y[(size_t)i] = sacc / h_pin[hld * (size_t)i + (size_t)i];
      }
      for (int i = 0; i < k; ++i) imqk::launch_axpy(d_x, d_V + (size_t)i * n, N_, y[(size_t)i], s);
    }
    if (trace) {
      const double wall = std::chrono::duration<double, std::milli>(
                              std::chrono::steady_clock::now() - t_start).count();
      fprintf(stderr, "[imq trace] gmres %d its: wall %.1f ms, matvec %.1f ms, mgs %.1f ms, "
              "setup %.1f ms\n", total, wall, t_mv, t_mgs,
              std::chrono::duration<double, std::milli>(t_start - t_enter).count());
    }
    imqk::launch_scatter(d_x, d_perm_, N_, d_b_, s);
    cuda_check(cudaMemcpyAsync(c, d_b_, n * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H c");
    cuda_check(cudaStreamSynchronize(s), "gmres");
    cuda_check(cudaGetLastError(), "gmres kernels");
    rep.iterations = total;
    rep.final_relative_residual = rel;
    rep.converged = rel <= tol;
  } catch (...) {
    cudaStreamSynchronize(s);
    cleanup();
    throw;
  }
  cleanup();
  if (trace)
    fprintf(stderr, "[imq trace] gmres total %.1f ms\n",
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_enter)
                .count());
  return rep;
}

}  // namespace imqh
