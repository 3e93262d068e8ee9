// operator.hpp -- the device-resident fast operator behind imq_operator.
//
// B200 counterpart of imq::FastOperator (reference fastmv.hpp:19-38):
// immutable after build; holds the Morton-sorted points, leaf offsets, work
// lists and transform tables in HBM plus the per-apply workspace.  apply()
// and solve() serialise on an internal mutex, which keeps the reference's
// "safe for concurrent application to distinct vectors" contract
// (fastmv.hpp:17-18) without duplicating the ~GB workspace.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <mutex>
#include <string>
#include <vector>

#include <memory>

#include "hostio.hpp"
#include "imq_kernels.hpp"

namespace imqh {

struct cuda_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
void cuda_check(cudaError_t e, const char* what);

struct SolveResult {
  int iterations = 0;
  double final_relative_residual = 0.0;
  bool converged = false;
  std::vector<double> cycle_residuals;
};

struct PairCounts {
  double far_pairs = 0, near_pairs = 0;  // exact, from the built tree
  int64_t far_items = 0, near_items = 0;
  int near_mode = 0;  // 0 plain (split sources), 1 symmetric per leaf, 2 chunk pairs
  double far_pairs_direct = 0;  // (target, block) pairs evaluated directly
  double cheb_node_pairs = 0;   // (Chebyshev node, block) pairs (incl. the level-(L-1) ring)
  int cheb_levels = 0;          // levels 1..cheb_levels through the Chebyshev pass
  int cheb_ring = 0;            // level-(L-1) ring through the level-(L-2) nodes
  int kernel_launches = 0;      // this library's kernels per apply_device
  int cheb_xring = 0;           // level-L outer rings through the level-(L-1) nodes
  double gemm_node_pairs = 0;   // of cheb_node_pairs: evaluated by tensor-core GEMMs (nodegemm.cu)
};

// Build-time options (imq_ext_operator_create_opts).  They can only DISABLE
// an approximation or make its gate STRICTER: the default operator uses the
// swept-safe settings, and no option (and no environment variable) can move
// a product further from the reference than the defaults allow.
enum : unsigned {
  kOptNoCheb = 1u << 0,    // no Chebyshev coarse pass (all far pairs direct)
  kOptNoRing = 1u << 1,    // no ring interpolation
  kOptNoInner = 1u << 2,   // inner lists at the level's full node count
  kOptNoXring = 1u << 3,   // no X-ring (level-L outer rings at the targets)
  kOptNoLsplit = 1u << 4,  // no per-leaf partial pass
  kOptNoSplit = 1u << 5,   // single far pass (implies no Chebyshev pass)
  kOptNearNoSym = 1u << 6, // per-target near field (no symmetric evaluation)
  kOptNearNoPair = 1u << 7,// no chunk-pair near field
  kOptCertReport = 1u << 8, // diagnostics: certificate estimated, never acted on
  kOptTrace = 1u << 9,      // diagnostics: GMRES stage timings on stderr
};
constexpr double kCertBudget = 2e-12;  // estimated relative deviation allowed
// Build-time interpolation certificate (operator.cu certify()).
struct CertReport {
  double estimate = 0;  // estimated rel. deviation of a product from the all-direct one
  double budget = 0;    // 0: not run (no interpolation)
  double scale = 0;     // max |b| of the probe product
  double by_kind[5] = {0, 0, 0, 0, 0};  // node levels, inner (NI), rings (NR), rings (NR2), X-ring
  int fallbacks = 0;    // interpolations switched off to meet the budget
  int rounds = 0;       // probe products run
};
struct OperatorOptions {
  unsigned flags = 0;
  // interpolation gates (t / h thresholds); values below the defaults are
  // raised to the defaults (stricter only)
  double ring_tau = 0, ring2_tau = 0, inner_tau = 0, xring_tau = 0;
  // certificate budget (relative); values above kCertBudget are lowered to it
  double cert_budget = 0;
  // scheduling (no effect on any result bit): far items' targets per lane,
  // far-field streams; 0 = automatic
  int far_rmax = 0, far_streams = 0;
};
constexpr double kRingTau = 1.25, kRing2Tau = 2.5, kInnerTau = 2.5, kXringTau = 5.0;

std::vector<int> shard_bounds(const std::vector<int>& leaf_start, int L, int world);
std::vector<double> parent_work(const std::vector<int>& leaf_start, int L, int M);
std::vector<int> shard_bounds_weighted(const std::vector<int>& leaf_start, int L, int world,
                                       const std::vector<double>& w);

// Device far-list enumeration vs the reference lists (far_list_check).
struct ListCheck {
  long long targets = 0, missing = 0, duplicated = 0, extra = 0;
  int max_deviation = 0;  // per target: missing + duplicated + extra
  int max_entries = 0;    // (level, block) entries one target's far passes evaluate
};

class DeviceOperator {
 public:
  DeviceOperator(const double* xy_host, size_t n, double t, int M, int levels,
                 const OperatorOptions& opt = OperatorOptions());
  ~DeviceOperator();
  DeviceOperator(const DeviceOperator&) = delete;
  DeviceOperator& operator=(const DeviceOperator&) = delete;

  int size() const { return N_; }
  int levels() const { return L_; }
  int order() const { return M_; }
  double shape() const { return t_; }
  int device() const { return device_; }
  const double* square() const { return sq_; }

  // Host vectors in original point order (imq_operator_apply semantics);
  // pinned or pageable.
  void apply_host(const double* u, double* b);
  // nrhs host vectors (U: nrhs x N, B: nrhs x N, original order) in a
  // copy / compute pipeline (imq_ext_operator_apply_batch).
  void apply_batch(int nrhs, const double* U, double* B);
  // Device vectors in original order; enqueued on `stream` (0 = the legacy
  // default stream, as everywhere in CUDA), no host synchronisation.
  void apply_device(const double* d_u, double* d_b, cudaStream_t stream);
  // Block product: rows of d_U / d_B (nrhs x N, original
  // order, device).  Groups of up to imqk::near_block_max() vectors go through
  // ONE near-field launch sequence in which every kernel value 1/sqrt(r^2+t^2)
  // is evaluated once and feeds all vectors of the group (the far field is
  // per vector: its GEMM form has no FP64 saving on B200); each
  // b_k equals the single product bit for bit.  Enqueued on `stream`.
  void apply_block_device(int nrhs, const double* d_U, double* d_B, cudaStream_t stream);
  // The same with host matrices; group k+1's copy-in and group k-1's copy-out
  // overlap group k's block product (pinned buffers; pageable ones are
  // copied by the driver's staging and serialise).
  void apply_block_host(int nrhs, const double* U, double* B);
  // Device vectors already in Morton order (no gather/scatter).
  void apply_sorted(const double* d_us, double* d_bs, cudaStream_t stream);

  SolveResult solve_host(const double* f, double tol, int max_iter, int restart, double* c);

  // Sorted-order helpers exposed for tests / multi-GPU orchestration.
  void copy_permutation(int* perm_host) const;
  void copy_leaf_start(std::vector<int>& out) const;
  PairCounts pair_counts();
  const CertReport& certificate() const { return cert_; }
  // Replays every far pass's list enumeration for <= max_targets targets
  // (all when N is smaller, else evenly spread) against the reference lists.
  ListCheck far_list_check(int max_targets);
  // Restricts far/near evaluation to targets at sorted positions [lo, hi)
  // (sharded application); b entries of other targets are left untouched.
  void restrict_targets(int p_lo, int p_hi);
  int target_lo() const { return target_lo_; }
  int target_hi() const { return target_hi_; }

  // Stage-by-stage access (multi-GPU sharding drives these individually);
  // the *_locked variants are the thread-safe entry points of the C ABI.
  void moments_locked(const double* d_us, cudaStream_t s) {
    std::lock_guard<std::mutex> lk(mtx_);
    Ordered o(*this, s);
    moments(d_us, s);
  }
  void far_near_locked(const double* d_us, double* d_out, const int* perm, cudaStream_t s,
                       int fb, int fe, int nb, int ne) {
    std::lock_guard<std::mutex> lk(mtx_);
    Ordered o(*this, s);
    const bool pending = near_pending_;
    near_pending_ = false;
    far_near(d_us, d_out, perm, s, fb, fe, nb, ne, pending);
    // later work on s is ordered after the near field even if this call did
    // not read it (a far-only range)
    if (pending) cuda_check(cudaStreamWaitEvent(s, ev_near_done_, 0), "near join");
  }
  // Starts the symmetric near field of d_us on the operator's near stream
  // (after the work queued on s); the next far_near_locked consumes it
  // instead of launching its own.  No-op unless the near field is symmetric
  // per leaf.  (Sharded ranks: overlaps the near field with the moments.)
  void near_begin(const double* d_us, cudaStream_t s);
  void moments(const double* d_us, cudaStream_t s);  // P2M + M2M + transform
  // Sharded ranks: own + halo moments and own-only coarse partials; the caller
  // all-reduces coarse_moments() over ranks, then calls moments_finish().
  // (Both lock and order themselves, like the *_locked entry points.)
  void moments_local(const double* d_us, cudaStream_t s);
  void coarse_moments(double2** ptr, size_t* count) const;
  void moments_finish(cudaStream_t s);
  bool sharded() const;
  // u (original order) -> Morton order; a sharded (restricted) operator
  // writes only the positions of its own and halo leaves (all it reads).
  void gather(const double* d_u, double* d_us, cudaStream_t s);
  // near_launched: the symmetric near field already runs on near_stream_
  // (apply_sorted_locked); the pass that reads its slots waits for ev_near_done_.
  void far_near(const double* d_us, double* d_out, const int* perm, cudaStream_t s,
                int far_begin, int far_end, int near_begin, int near_end,
                bool near_launched = false);
  double2* coef_ptr() const { return d_coef_; }
  const int* perm_ptr() const { return d_perm_; }
  size_t coef_count() const { return coef_count_; }
  const imqk::TreeParams& params() const { return P_; }
  cudaStream_t stream() const { return stream_; }
  const std::vector<int4>& far_items_host() const { return far_items_h_; }
  const std::vector<int4>& near_items_host() const { return near_items_h_; }
  // restricted operators: the non-empty leaves whose u the rank reads (own +
  // halo), Morton order; empty when unrestricted
  const std::vector<int>& local_leaves_host() const { return local_leaves_h_; }

 private:
  // Device-side ordering of every entry point that touches the operator's
  // internal buffers: each waits for the previous one's work (on whatever
  // stream it ran) and marks its own end, so calls on different streams never
  // overlap on the GPU.
  struct Ordered {
    DeviceOperator& op;
    cudaStream_t s;
    Ordered(DeviceOperator& o, cudaStream_t st) : op(o), s(st) {
      imqh::cuda_check(cudaStreamWaitEvent(s, op.ev_last_, 0), "order wait");
    }
    ~Ordered() { cudaEventRecord(op.ev_last_, s); }
  };
  void build(const double* xy_host);
  void build_items(int p_lo, int p_hi);
  void build_pair_items(int p_lo, int p_hi);
  void build_cheb(int p_lo, int p_hi);
  void certify();
  CertReport cert_{};
  int kernel_launches_per_apply() const;
  void fill_eval_counts();
  std::vector<double> far_by_level_, lists_by_level_;
  // rings: level-(L-1) ring (target, block) pairs; per level l, ring entries of
  // the level-l lists (summed over non-empty boxes) and of the level-(l-1) boxes
  double ring_direct_ = 0;
  double xring_direct_ = 0, xring_lists_ = 0;  // level-L outer rings: target pairs, X lists
  std::vector<double> ring_child_by_level_, ring_par_by_level_;
  void setup_sharded_moments(int p_lo, int p_hi);
  void release();
  void apply_sorted_locked(const double* d_us, double* d_bs, const int* perm,
                           cudaStream_t s);
  // nv <= near_block_max() vectors (original order, strides ldu / ldb); the
  // caller holds the lock and the Ordered guard
  void apply_block_locked(int nv, const double* d_U, size_t ldu, double* d_B, size_t ldb,
                          cudaStream_t s);
  bool block_near_ok() const;
  double* d_blk_us_ = nullptr;    // [blk_cap_][N] Morton-ordered block vectors
  double* d_blk_part_ = nullptr;  // [blk_cap_][5][N] near-field slots per vector
  int blk_cap_ = 0;
  double* d_blk_u_[2] = {nullptr, nullptr};  // host path: group slots [blk_io_cap_][N]
  double* d_blk_b_[2] = {nullptr, nullptr};
  int blk_io_cap_ = 0;

  int device_ = 0;
  OperatorOptions opt_{};
  bool opt(unsigned f) const { return (opt_.flags & f) != 0; }
  cudaStream_t stream_ = nullptr;
  static constexpr int kAuxStreams = 3;  // far-field work groups run concurrently
  cudaStream_t aux_[kAuxStreams] = {};
  int far_streams_ = 1 + kAuxStreams;
  cudaEvent_t ev_fork_ = nullptr;
  cudaEvent_t ev_last_ = nullptr;  // end of the last enqueued entry point (Ordered)
  cudaStream_t near_stream_ = nullptr;  // chunk-pair near field, concurrent with far
  cudaEvent_t ev_near_fork_ = nullptr, ev_near_done_ = nullptr;
  cudaStream_t hp_stream_ = nullptr;  // high-priority critical path (near field overlapped)
  bool near_pending_ = false;          // near_begin ran; far_near_locked waits for it
  cudaEvent_t ev_hp_done_ = nullptr;
  cudaEvent_t ev_join_[kAuxStreams] = {};
  int N_ = 0, M_ = 0, K_ = 0, Ke_ = 0, L_ = 0, pending_levels_ = 0;
  double t_ = 0.0;
  double sq_[3] = {0, 0, 0};
  imqk::TreeParams P_{};
  imqk::TransformTable T_{};
  std::mutex mtx_;

  double* d_xs_ = nullptr;
  double* d_ys_ = nullptr;
  uint32_t* d_leaf_ = nullptr;
  int* d_perm_ = nullptr;
  int* d_leaf_start_ = nullptr;
  int4* d_far_items_ = nullptr;
  int4* d_near_items_ = nullptr;
  int n_far_ = 0, n_near_ = 0;
  std::vector<int4> far_items_h_, near_items_h_;
  std::vector<int> far_group_off_;   // far items grouped by points per lane
  std::vector<int> near_group_off_;  // near items grouped by points per lane
  int* d_tr_off_ = nullptr;
  int* d_tr_idx_ = nullptr;
  double* d_tr_val_ = nullptr;
  double* d_binom_ = nullptr;
  double2* d_m2t_ = nullptr;  // fused M2M tables per parent level (k_m2m_tr), or none
  size_t m2t_stride_ = 0;
  const double2* m2t_V(int l) const { return d_m2t_ + m2t_stride_ * (size_t)(l - 1); }
  const double2* m2t_W(int l) const {
    return m2t_V(l) + (size_t)4 * (M_ + 1) * (M_ + 1);
  }
  double2* d_mu_ = nullptr;
  double2* d_coef_ = nullptr;
  size_t coef_count_ = 0;
  double* d_u_ = nullptr;   // original-order input staging
  double* d_us_ = nullptr;  // sorted input
  double* d_far_ = nullptr; // sorted far field
  double* d_b_ = nullptr;   // original-order output staging
  double* d_part_ = nullptr;  // [3][N] near-field row partials (small problems)
  int near_split_ = 1;
  bool near_sym_ = false;  // symmetric near-field evaluation (small leaves)
  bool near_pair_ = false; // chunk-pair symmetric near field (large leaves)
  bool far_split_ = false; // far field in a coarse (levels 1..L-2) and a fine pass
  std::vector<int> pair_group_off_;  // chunk-pair items grouped by R = 1..kPairR
  // coarse far field by Chebyshev interpolation (build_cheb, cheb.cu)
  bool cheb_ = false;
  int cheb_lc_ = 0, n_cheb_items_ = 0, n_ceval_ = 0;
  size_t cheb_nodes_ = 0;
  std::vector<long long> cheb_base_;   // first box of level l in the node arrays
  std::vector<int> cheb_group_off_, cbox_off_;
  imqk::TreeParams Pn_{};              // P_ with the node coordinates as "points"
  double *d_cnx_ = nullptr, *d_cny_ = nullptr, *d_cval_ = nullptr, *d_ccoef_ = nullptr;
  uint32_t* d_cnleaf_ = nullptr;
  int4 *d_cheb_items_ = nullptr, *d_ceval_items_ = nullptr;
  int* d_cboxes_ = nullptr;
  // level-(L-1) ring through the level-(L-2) boxes' NR x NR nodes (build_cheb)
  bool ring_ = false;
  int ring_l0_ = 0;  // rings of levels ring_l0_..L-1
  std::vector<int> ring_v_;            // ring variant per parent level (kRingNr)
  std::vector<int> inner_v_;           // level's own inner list at NI x NI nodes
  std::vector<long long> cnode_base_;  // first Chebyshev node of each level
  size_t cheb_coefs_ = 0;
  std::vector<long long> ring_nbase_;  // first ring node of each parent level
  // the level-L outer ring through NX x NX nodes of the level-(L-1) boxes
  bool xring_ = false;
  int n_xring_items_ = 0, n_xboxes_ = 0;
  size_t xring_nodes_ = 0;
  std::vector<int> xring_group_off_;
  imqk::TreeParams Px_{};
  double *d_xnx_ = nullptr, *d_xny_ = nullptr, *d_xval_ = nullptr;
  uint32_t* d_xnleaf_ = nullptr;
  int4* d_xring_items_ = nullptr;
  // node passes as tensor-core GEMMs (nodegemm.cu): the X-node pass, the
  // node pass of levels 2..lc, the rings (make_gemm_pass)
  struct GemmPass {
    bool on = false;
    int box_level = 0, n_nodes = 0, n_deltas = 0, k2pad = 0;
    imqk::GemmClasses cls{};
    double* d_A = nullptr;
    imqk::GemmDelta* d_D = nullptr;
    int* d_boxes = nullptr;
    int2* d_order = nullptr;  // CTA -> (class, tile), classes interleaved
    double* out = nullptr;  // node values of box q at out + q * n_nodes
  };
  struct GemmOff {
    int level, dx, dy;
  };
  void make_gemm_pass(GemmPass& g, int box_level, int n_per_dim, const std::vector<double>& rel,
                      const std::vector<int>& boxes, bool by_class,
                      const std::function<void(int, std::vector<GemmOff>&)>& offsets,
                      double* out);
  void free_gemm_pass(GemmPass& g);
  void launch_gemm_pass(const GemmPass& g, cudaStream_t s);
  GemmPass gx_;                          // X-node pass (level L-1 boxes)
  std::vector<GemmPass> gnode_, gring_;  // per level l: node pass of level l / ring of level l+1
  bool xgemm_ = false;

  int* d_xboxes_ = nullptr;
  int n_ring_items_ = 0;
  size_t ring_nodes_ = 0;
  std::vector<int> ring_group_off_;
  imqk::TreeParams Pr_{};
  double *d_rnx_ = nullptr, *d_rny_ = nullptr, *d_rval_ = nullptr, *d_rcoef_ = nullptr;
  uint32_t* d_rnleaf_ = nullptr;
  int4* d_ring_items_ = nullptr;
  int4* d_pull_items_ = nullptr;  // sharded symmetric near field: boundary slots
  int n_pull_ = 0;
  int n_far_fine_ = 0;     // far items [0, n_far_fine_) fine, the rest coarse
  // partial pass (far_split_): per-leaf items for the inner ring of level L
  int n_lpart_items_ = 0;
  bool lpart_leaf2_ = false;  // partial pass: two leaves per warp (k_m2p_leaf2)
  std::vector<int> lpart_group_off_;
  int4* d_lpart_items_ = nullptr;
  std::vector<int> far_cgroup_off_;
  double* d_farc_ = nullptr;  // coarse-pass far partial (sorted order)
  int n_pair_items_ = 0, n_chunks_ = 0;
  int4* d_pair_items_ = nullptr;
  double* d_pair_part_ = nullptr;
  int2* d_chunks_ = nullptr;
  int* d_contrib_off_ = nullptr;
  int* d_contrib_ = nullptr;
  double* d_near_s_ = nullptr;
  // host I/O (apply_batch): copy streams, second device slot, pinned staging
  static constexpr size_t kIoChunk = (size_t)8 << 20;
  void io_setup(bool pin_in, bool pin_out, bool two_slots);
  cudaStream_t cin_ = nullptr, cout_ = nullptr;
  cudaEvent_t ev_io_start_ = nullptr, ev_in_[2] = {}, ev_gath_[2] = {}, ev_done_[2] = {},
              ev_out_[2] = {};
  std::vector<cudaEvent_t> ev_chunk_[2];
  double* d_u2_ = nullptr;
  double* d_b2_ = nullptr;
  double* pin_in_[2] = {nullptr, nullptr};
  double* pin_out_[2] = {nullptr, nullptr};
  std::unique_ptr<CopyPool> pool_;
  void* solve_ws_ = nullptr;  // GMRES device workspace (cached, grown on demand)
  size_t solve_ws_bytes_ = 0;
  void* solve_pin_ = nullptr;  // pinned GMRES staging (Hessenberg columns, flags)
  size_t solve_pin_bytes_ = 0;
  std::vector<int> leaf_start_h_;
  std::vector<int> need_par_h_, local_leaves_h_;  // sharded moments (own + halo)
  int par_lo_ = 0, par_hi_ = 0;
  int* d_need_par_ = nullptr;
  int* d_local_leaves_ = nullptr;
  double2* d_own_lvl_ = nullptr;
  int target_lo_ = 0, target_hi_ = 0;
  bool have_counts_ = false;
  PairCounts counts_{};
};

}  // namespace imqh
