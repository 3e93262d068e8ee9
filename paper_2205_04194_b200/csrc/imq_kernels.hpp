// imq_kernels.hpp -- host-visible launch wrappers for the sm_100a kernels.
//
// Data layout in HBM (all device arrays owned by DeviceOperator):
//   xs, ys      [N]   double  point coordinates in Morton (leaf-major) order
//   leaf        [N]   uint32  finest-level Morton key of each sorted point
//   perm        [N]   int32   sorted position -> original index (stable sort,
//                             so each leaf lists its points in ascending index
//                             order exactly like BlockTree::buckets,
//                             partition.cpp:53-54)
//   leaf_start  [4^(L+1)+1]   first sorted position of every leaf; block q at
//                             level l covers leaves [q<<2(L-l), (q+1)<<2(L-l))
//   mu          [sum_l 4^(l+1) * Ke] double2  raw planar moments per block,
//               mu_{m,i} = sum_j u_j |e_j|^{2i} e_j^m, e_j = y_j - z (complex)
//   coef        [sum_l 4^(l+1) * K]  double2  far-field coefficients C_{m,k}
//               in Horner order (m = M..0, k = M..m); see DESIGN.md §3.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace imqk {

constexpr int kMaxLevels = 14;  // 2(L+1) <= 30 Morton bits

struct TreeParams {
  int N, M, K, Ke, L;
  double t, t2;
  double ox, oy;                    // bounding-square origin
  double cell[kMaxLevels + 1];      // cell[l] = side / 2^(l+1), as partition.cpp:46
  long long mu_off[kMaxLevels + 1];    // first double2 of level l in mu
  long long coef_off[kMaxLevels + 1];  // first double2 of level l in coef
  const double* xs;
  const double* ys;
  const uint32_t* leaf;
  const int* leaf_start;
  int p2m_wpl;  // warps per leaf in the leaf P2M (1, 2, 4, 8)
};

// Transform table mu -> C: for output slot o (Horner order),
// C[o] = sum_{e in [off[o], off[o+1])} val[e] * mu[idx[e]].
struct TransformTable {
  const int* off;
  const int* idx;
  const double* val;
  int nnz;
};

// ---- tree / binning (tree.cu)
void launch_minmax(const double* xy, long long n, double* partial, int nparts, double* out5,
                   cudaStream_t s);
int minmax_parts(long long n);
void launch_bin(const double* xy, long long n, double ox, double oy, double cellL, int gridL,
                uint32_t* keys, int* idx, cudaStream_t s);
void launch_gather_points(const double* xy, const int* perm, long long n, double* xs,
                          double* ys, cudaStream_t s);
void launch_leaf_start(const uint32_t* keys_sorted, long long n, long long n_leaves,
                       int* leaf_start, cudaStream_t s);
void launch_gather(const double* src, const int* perm, long long n, double* dst,
                   cudaStream_t s);
// Only the sorted positions of the listed leaves.
void launch_gather_leaves(const double* src, const int* perm, const int* leaf_start,
                          const int* leaves, int n_leaves, double* dst, cudaStream_t s);
void launch_scatter(const double* src, const int* perm, long long n, double* dst,
                    cudaStream_t s);
size_t sort_temp_bytes(long long n, int bits);
void launch_sort(void* temp, size_t temp_bytes, const uint32_t* k_in, uint32_t* k_out,
                 const int* v_in, int* v_out, long long n, int bits, cudaStream_t s);

// ---- expansion (expansion.cu)
// leaf_list == nullptr: every finest block; else the n_list listed leaves.
void launch_p2m_leaf(const TreeParams& P, const double* u_s, double2* mu, const int* leaf_list,
                     int n_list, cudaStream_t s);
void launch_m2m(const TreeParams& P, int level, double2* mu, const double* binom,
                cudaStream_t s);
// Fused M2M + transform (k_m2m_tr): parents plist[0..np) (or p0 .. p0+np-1)
// at `level` from the children's moments mu_in (level + 1, indexed by child
// block) into mu_out (level, indexed by parent block); coef_child != nullptr:
// also the children's far coefficients (level + 1), coef_parent: the
// parents'.  V, W: the level's translation tables ([4][M+1][M+1] and
// [4][M/2+1][M/2+1] double2, m2m_tables() in host_math).  Needs
// m2m_tr_smem() <= the opt-in shared-memory limit (M <= 24 at the B200's
// 227 KB).
size_t m2m_tr_smem(int M, int Ke, int K, int nnz);
void launch_m2m_tr(const TreeParams& P, int level, const int* plist, long long p0, long long np,
                   const double2* mu_in, double2* mu_out, double2* coef_child,
                   double2* coef_parent, const double2* V, const double2* W,
                   const TransformTable& T, cudaStream_t s);
// Levels [l_lo, l_hi] (<= 0: all); block_list restricts one level's blocks.
void launch_transform(const TreeParams& P, const double2* mu, double2* coef,
                      const TransformTable& T, cudaStream_t s, int l_lo = 0, int l_hi = 0,
                      const int* block_list = nullptr, int n_list = 0);
// Far work items are grouped by points-per-lane R = ceil(count/32):
// group R occupies [group_off[R-1], group_off[R]) of `items`.  Launches the
// items with index in [begin, end).  Group launches are spread round-robin
// over `streams` (streams[0] first, largest R first) so that small groups run
// in the tail of the large ones; the caller forks/joins the streams.
// near_part != nullptr: the symmetric near field already ran; the far kernel's
// epilogue writes out[perm[q]] = far + sum of the nslots near partials.
void launch_m2p_far(const TreeParams& P, const int4* items, const int* group_off, int begin,
                    int end, const double2* coef, double* far_s, const cudaStream_t* streams,
                    int nstreams, const double* near_part = nullptr, int nslots = 0,
                    double* out = nullptr, const int* perm = nullptr,
                    const double* far_add = nullptr, int lmin = 1, int lmax = 0,
                    int ring = 0, int lsplit = 0, bool leaf2 = false);
bool m2p_specialised(int M);
// The far passes' enumeration modes of an operator (k_far_cover replays them).
struct CoverModes {
  int split;    // coarse / fine passes (else one pass over levels 1..L)
  int cheb;     // levels 1..lc through Chebyshev node items
  int lc;       // last node-pass level (L - 2)
  int ring;     // ring items on
  int ring_l0;  // rings of levels ring_l0..L-1
  int xring;    // X-ring items (level-(L-1) inner + level-L outer ring at X's nodes)
  int lsplit;   // per-leaf partial pass
  int leaf2;    // ... run two leaves per warp (k_m2p_leaf2, leaf_inner_list)
};
// out[i] = {missing, duplicated, extra, entries} of targets[i]'s far lists
struct GemmDelta;
// passes run as tensor-core GEMMs (nullptr: through build_far_list): node pass
// of level l (4 box classes), ring of level l + 1 at level-l boxes (1 class),
// X-node pass (4 classes); offsets per class
struct CoverGemm {
  const GemmDelta* node[kMaxLevels + 1];
  int node_nd[kMaxLevels + 1];
  const GemmDelta* ring[kMaxLevels + 1];
  int ring_nd[kMaxLevels + 1];
  const GemmDelta* x;
  int x_nd;
};
void launch_far_cover(const TreeParams& P, const int* targets, int n_t, const CoverModes& Mo,
                      const CoverGemm& Gm, int4* out, cudaStream_t s);

// ---- coarse far field by Chebyshev interpolation (cheb.cu)
#ifndef IMQ_CHEB_N
#define IMQ_CHEB_N 18
#endif
constexpr int kChebN = IMQ_CHEB_N;  // nodes per dimension (degree kChebN - 1), even
// The ring of level L-1 (build_far_list) is interpolated on the level-(L-2)
// boxes at kChebNR^2 nodes (its block centres sit 2.5 half-widths from the box
// centre instead of 4), then restricted to the level-(L-1) boxes at kChebN.
#ifndef IMQ_CHEB_NR
#define IMQ_CHEB_NR 20
#endif
constexpr int kChebNR = IMQ_CHEB_NR;
// Rings whose parent boxes have t >= 2.5 h use fewer nodes (variant 1).
#ifndef IMQ_CHEB_NR2
#define IMQ_CHEB_NR2 16
#endif
constexpr int kChebNR2 = IMQ_CHEB_NR2;
constexpr int kRingNr[2] = {kChebNR, kChebNR2};
// The level-L outer ring of a level-(L-1) box X through NX x NX nodes of X,
// added into X's series (used where t >= tau_x h_X).
#ifndef IMQ_CHEB_NX
#define IMQ_CHEB_NX 12
#endif
constexpr int kChebNX = IMQ_CHEB_NX;
// The own inner lists of the coarse levels with t >= 2.5 h (rings on) through
// NI x NI nodes, their series added into the level's degree-(NC-1) series.
#ifndef IMQ_CHEB_NI
#define IMQ_CHEB_NI 16
#endif
constexpr int kChebNI = IMQ_CHEB_NI;
void cheb_set_inner_tables(const double* T_ni);
void launch_cheb_nodes_inner(const TreeParams& P, int l, long long node_base, double* nx,
                             double* ny, cudaStream_t s);
// coef[X] (NC x NC) += the NI x NI Chebyshev coefficients of the node values
// of each listed box (values at vals + box * NI^2).
void launch_cheb_inner_coef(const int* boxes, int n_boxes, const double* vals, double* coef,
                            cudaStream_t s);
void cheb_set_x_tables(const double* T_nx);
void launch_cheb_nodes_x(const TreeParams& P, int l, double* nx, double* ny, cudaStream_t s);
// coef[X] (NC x NC, x-degree major) += the NX x NX Chebyshev coefficients of
// the node values of each listed box X.
void launch_cheb_xring_coef(const int* boxes, int n_boxes, const double* vals, double* coef,
                            cudaStream_t s);
void cheb_set_tables(const double* T, const double* S_left, const double* S_right);
// Ring variant v (nr = kRingNr[v] nodes per dimension): T_nr[k * nr + i],
// B[half][k' * nr + i]: ring node values on a box A (nr x nr nodes) ->
// degree-(NC-1) coefficients on its child half (interpolation at the child's
// NC nodes of the degree-(nr-1) interpolant).
void cheb_set_ring_tables(int v, const double* T_nr, const double* B_left, const double* B_right);
// nr x nr nodes of every box of level l, written from node index node_base.
void launch_cheb_nodes_ring(const TreeParams& P, int l, int v, long long node_base, double* nx,
                            double* ny, cudaStream_t s);
// One CTA per listed box A: coef_c[child] = B V_A B^T (ring, values at
// ring_vals + a * nr^2) + S C_A S^T (series of A restricted), four children.
void launch_cheb_ring_coef(int v, const int* boxes, int n_boxes, long long base_a,
                           const double* coef_a, const double* ring_vals, double* coef_c,
                           cudaStream_t s);
void launch_cheb_nodes(const TreeParams& P, int l, long long box_base, double* nx, double* ny,
                       cudaStream_t s);
void launch_cheb_coef(int l, const int* boxes, int n_boxes, long long base_l,
                      long long base_parent, const double* vals, double* coef, cudaStream_t s);
void launch_cheb_eval(const TreeParams& P, int lc, const int4* items, int n_items,
                      long long base_lc, const double* coef, double* out, cudaStream_t s);
int cheb_eval_points_per_item();
// Certificate (operator.cu certify()): per listed box, {largest Chebyshev
// coefficient of degree >= n-2 in x or y, max |value|} of its n x n node
// values at vals + box * n^2; max |x_i| into *out (device).
void launch_cheb_tail(const int* boxes, int n_boxes, const double* vals, int n, double2* out,
                      cudaStream_t s);
void launch_absmax(const double* x, long long n, double* out, cudaStream_t s);
// u_i = random_vector(n, seed)[i] (reference.cpp:94-108) on the device.
void launch_random_vector(double* out, long long n, unsigned long long seed, cudaStream_t s);
int far_max_points_per_lane();

// ---- far field at Chebyshev nodes as tensor-core GEMMs (nodegemm.cu)
// One source offset of a box class: the source block at level `level` is the
// box's cell (shifted to that level) + (dx, dy); A = the basis at every node
// for that offset, k-major [k2pad][8 * ceil(n_nodes / 8)] (rows 2j, 2j+1 =
// Re, -Im of the basis of Horner coefficient j).
struct GemmDelta {
  int level, dx, dy, pad;
  const double* A;
};
// Box classes of one launch (boxes of class c: boxes[box_off[c] .. box_off[c+1]),
// offsets deltas[c * n_deltas ..], CTAs [tile_off[c], tile_off[c+1]) of
// node_gemm_tile() boxes each).
struct GemmClasses {
  int n;
  int box_off[5];
  int tile_off[5];
  // CTA -> (class, tile of the class), classes interleaved so the tiles that
  // cover the same parents run together (their sources overlap: L2 reuse);
  // null: CTAs in class order
  const int2* order;
};
// out[box * n_nodes + n] = sum_delta Re sum_j Phi_delta[n][j] C_j(src(box, delta))
void launch_node_gemm(const TreeParams& P, int box_level, const int* boxes,
                      const GemmClasses& G, const GemmDelta* deltas, int n_deltas, int k2pad,
                      const double2* coef, double* out, int n_nodes, cudaStream_t s);
int node_gemm_k2pad(int K);
int node_gemm_tile();
// padded m-tiles of a node count (0: no GEMM kernel for it)
int node_gemm_mt(int n_nodes);
// A[d][k][n] for offsets d (source centre sx, sy relative to the box centre)
// at nodes (nx, ny) relative to the box centre; mp = 8 node_gemm_mt(n_nodes)
void launch_gemm_basis(double* A, const double* sx, const double* sy, int n_off, const double* nx,
                       const double* ny, int n_nodes, int mp, int k2pad, int M, double t2,
                       cudaStream_t s);

// ---- direct interactions (direct.cu)
// Near work items (one leaf each) grouped by points-per-lane like the far ones.
void launch_p2p_near(const TreeParams& P, const int4* items, const int* group_off, int begin,
                     int end, const double* u_s, const double* far_s, double* out,
                     const int* perm, double* part, cudaStream_t s);
void launch_near_combine(int lo, int hi, int N, int nparts, const double* far_s,
                         const double* part, double* out, const int* perm, cudaStream_t s);
int near_max_points_per_lane();
// Symmetric near field (all leaves <= 32 * near_max_points_per_lane() points,
// whole point set): part holds 5 N-vectors (slot 0 forward, 1..4 reverse),
// slots 1..4 zeroed by the caller; combine with launch_near_combine(..., 5).
void launch_p2p_near_sym(const TreeParams& P, const int4* items, const int* group_off, int begin,
                         int end, const double* u_s, double* part, cudaStream_t s);
// Block product: nv <= near_block_max() vectors (vector v at u_s + v ustride,
// its 5 slots at part + v pstride) share every kernel evaluation; each
// vector's sums equal the single-vector launch bit for bit.
int near_block_max();
void launch_p2p_near_sym_block(const TreeParams& P, const int4* items, const int* group_off,
                               int begin, int end, int nv, const double* u_s, size_t ustride,
                               double* part, size_t pstride, cudaStream_t s);
// Chunk-pair symmetric near field (large leaves): items {a_start, a_cnt,
// b_start, b_cnt} (chunks <= 128 points), part = n_items x 256 doubles; the
// reduction adds each chunk's rows (contrib CSR over chunks): out[q] = near
// (far_s == nullptr) or out[perm ? perm[q] : q] = far_s[q] + near.
constexpr int kNearChunk = 128;  // = 32 * kPairR
constexpr int kPairR = 4;  // chunk = 32 * kPairR points; items grouped by R = 1..kPairR
void launch_p2p_pair(const TreeParams& P, const int4* items, const int* group_off,
                     const double* u_s, double* part, cudaStream_t s);
// Sharded symmetric near field: slots of own leaves whose backward neighbour
// belongs to another rank (items {b_start, b_cnt | dir << 16, c_start, c_cnt}).
void launch_p2p_pull(const TreeParams& P, const int4* items, int n_items, const double* u_s,
                     double* part, cudaStream_t s);
void launch_pair_reduce(const int2* chunks, int n_chunks, const int* contrib_off,
                        const int* contrib, const double* part, double* out,
                        const double* far_s, const int* perm, cudaStream_t s);
void launch_direct(const double* txy, long long nt, const double* sxy, const double* sval,
                   long long ns, double t2, double* out, cudaStream_t s);

// ---- vector kernels for the device-resident GMRES (blas.cu)
int dot_parts(long long n);
void launch_dot(const double* a, const double* b, long long n, double* partial, int nparts,
                double* out, int take_sqrt, cudaStream_t s);
void launch_axpy_dev(double* y, const double* x, long long n, const double* alpha_dev,
                     double sign, cudaStream_t s);
void launch_axpy(double* y, const double* x, long long n, double alpha, cudaStream_t s);
void launch_div(double* out, const double* x, long long n, double d, cudaStream_t s);
void launch_sub(double* r, const double* f, const double* w, long long n, cudaStream_t s);
void launch_nonfinite(const double* x, long long n, int* flag, cudaStream_t s);
double measure_dfma_peak(int iters, float* ms_out);  // TFLOP/s of the DFMA pipe
// Whole MGS of one Arnoldi step (h[0..j+1], non-finite flag) in one
// cooperative launch; partial holds 2 * mgs_grid(n) doubles.  With vnext set,
// the kernel also writes v_{j+1} = w / h[j+1] there (w is then left stale).
int mgs_grid(long long n);
cudaError_t launch_mgs(const double* V, double* w, long long n, long long ld, int j,
                       double* partial, int nparts, double* h, int* flag, double* vnext,
                       cudaStream_t s);

}  // namespace imqk
