// nodegemm.cu -- far field at Chebyshev nodes as GEMMs on the FP64 tensor
// cores (mma.sync m8n8k4 f64).
//
// The nodes of every box of a level sit at the same positions relative to
// the box, and a box's interaction list is a fixed set of offsets (clipped at
// the domain edge, empty blocks contributing nothing).  So the field of the
// source block at offset delta, evaluated at node n of ANY box, is
//     V[n] = Re sum_j Phi_delta[n][j] C_j(src)
// with the SAME basis Phi_delta[n][j] = rho^-1 conj(xi)^m q^(k-m) (the
// reference's truncated expansion, fastmv.cpp:104-138, in the monomial form
// of DESIGN.md §3; j over the Horner-ordered coefficients (m, k)).  The node
// pass of a box class is then one GEMM per offset,
//     V[n][box] += sum_k A_delta[k][n] B_delta[k][box],
// A_delta = the basis (real form: rows 2j, 2j+1 = Re, -Im), B_delta = the
// source coefficients of each box's delta-neighbour (Re, Im interleaved,
// exactly the coefficient array).  This replaces the per-(node, source)
// complex Horner of k_m2p_far (LDS-fed, ~76 % of the FP64 pipe) by dense
// tensor-core tiles with no idle target slots; in real arithmetic it is the
// same sum.
//
// CTA: 32 boxes x all nodes (MT m-tiles of 8), 4 consumer warps as 2 box
// pairs x 2 node halves (each A fragment feeds two tensor-core ops) + two
// producer warps; k in chunks of 16 (4 mma k-steps), A and B chunks staged by
// TMA bulk copies (one per A row and per box row, dealt to the producers'
// lanes, completion on the stage's `full` mbarrier; the consumers hand a
// stage back through its `empty` mbarrier) in a 2-stage ring.  Measured at
// config 4 (X-node pass, 65,536 boxes x 144 nodes x 27 offsets; ncu, tensor
// pipe active), TMA staging: 32 boxes / k16 / 2 stages 4.73 ms (86.3 %),
// 32 / 32 / 2 4.82 ms (84.2 %), 64 / 16 / 2 5.26 ms (78.2 %), 64 / 16 / 3
// 5.29 ms, 32 / 16 / 3 5.63 ms (71.6 %: 2 CTAs per SM), 32 / 8 / 3 6.72 ms
// (60.8 %: one producer warp cannot issue 40 copies per half-size step).
// With per-thread cp.async staging the same tile took 5.33 ms (76.8 %); the
// Horner pass it replaces 6.96 ms.
#include <algorithm>
#include <mutex>
#include <set>
#include <stdexcept>
#include <string>
#include <utility>

#include "imq_device.cuh"
#include "imq_kernels.hpp"

#ifndef IMQ_GEMM_NB
#define IMQ_GEMM_NB 32
#endif
#ifndef IMQ_GEMM_KC
#define IMQ_GEMM_KC 16
#endif
#ifndef IMQ_GEMM_SMALL
#define IMQ_GEMM_SMALL 0  // passes with fewer 32-box tiles per SM than this use 16-box tiles (8: one rank of 8 at config 4 1.14 ms vs 0.95 ms: off)
#endif
#ifndef IMQ_GEMM_ST
#define IMQ_GEMM_ST 2
#endif
#ifndef IMQ_GEMM_PRODUCERS
#define IMQ_GEMM_PRODUCERS 2
#endif

namespace imqk {

namespace {

using namespace imqdev;

// boxes per CTA (warps = kGtN / 8: box pairs x 2 node halves), k chunk, stages
constexpr int kGtN = IMQ_GEMM_NB, kGtKC = IMQ_GEMM_KC, kGtStages = IMQ_GEMM_ST;
constexpr int kGtNSmall = 16;  // boxes per CTA when the pass has too few tiles to fill the GPU
constexpr int kGtMaxDelta = 32;
constexpr int kGtProducers = IMQ_GEMM_PRODUCERS;  // staging warps per CTA
constexpr int kGtSBn = kGtKC % 16 == 0 ? kGtKC + 4 : kGtKC + 12;  // B rows [box][k]: stride = 4 (mod 16)
static_assert(kGtN >= kGtNSmall, "tile sizes");

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__host__ __device__ constexpr int gemm_sa(int MT) {  // A rows [k][node]: stride = 4 (mod 16)
  return 8 * MT + ((4 - (8 * MT) % 16) + 16) % 16;
}
constexpr size_t gemm_smem(int MT, int NB) {
  return (size_t)kGtStages * kGtKC * gemm_sa(MT) * sizeof(double) +
         (size_t)kGtStages * NB * kGtSBn * sizeof(double) +
         (size_t)kGtMaxDelta * NB * sizeof(const double*) + (size_t)2 * kGtStages * sizeof(uint64_t);
}

// rows of absent sources (outside the grid, empty blocks) are copied from here
constexpr int kGtZeros = 512;
__device__ __align__(16) double g_gemm_zeros[kGtZeros];

__device__ __forceinline__ int gemm_block_count(const TreeParams& P, int level, uint32_t q) {
  const int sh = 2 * (P.L - level);
  return P.leaf_start[(size_t)(q + 1) << sh] - P.leaf_start[(size_t)q << sh];
}

// MT: m-tiles (nodes padded to 8 MT).  The (offset, k-chunk) steps run as one
// flattened cp.async pipeline of kGtStages stages: no bubble at offset
// boundaries, no register staging.  Source pointers of every (offset, box)
// are resolved once at the start (null: outside the grid or empty block ->
// zero-filled B rows).
// MG: node-tile groups (warps = NB / 16 box pairs x MG, MT / MG m-tiles each);
// NB: boxes per CTA
template <int MT, int MG, int NB>
__global__ void __launch_bounds__((NB / 16 * MG + kGtProducers) * 32) k_node_gemm(
    const TreeParams P, int box_level, const int* __restrict__ boxes_all, const GemmClasses G,
    const GemmDelta* __restrict__ deltas_all, int n_deltas, int k2pad,
    const double2* __restrict__ coef, double* __restrict__ out, int n_nodes) {
  constexpr int MP = 8 * MT;
  constexpr int SA = gemm_sa(MT);
  extern __shared__ __align__(16) double gsm[];
  double* As = gsm;                                   // [stage][KC][SA]
  double* Bs = gsm + (size_t)kGtStages * kGtKC * SA;  // [stage][N][SBn]
  const double** srcs = reinterpret_cast<const double**>(Bs + (size_t)kGtStages * NB * kGtSBn);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int r = lane >> 2, c = lane & 3;
  // this CTA's box class: its boxes and its offsets (tiles never straddle classes)
  int cls = 0, tile;
  if (G.order) {
    const int2 o = G.order[blockIdx.x];
    cls = o.x;
    tile = o.y;
  } else {
    while (cls + 1 < G.n && (int)blockIdx.x >= G.tile_off[cls + 1]) ++cls;
    tile = (int)blockIdx.x - G.tile_off[cls];
  }
  const int* boxes = boxes_all + G.box_off[cls];
  const int n_boxes = G.box_off[cls + 1] - G.box_off[cls];
  const GemmDelta* deltas = deltas_all + (size_t)cls * n_deltas;
  const int b0 = tile * NB;
  for (int e = tid; e < n_deltas * NB; e += blockDim.x) {
    const int di = e / NB, n = e % NB;
    const GemmDelta D = deltas[di];
    const double* p = nullptr;
    if (b0 + n < n_boxes) {
      int bi, bj;
      demorton((uint32_t)boxes[b0 + n], bi, bj);
      const int sh = D.level - box_level;
      const int si = (bi << sh) + D.dx, sj = (bj << sh) + D.dy, g = 1 << (D.level + 1);
      if (si >= 0 && sj >= 0 && si < g && sj < g) {
        const uint32_t q = morton((uint32_t)si, (uint32_t)sj);
        if (gemm_block_count(P, D.level, q) > 0)
          p = reinterpret_cast<const double*>(coef + P.coef_off[D.level] + (size_t)q * P.K);
      }
    }
    srcs[e] = p ? p : g_gemm_zeros;
  }
  // B stages start as zeros: a chunk shorter than the k chunk leaves the rest
  // of its rows as they were, and those meet zero rows of A (0 x finite)
  for (int e = tid; e < kGtStages * NB * kGtSBn; e += blockDim.x) Bs[e] = 0.0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  uint64_t* bars = reinterpret_cast<uint64_t*>(srcs + (size_t)kGtMaxDelta * NB);
  // full[stage]: the producer's expect_tx arrival + the copies' bytes;
  // empty[stage]: one arrival per consumer warp when it is done reading
  static_assert(MT % MG == 0 && NB % 16 == 0, "m-tiles over MG warp rows, box pairs");
  constexpr int MH = MT / MG, NP = NB / 16, NW = NP * MG;
  uint64_t* full = bars;
  uint64_t* empty = bars + kGtStages;
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < kGtStages; ++i) {
      mbar_init(&full[i], kGtProducers);
      mbar_init(&empty[i], NW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int k2 = 2 * P.K, nchunk = k2pad / kGtKC, nsteps = n_deltas * nchunk;
  if (warp >= NW) {
    // producer warps: stage step after step as the consumers free the ring.
    // The kGtKC A rows (row k0 + k, all nodes) and the NB box rows (the
    // coefficients k0.. of each box's source, only the part below 2K: the
    // rest of the row keeps finite values of an earlier chunk, times zero
    // rows of A) are dealt round-robin to the producers' lanes: a bulk copy
    // issues lane by lane (UBLKCP), ~48 of them per step are more than one
    // warp can issue in the time the consumers need for the step's DMMAs.
    const int pw = warp - NW;
    for (int step = 0; step < nsteps; ++step) {
      const int di = step / nchunk, k0 = (step % nchunk) * kGtKC, st = step % kGtStages;
      if (step >= kGtStages) mbar_wait(&empty[st], (uint32_t)((step / kGtStages - 1) & 1));
      const int kb = min(kGtKC, k2 - k0);
      uint64_t* bar = &full[st];
      if (lane == 0) {  // this producer's share of the step's bytes
        int na = 0, nb = 0;
        for (int i = pw; i < kGtKC + NB; i += kGtProducers) (i < kGtKC ? na : nb) += 1;
        mbar_arrive_expect_tx(bar, (uint32_t)((na * MP + nb * kb) * sizeof(double)));
      }
      __syncwarp();
      const double* A = deltas[di].A + (size_t)k0 * MP;
      double* as = As + (size_t)st * kGtKC * SA;
      double* bs = Bs + (size_t)st * NB * kGtSBn;
      const double* const* sp = srcs + di * NB;
      for (int i = pw + kGtProducers * lane; i < kGtKC + NB; i += kGtProducers * 32) {
        if (i < kGtKC)
          tma_load_1d(as + i * SA, A + (size_t)i * MP, MP * sizeof(double), bar);
        else
          tma_load_1d(bs + (i - kGtKC) * kGtSBn, sp[i - kGtKC] + k0, kb * sizeof(double), bar);
      }
    }
    return;
  }
  // consumer warp w: boxes of n-tiles 2 np, +1 and m-tiles [mh MH, +MH), np =
  // w % (N / 16), mh = w / (N / 16): every A fragment feeds two tensor-core ops
  const int np = warp % NP, mh = warp / NP;
  double acc[MH][2][2];
#pragma unroll
  for (int mt = 0; mt < MH; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
  for (int step = 0; step < nsteps; ++step) {
    const int st = step % kGtStages;
    mbar_wait(&full[st], (uint32_t)((step / kGtStages) & 1));
    const int kleft = k2 - (step % nchunk) * kGtKC;  // the last chunk's k-steps past 2K are all zero
    const double* as = As + (size_t)st * kGtKC * SA + mh * MH * 8 + r;
    const double* bs = Bs + (size_t)st * NB * kGtSBn + (size_t)(np * 16 + r) * kGtSBn;
#pragma unroll
    for (int ks = 0; ks < kGtKC / 4; ++ks) {
      if (4 * ks >= kleft) break;
      const double b0 = bs[ks * 4 + c], b1 = bs[8 * kGtSBn + ks * 4 + c];
      const double* ar = as + (ks * 4 + c) * SA;
#pragma unroll
      for (int mt = 0; mt < MH; ++mt) {
        const double a = ar[mt * 8];
        dmma(acc[mt][0][0], acc[mt][0][1], a, b0);
        dmma(acc[mt][1][0], acc[mt][1][1], a, b1);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);  // this warp is done with stage st
  }
  // C fragment: rows (mh MH + mt) 8 + r (nodes), columns (2 np + nt) 8 + 2c, +1 (boxes)
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int bx = b0 + (2 * np + nt) * 8 + 2 * c + h;
      if (bx >= n_boxes) continue;
      double* o = out + (size_t)boxes[bx] * n_nodes;
#pragma unroll
      for (int mt = 0; mt < MH; ++mt) {
        const int n = (mh * MH + mt) * 8 + r;
        if (n < n_nodes) o[n] = acc[mt][nt][h];
      }
    }
}

}  // namespace

// nodes -> (MT, MG): MT m-tiles of 8 (padded), MG warp rows of <= 10 m-tiles
int node_gemm_mt(int n_nodes) {
  switch ((n_nodes + 7) / 8) {
    case 18: return 18;                    // 12 x 12 (X-ring)
    case 32: return 32;                    // 16 x 16
    case 41: case 42: return 42;           // 18 x 18
    case 50: return 50;                    // 20 x 20
    default: return 0;
  }
}

void launch_node_gemm(const TreeParams& P, int box_level, const int* boxes,
                      const GemmClasses& G, const GemmDelta* deltas, int n_deltas, int k2pad,
                      const double2* coef, double* out, int n_nodes, cudaStream_t s) {
  if (G.n < 1 || G.tile_off[G.n] <= 0) return;
  if (k2pad % kGtKC) throw std::invalid_argument("node gemm: k2pad must be a multiple of the k chunk");
  if (n_deltas > kGtMaxDelta) throw std::invalid_argument("node gemm: too many offsets");
  if (k2pad > kGtZeros) throw std::invalid_argument("node gemm: order too large for the zero block");
  auto run = [&](auto kern, size_t smem, int warps, const GemmClasses& Gx) {
    const unsigned grid = (unsigned)Gx.tile_off[Gx.n];
    // the attribute is per (kernel, device); every instantiation has the same
    // function-pointer type, so key by the pointer
    static std::mutex mtx;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    cudaGetDevice(&dev);
    {
      std::lock_guard<std::mutex> lk(mtx);
      if (done.insert({(const void*)kern, dev}).second &&
          cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem) != cudaSuccess) {
        cudaGetLastError();
        done.erase({(const void*)kern, dev});
        throw std::runtime_error("node gemm: shared-memory attribute");
      }
    }
    kern<<<grid, (warps + kGtProducers) * 32, smem, s>>>(P,  // + the producer warps
        box_level, boxes, Gx, deltas, n_deltas, k2pad, coef,
                                        out, n_nodes);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
      throw std::runtime_error(std::string("node gemm launch (") + std::to_string(n_nodes) +
                               " nodes, " + std::to_string(smem) + " B shared): " +
                               cudaGetErrorString(e));
  };
  // the grid is laid out in tiles of kGtN boxes; a pass with fewer tiles than
  // ~2 per SM slot (e.g. one rank's share of a sharded product) runs tiles of
  // kGtNSmall boxes instead -- the class tile offsets scale with the tile size
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const bool small = (long long)G.tile_off[G.n] < (long long)IMQ_GEMM_SMALL * sms;
  GemmClasses Gs = G;
  if (small) {
    Gs.order = nullptr;  // the interleaved order is laid out for kGtN-box tiles
    Gs.tile_off[0] = 0;
    for (int c = 0; c < G.n; ++c)
      Gs.tile_off[c + 1] = Gs.tile_off[c] + (G.box_off[c + 1] - G.box_off[c] + kGtNSmall - 1) / kGtNSmall;
  }
  auto go = [&](auto kbig, auto ksmall, int mt, int mg) {
    if (small)
      run(ksmall, gemm_smem(mt, kGtNSmall), kGtNSmall / 16 * mg, Gs);
    else
      run(kbig, gemm_smem(mt, kGtN), kGtN / 16 * mg, G);
  };
  switch (node_gemm_mt(n_nodes)) {
    case 18: go(k_node_gemm<18, 2, kGtN>, k_node_gemm<18, 2, kGtNSmall>, 18, 2); break;
    case 32: go(k_node_gemm<32, 4, kGtN>, k_node_gemm<32, 4, kGtNSmall>, 32, 4); break;
    case 42: go(k_node_gemm<42, 6, kGtN>, k_node_gemm<42, 6, kGtNSmall>, 42, 6); break;
    case 50: go(k_node_gemm<50, 5, kGtN>, k_node_gemm<50, 5, kGtNSmall>, 50, 5); break;
    default: throw std::invalid_argument("node gemm: unsupported node count");
  }
}

// A[d][k][n] (k-major, n padded to 8 MT): the basis of Horner coefficient j =
// k / 2 at node n for source offset d: rho^-1 conj(xi)^m q^(k-m) (rows 2j, 2j+1
// = Re, -Im), from the node position relative to its box centre (nx, ny)
// minus the source centre relative to it (sx[d], sy[d]).
__global__ void k_gemm_basis(double* __restrict__ A, const double* __restrict__ sx,
                             const double* __restrict__ sy, int n_off, const double* __restrict__ nx,
                             const double* __restrict__ ny, int n_nodes, int mp, int k2pad, int M,
                             double t2) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)n_off * mp) return;
  const int d = (int)(t / mp), n = (int)(t % mp);
  double* Ad = A + (size_t)d * k2pad * mp;
  if (n >= n_nodes) {
    for (int k = 0; k < k2pad; ++k) Ad[(size_t)k * mp + n] = 0.0;
    return;
  }
  const double dx = nx[n] - sx[d], dy = ny[n] - sy[d];
  const double r = 1.0 / sqrt(fma(dx, dx, fma(dy, dy, t2))), q = r * r;
  const double xr = dx * q, xi = -dy * q;
  int jb = 0;  // first Horner slot of group m (groups m = M..0, k = top(m)..m)
  for (int m = M; m >= 0; --m) {
    double mr = 1.0, mi = 0.0;  // conj(xi)^m
    for (int e = 0; e < m; ++e) {
      const double tr = mr * xr - mi * xi;
      mi = mr * xi + mi * xr;
      mr = tr;
    }
    const int top = M - ((M - m) & 1);
    double f = r;  // r q^(k - m)
    for (int k = m; k <= top; ++k) {
      const int j = jb + (top - k);
      Ad[(size_t)(2 * j) * mp + n] = f * mr;
      Ad[(size_t)(2 * j + 1) * mp + n] = -f * mi;
      f *= q;
    }
    jb += top - m + 1;
  }
  for (int k = 2 * jb; k < k2pad; ++k) Ad[(size_t)k * mp + n] = 0.0;
}

void launch_gemm_basis(double* A, const double* sx, const double* sy, int n_off, const double* nx,
                       const double* ny, int n_nodes, int mp, int k2pad, int M, double t2,
                       cudaStream_t s) {
  const long long n = (long long)n_off * mp;
  if (n > 0)
    k_gemm_basis<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(A, sx, sy, n_off, nx, ny, n_nodes, mp,
                                                            k2pad, M, t2);
}

int node_gemm_k2pad(int K) { return ((2 * K + kGtKC - 1) / kGtKC) * kGtKC; }
int node_gemm_tile() { return kGtN; }

}  // namespace imqk
