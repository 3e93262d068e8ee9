// TEST / MEASUREMENT INFRASTRUCTURE (compiled only into oracle/_ref/, never
// shipped): a bounded, stage-by-stage timing of the REFERENCE'S OWN fast-matvec
// routines on the exact geometry of a large configuration (config 4: N =
// 16.8M, L = 8), for bench.py's CPU baseline and --impl reference arm.
//
// A full config-4 product of the reference takes ~168 s to build (the
// O(grid^4) list build, partition.cpp:56-72) plus ~8 min to apply on 8 cores,
// and its trig cache needs ~37 GB (fastmv.cpp:41-74) -- too long for a bench
// step.  This driver times the reference's public per-stage routines
// (fastmv.hpp) on stratified samples of the same problem and scales each by
// its exact work ratio:
//   moments  imq::compute_moments (fastmv.cpp:140-148 -> accumulate_moments
//            79-100) over every block of every level, restricted to the points
//            of `n_mom` randomly chosen finest blocks (the work of a block is
//            linear in its points): t_mom * (N / sampled points);
//   far      imq::apply_far (fastmv.cpp:150-159 -> accumulate_far_block
//            104-138) of every source block of the interaction lists of the
//            sampled target leaves' ancestors, onto those targets (threads
//            take source blocks, private b): t_far * (N / sampled targets);
//   near     imq::apply_near (fastmv.cpp:161-182, its own OpenMP loop) over
//            the sampled target leaves: t_near * (N / sampled targets).
// The operator structs are filled the way build_operator does
// (fastmv.cpp:32-77, partition.cpp:36-85), with the reference's own
// bounding_square / block_of, but only for the sampled blocks (no O(grid^4)
// list build, no full-size cache).  The far stage evaluates dummy moments
// (all ones): its cost does not depend on the moment values.
#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <vector>

#include "imq/fastmv.hpp"
#include "imq/partition.hpp"
#include "imq/specfun.hpp"

namespace {

using Clock = std::chrono::steady_clock;
double secs(Clock::time_point a, Clock::time_point b) {
  return std::chrono::duration<double>(b - a).count();
}

uint64_t splitmix(uint64_t& s) {
  s += 0x9E3779B97F4A7C15ull;
  uint64_t z = s;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Tree skeleton: square, levels, grids, centers (partition.cpp:44-52).
imq::BlockTree skeleton(const imq::Square& sq, int L) {
  imq::BlockTree tree;
  tree.square = sq;
  tree.L = L;
  tree.levels.resize(L);
  for (int l = 1; l <= L; ++l) {
    imq::BlockTree::Level& lv = tree.levels[l - 1];
    lv.grid = 1 << (l + 1);
    const int nb = lv.grid * lv.grid;
    lv.buckets.assign(nb, {});
    lv.slist.assign(nb, {});
    lv.centers.resize(nb);
    const double cell = sq.side / lv.grid;
    for (int i = 0; i < lv.grid; ++i)
      for (int j = 0; j < lv.grid; ++j)
        lv.centers[i * lv.grid + j] = {sq.origin.x1 + (i + 0.5) * cell, sq.origin.x2 + (j + 0.5) * cell};
  }
  tree.near_lists.assign((size_t)tree.levels[L - 1].grid * tree.levels[L - 1].grid, {});
  return tree;
}

// Per-level point cache of fastmv.cpp:53-74 for the operator's points.
void fill_cache(imq::FastOperator& op) {
  const int M = op.order.M, N = op.size();
  op.cache.assign(op.L, {});
  for (int l = 1; l <= op.L; ++l) {
    const imq::BlockTree::Level& lv = op.tree.levels[l - 1];
    imq::FastOperator::PointCache& pc = op.cache[l - 1];
    pc.rho.assign(N, 0.0);
    pc.cosm.assign((size_t)N * (M + 1), 0.0);
    pc.sinm.assign((size_t)N * (M + 1), 0.0);
    for (int blk = 0; blk < (int)lv.buckets.size(); ++blk) {
      const imq::Point2 z = lv.centers[blk];
      for (int j : lv.buckets[blk]) {
        const double dx = op.points[j].x1 - z.x1, dy = op.points[j].x2 - z.x2;
        const double rho = std::sqrt(dx * dx + dy * dy);
        pc.rho[j] = rho;
        double cw = 1.0, sw = 0.0;
        if (rho > 0.0) {
          cw = dx / rho;
          sw = dy / rho;
        }
        double* cm = &pc.cosm[(size_t)j * (M + 1)];
        double* sm = &pc.sinm[(size_t)j * (M + 1)];
        cm[0] = 1.0;
        sm[0] = 0.0;
        for (int m = 1; m <= M; ++m) {
          cm[m] = cm[m - 1] * cw - sm[m - 1] * sw;
          sm[m] = sm[m - 1] * cw + cm[m - 1] * sw;
        }
      }
    }
  }
}

}  // namespace

extern "C" {

// xy: n interleaved points; u: n values.  Samples (seeded): n_mom random
// non-empty finest blocks for the moments; ~n_tgt target leaves for far +
// near, as whole 8 x 8-leaf tiles.
// out[0..6] = {t_moments, t_far, t_near (s, sampled), points in the moment
// sample, sampled targets, far (target, block) pairs evaluated, estimated
// full-product seconds}.  Returns 0, or -1 on bad input.
int imqref_sample_time(const double* xy, long long n, double t, int M, int L, const double* u,
                       int n_mom, int n_tgt, unsigned long long seed, int threads, double* out) {
  if (!xy || !u || !out || n < 1 || L < 2 || M < 0 || n_mom < 1 || n_tgt < 1) return -1;
  if (threads > 0) omp_set_num_threads(threads);
  {  // start the OpenMP team outside the timed regions
    volatile double w = 0.0;
#pragma omp parallel
    { w = w + 1.0; }
  }
  std::vector<imq::Point2> pts((size_t)n);
  for (long long i = 0; i < n; ++i) pts[(size_t)i] = {xy[2 * i], xy[2 * i + 1]};
  const imq::Square sq = imq::bounding_square(pts);
  imq::BlockTree ref_tree = skeleton(sq, L);  // for block_of
  const int gL = 1 << (L + 1);
  // finest block of every point (partition.cpp:25-33) and bucket counts
  std::vector<int> leaf((size_t)n);
  std::vector<int> occ((size_t)gL * gL, 0);
  for (long long i = 0; i < n; ++i) {
    leaf[(size_t)i] = ref_tree.block_of(L, pts[(size_t)i]);
    ++occ[(size_t)leaf[(size_t)i]];
  }
  std::vector<int> nonempty;
  for (int b = 0; b < gL * gL; ++b)
    if (occ[(size_t)b]) nonempty.push_back(b);
  uint64_t s = seed;
  // random non-empty leaves (moments: the work of a block is linear in its points)
  auto pick = [&](int k) {
    std::vector<char> sel((size_t)gL * gL, 0);
    k = std::min<int>(k, (int)nonempty.size());
    for (int c = 0; c < k;) {
      const int b = nonempty[(size_t)(splitmix(s) % nonempty.size())];
      if (!sel[(size_t)b]) {
        sel[(size_t)b] = 1;
        ++c;
      }
    }
    return sel;
  };
  // target leaves in whole level-(L-3) blocks (8 x 8 leaves), so that the
  // target blocks of every level are as full as in a complete product and
  // each apply_far call does a complete product's amount of work
  auto pick_tiles = [&](int k) {
    const int tl = std::min(3, L - 1), tg = gL >> tl;  // tiles per dimension
    std::vector<char> sel((size_t)gL * gL, 0), used((size_t)tg * tg, 0);
    const int want = std::max(1, std::min(k >> (2 * tl), tg * tg));
    for (int c = 0; c < want;) {
      const int tile = (int)(splitmix(s) % (uint64_t)(tg * tg));
      if (used[(size_t)tile]) continue;
      used[(size_t)tile] = 1;
      ++c;
      const int ti = tile / tg, tj = tile % tg;
      for (int a = ti << tl; a < (ti + 1) << tl; ++a)
        for (int b = tj << tl; b < (tj + 1) << tl; ++b)
          if (occ[(size_t)(a * gL + b)]) sel[(size_t)(a * gL + b)] = 1;
    }
    return sel;
  };

  // ---------------- moments: all levels over the points of n_mom leaves
  double t_mom = 0.0, mom_pts = 0.0;
  {
    const std::vector<char> sel = pick(n_mom);
    imq::FastOperator op{imq::KernelParams(t), imq::ExpansionOrder(M)};
    for (long long i = 0; i < n; ++i)
      if (sel[(size_t)leaf[(size_t)i]]) op.points.push_back(pts[(size_t)i]);
    std::vector<double> uu;
    for (long long i = 0; i < n; ++i)
      if (sel[(size_t)leaf[(size_t)i]]) uu.push_back(u[i]);
    op.L = L;
    op.tree = skeleton(sq, L);
    for (int j = 0; j < op.size(); ++j)
      for (int l = 1; l <= L; ++l)
        op.tree.levels[l - 1].buckets[(size_t)op.tree.block_of(l, op.points[(size_t)j])].push_back(j);
    op.dtab = imq::coeff_d_table(M);
    op.pn0.resize(op.order.K);
    imq::assoc_legendre_table(M, 0.0, 1.0, op.pn0.data());
    fill_cache(op);
    mom_pts = (double)op.size();
    // every non-empty (level, block) of the sample, one parallel loop (the
    // reference's is per level over all blocks, fastmv.cpp:192-197; a sparse
    // sample would be dominated by its empty-block scheduling)
    std::vector<std::pair<int, int>> blocks;
    for (int l = 1; l <= L; ++l)
      for (int blk = 0; blk < (int)op.tree.levels[l - 1].buckets.size(); ++blk)
        if (!op.tree.levels[l - 1].buckets[(size_t)blk].empty()) blocks.push_back({l, blk});
    double sink = 0.0;
    const auto a = Clock::now();
#pragma omp parallel for schedule(dynamic, 4) reduction(+ : sink)
    for (size_t k = 0; k < blocks.size(); ++k) {
      const imq::Moments mm = imq::compute_moments(op, blocks[k].first, blocks[k].second, uu);
      sink += mm.w[0];
    }
    t_mom = secs(a, Clock::now());
    if (sink == 12345.6789) out[0] = 0;  // keep the moments live
  }

  // ---------------- far + near: the sampled target leaves
  double t_far = 0.0, t_near = 0.0, n_targets = 0.0, far_pairs = 0.0;
  {
    const std::vector<char> tsel = pick_tiles(n_tgt);
    // near needs the sampled leaves and their 3x3 neighbourhoods
    std::vector<char> nsel((size_t)gL * gL, 0);
    for (int b = 0; b < gL * gL; ++b) {
      if (!tsel[(size_t)b]) continue;
      const int bi = b / gL, bj = b % gL;
      for (int qi = std::max(0, bi - 1); qi <= std::min(gL - 1, bi + 1); ++qi)
        for (int qj = std::max(0, bj - 1); qj <= std::min(gL - 1, bj + 1); ++qj)
          nsel[(size_t)(qi * gL + qj)] = 1;
    }
    imq::FastOperator op{imq::KernelParams(t), imq::ExpansionOrder(M)};
    std::vector<double> uu;
    std::vector<char> is_target;
    for (long long i = 0; i < n; ++i) {
      const int b = leaf[(size_t)i];
      if (!nsel[(size_t)b]) continue;
      op.points.push_back(pts[(size_t)i]);
      uu.push_back(u[i]);
      is_target.push_back(tsel[(size_t)b]);
    }
    op.L = L;
    op.tree = skeleton(sq, L);
    for (int j = 0; j < op.size(); ++j) {
      if (is_target[(size_t)j]) {  // targets are bucketed at every level
        n_targets += 1.0;
        for (int l = 1; l <= L - 1; ++l)
          op.tree.levels[l - 1].buckets[(size_t)op.tree.block_of(l, op.points[(size_t)j])].push_back(j);
      }
      op.tree.levels[L - 1].buckets[(size_t)op.tree.block_of(L, op.points[(size_t)j])].push_back(j);
    }
    // interaction lists (partition.cpp:56-72), stored source-major: slist[src]
    // holds the target blocks (those with sampled targets) whose list has src
    std::vector<std::pair<int, int>> work;  // (level, source block)
    for (int l = 1; l <= L; ++l) {
      imq::BlockTree::Level& lv = op.tree.levels[l - 1];
      const int g = lv.grid;
      for (int tb = 0; tb < g * g; ++tb) {
        bool has = false;
        for (int j : lv.buckets[(size_t)tb]) has = has || is_target[(size_t)j];
        if (!has) continue;
        const int i = tb / g, j = tb % g;
        const int lo_i = l == 1 ? 0 : std::max(0, 2 * (i / 2) - 2), hi_i = l == 1 ? g - 1 : std::min(g - 1, 2 * (i / 2) + 3);
        const int lo_j = l == 1 ? 0 : std::max(0, 2 * (j / 2) - 2), hi_j = l == 1 ? g - 1 : std::min(g - 1, 2 * (j / 2) + 3);
        for (int qi = lo_i; qi <= hi_i; ++qi)
          for (int qj = lo_j; qj <= hi_j; ++qj) {
            if (std::max(std::abs(qi - i), std::abs(qj - j)) < 2) continue;
            const int sb = qi * g + qj;
            // non-empty source blocks only (fastmv.cpp:207), counted on the full set
            const int shift = L - l;
            bool ne = false;
            for (int a = qi << shift; a < (qi + 1) << shift && !ne; ++a)
              for (int b = qj << shift; b < (qj + 1) << shift && !ne; ++b) ne = occ[(size_t)(a * gL + b)] > 0;
            if (!ne) continue;
            if (lv.slist[(size_t)sb].empty()) work.push_back({l, sb});
            lv.slist[(size_t)sb].push_back(tb);
          }
      }
    }
    op.dtab = imq::coeff_d_table(M);
    op.pn0.resize(op.order.K);
    imq::assoc_legendre_table(M, 0.0, 1.0, op.pn0.data());
    // apply_far reads only the targets' coordinates (no cache); level L's
    // buckets hold the near-field sources too, so the far work at level L is
    // restricted to the sampled targets by the target blocks' lists above
    // (their buckets are the sampled leaves, all of whose points are targets)
    imq::Moments dummy;
    dummy.v.assign(op.order.K, 1.0);
    dummy.w.assign(op.order.K, 1.0);
    // largest source blocks first (their target lists span the coarse levels):
    // dynamic scheduling then balances the threads
    std::vector<double> cost(work.size(), 0.0);
    for (size_t k = 0; k < work.size(); ++k)
      for (int tb : op.tree.levels[work[k].first - 1].slist[(size_t)work[k].second])
        cost[k] += (double)op.tree.levels[work[k].first - 1].buckets[(size_t)tb].size();
    {
      std::vector<size_t> ord(work.size());
      for (size_t k = 0; k < ord.size(); ++k) ord[k] = k;
      std::stable_sort(ord.begin(), ord.end(), [&](size_t x, size_t y) { return cost[x] > cost[y]; });
      std::vector<std::pair<int, int>> w2;
      for (size_t k : ord) {
        w2.push_back(work[k]);
        far_pairs += cost[k];
      }
      work.swap(w2);
    }
    const int nth = omp_get_max_threads();
    std::vector<std::vector<double>> bpriv((size_t)nth, std::vector<double>((size_t)op.size(), 0.0));
    const auto a = Clock::now();
#pragma omp parallel
    {
      std::vector<double>& b = bpriv[(size_t)omp_get_thread_num()];
#pragma omp for schedule(dynamic, 1)
      for (size_t k = 0; k < work.size(); ++k) imq::apply_far(op, work[k].first, work[k].second, dummy, b);
    }
    t_far = secs(a, Clock::now());
    // near field: near lists of the sampled leaves only (partition.cpp:75-83)
    for (int b = 0; b < gL * gL; ++b) {
      if (!tsel[(size_t)b]) continue;
      const int bi = b / gL, bj = b % gL;
      for (int qi = std::max(0, bi - 1); qi <= std::min(gL - 1, bi + 1); ++qi)
        for (int qj = std::max(0, bj - 1); qj <= std::min(gL - 1, bj + 1); ++qj)
          op.tree.near_lists[(size_t)b].push_back(qi * gL + qj);
    }
    std::vector<double> b((size_t)op.size(), 0.0);
    const auto c = Clock::now();
    imq::apply_near(op, uu, b);
    t_near = secs(c, Clock::now());
  }
  out[0] = t_mom;
  out[1] = t_far;
  out[2] = t_near;
  out[3] = mom_pts;
  out[4] = n_targets;
  out[5] = far_pairs;
  out[6] = t_mom * ((double)n / mom_pts) + (t_far + t_near) * ((double)n / n_targets);
  return 0;
}

}  // extern "C"
