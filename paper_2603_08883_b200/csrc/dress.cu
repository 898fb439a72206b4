// dress.cu — one exact dressing step on a canonically sorted device store.
//
// Restates dress_single (iqcc/dressing.hpp:197-220) without sorting the
// products.  For an entangler P with key-bit set Mset (its x and z bits at
// canonical positions b_1 < ... < b_m), the products T^P of the
// anticommuting terms T are ordered by a closed-form permutation of the
// (sorted) anticommuting subsequence a_1 < ... < a_A:
//
//   rank(T^P) = C(T) + sum_l  [bit_{b_l}(T)=0 ? +N1_l(T) : -N0_l(T)]
//
// where C(T) = #anticommuting terms before T, and N0_l/N1_l count the
// anticommuting terms in T's trie node at level b_l (terms sharing T's
// canonical prefix [0, b_l)) whose bit b_l is 0 / 1.  (Two keys compare in
// the opposite order after ^P iff their first differing position is in
// Mset.)  Node boundaries are where the LCP position between neighbouring
// physical terms drops below b_l, so everything reduces to forward/backward
// "last/next boundary" scans over the LCP array with per-level thresholds —
// the sortless idea of the paper's Appendix D (PAPER.md:630-676,
// iqcc/dressing.hpp:228-307) done as streaming scans instead of a heap
// k-way merge.  The survivors (all terms, c or c*cos) and the now-sorted
// products (+-fl(c*sin), sign from the phase) are then merged in one
// merge-path pass that adds the (at most one) partner coefficient, applies
// keep_term (iqcc/pauli.hpp:180-184) and compacts with a decoupled
// look-back — bit-identical to merge_sums (iqcc/pauli.hpp:383-415) because
// every output coefficient has at most two addends.
//
// Kernels (HBM-bound, integer/popcount work; no tensor cores):
//   k_classify      per term: LCP vs predecessor, anticommute bit (ballot),
//                   key bits at the m levels                       [reads keys]
//   k_tile_agg      per 2048-term tile: anticommute count + per-threshold
//                   first/last boundary                            [lcp, fmask]
//   k_group_agg / k_group_scan / k_tile_carry   carries across tiles
//   k_rank          in-tile scans -> product rank -> inv_perm[rank] = term
//   k_partition     merge-path split per output tile
//   k_merge         survivors (x) products merge, combine, drop, compact
#include <algorithm>
#include <cstdlib>
#include <climits>
#include <cstring>
#include <optional>
#include <stdexcept>

#include "engine.cuh"

namespace iqcc_b200 {

constexpr int TT = 256;  // threads per scan tile
constexpr int TI = 8;    // terms per thread
constexpr int TILE = TT * TI;
// tiles per carry group: 256 for small shards (latency), 1024 when that keeps
// the single-block group scan short
constexpr int kGroupSmall = 256, kGroupLarge = 1024;
constexpr int kMaxGroups = 4096;  // k_group_scan capacity: 2^28 terms per device shard

struct Thr {
  int t[kThrPerChunk];
  int n;     // thresholds in use (2 * levels)
  int nlev;  // levels in this chunk
};

// ---------------------------------------------------------------- classify
#ifndef IQCC_CLS_MINB
#define IQCC_CLS_MINB 4
#endif
#ifndef IQCC_MERGE_MINB
#define IQCC_MERGE_MINB 6
#endif
// resident 256-thread CTAs per SM the merge is compiled for: B = 4 (200-256
// qubits) rows are twice as wide, so fewer, fatter CTAs (no spills)
__host__ __device__ constexpr int merge_minb(int B, int NT) {
  return (B >= 4 ? 3 : IQCC_MERGE_MINB) * 256 / NT > 0 ? (B >= 4 ? 3 : IQCC_MERGE_MINB) * 256 / NT : 1;
}
#ifndef IQCC_RANK_MINB
#define IQCC_RANK_MINB 5
#endif
// Output slots.  Every present survivor and every product owns an output
// slot ("pmask" / "qmask" bits) unless a compress whose cut is at least theta
// follows the step (theta = eps: known; theta just under the previous cut:
// speculated, verified after the merge by counting the slotted terms with
// |c| >= theta) and its value cannot reach theta:
//  * a commuting survivor keeps its value c and never meets a product (the
//    partner of a product T^P anticommutes with P like T): slot iff |c| >= thc;
//  * an anticommuting survivor always keeps its slot (ths = 0), so a partner
//    pair's sum always has a slot;
//  * a product without a partner keeps fl(c*sin): slot iff |c*sin| >= thq.
// With thc = thq = theta every term of the dressed sum with |c| >= theta has a
// slot; terms without one are below theta.  theta = 0: every term has a slot.
struct SlotRule {
  double cs, sn;
  double thc, ths, thq;  // commuting survivor / anticommuting survivor / product
  // the derivative of a dressing (dress_derivative, iqcc/optimizer.hpp:31-48)
  // keeps only the anticommuting part: commuting survivors and the identity
  // get no slot
  int anti_only;
};

__host__ __device__ inline SlotRule make_slot_rule(double cs, double sn, double theta) {
  return SlotRule{cs, sn, theta, 0.0, theta, 0};
}

__device__ __forceinline__ bool survivor_slot(const SlotRule& r, bool present, bool id, bool anti,
                                              double c) {
  if (!present) return false;
  if (id) return !r.anti_only;
  return anti ? (r.ths == 0.0 || fabs(__dmul_rn(c, r.cs)) >= r.ths) : (!r.anti_only && fabs(c) >= r.thc);
}
__device__ __forceinline__ bool product_slot(const SlotRule& r, bool anti_present, double c) {
  if (!anti_present) return false;
  return r.thq == 0.0 || fabs(__dmul_rn(c, r.sn)) >= r.thq;
}

template <int B, int IT>
__global__ void __launch_bounds__(256, B >= 4 ? 2 : IQCC_CLS_MINB) k_classify(const ull* __restrict__ keys,
                                                  const double* __restrict__ coef, Filter filt,
                                                  size_t M, Key<B> P, short* __restrict__ lcp,
                                                  unsigned* __restrict__ fmask,
                                                  unsigned* __restrict__ pmask, SlotRule rule,
                                                  unsigned* __restrict__ qmask) {
  const int lane = threadIdx.x & 31;
  const size_t base = blockIdx.x * (size_t)(256 * IT);
  Key<B> k[IT], pk[IT];
  double c[IT];
#pragma unroll
  for (int j = 0; j < IT; ++j) {  // issue every load first
    const size_t i = base + (size_t)j * 256 + threadIdx.x;
    if (i < M) {
      k[j] = load_key<B>(keys, i);
      c[j] = __ldg(coef + i);
    }
    if (lane == 0 && i > 0 && i - 1 < M) pk[j] = load_key<B>(keys, i - 1);
  }
#pragma unroll
  for (int j = 0; j < IT; ++j) {
    const size_t i = base + (size_t)j * 256 + threadIdx.x;
#pragma unroll
    for (int w = 0; w < 2 * B; ++w) {
      const ull up = __shfl_up_sync(0xffffffffu, k[j].w[w], 1);
      if (lane > 0) pk[j].w[w] = up;
    }
    bool f = false, sl = false, qs = false;
    if (i < M) {
      lcp[i] = (short)(i > 0 ? key_lcp<B>(pk[j], k[j]) : -1);
      // dead slots and terms dropped by a pending compress filter are absent:
      // they emit nothing and generate no product
      const bool id = i == 0 && key_is_identity<B>(k[j]);
      const bool pr = filter_keep(filt, i, c[j], id);
      f = pr && anticommutes<B>(k[j], P);
      sl = survivor_slot(rule, pr, id, f, c[j]);
      qs = product_slot(rule, f, c[j]);
    }
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    const unsigned pal = __ballot_sync(0xffffffffu, sl);
    const unsigned qal = __ballot_sync(0xffffffffu, qs);
    const size_t i0 = i - lane;
    if (lane == 0 && i0 < M) {
      fmask[i0 >> 5] = bal;
      pmask[i0 >> 5] = pal;
      qmask[i0 >> 5] = qal;
    }
  }
}

// ------------------------------------------------- popcount prefix (pmask)
constexpr int PW = 1024;  // words per block
__global__ void __launch_bounds__(256) k_popc_blocks(const unsigned* __restrict__ words, size_t W,
                                                     unsigned* __restrict__ bsum) {
  __shared__ unsigned sm[256 / 32 + 2];
  const size_t w0 = blockIdx.x * (size_t)PW + threadIdx.x * 4;
  unsigned c = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (w0 + k < W) c += __popc(words[w0 + k]);
  unsigned tot;
  block_exclusive<256>(c, 0u, OpAdd(), sm, &tot);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

// in-place exclusive scan of nb block counts; `base` (optional, device)
// offsets the prefix and the total (a chunk continuing the previous one)
__global__ void __launch_bounds__(1024) k_scan_blocks(unsigned* __restrict__ bsum, size_t nb,
                                                      unsigned* total, const unsigned* base = nullptr) {
  __shared__ unsigned sm[1024 / 32 + 2];
  const size_t per = (nb + 1023) / 1024;
  const size_t lo = threadIdx.x * per, hi = min(nb, lo + per);
  const unsigned b0 = base ? *base : 0u;
  unsigned c = 0;
  for (size_t k = lo; k < hi; ++k) c += bsum[k];
  unsigned tot;
  unsigned run = block_exclusive<1024>(c, 0u, OpAdd(), sm, &tot) + b0;
  tot += b0;
  for (size_t k = lo; k < hi; ++k) {
    const unsigned v = bsum[k];
    bsum[k] = run;
    run += v;
  }
  if (threadIdx.x == 0) *total = tot;
}

__global__ void __launch_bounds__(256) k_popc_prefix(const unsigned* __restrict__ words, size_t W,
                                                     const unsigned* __restrict__ bpfx,
                                                     unsigned* __restrict__ pre) {
  __shared__ unsigned sm[256 / 32 + 2];
  const size_t w0 = blockIdx.x * (size_t)PW + threadIdx.x * 4;
  unsigned c[4], t = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    c[k] = w0 + k < W ? __popc(words[w0 + k]) : 0u;
    t += c[k];
  }
  unsigned run = block_exclusive<256>(t, 0u, OpAdd(), sm, (unsigned*)nullptr) + bpfx[blockIdx.x];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (w0 + k < W) pre[w0 + k] = run;
    run += c[k];
  }
}

/// # present terms before index a.
__device__ __forceinline__ size_t present_before(const unsigned* __restrict__ pmask,
                                                 const unsigned* __restrict__ pre, size_t W,
                                                 unsigned total, size_t a) {
  const size_t w = a >> 5;
  if (w >= W) return total;
  return (size_t)pre[w] + __popc(pmask[w] & ((1u << (a & 31)) - 1u));
}

// ---------------------------------------------------------- carry scans
// One warp per threshold (blockDim = 32 * nthr): the thresholds' scans run
// side by side instead of one after another behind block barriers, so the
// carry phase costs a few microseconds of latency per launch at any shard
// size.  Tile counts and their prefix are computed once per block into
// shared memory.  Values are relative to the group start (group level) or
// global (carry level), as the rank kernels expect.

// tile-count exclusive prefix of the block's group (relative), by warp 0
template <int GROUP>
__device__ __forceinline__ int group_tile_prefix(const int* __restrict__ tile_cnt, size_t g0,
                                                 size_t nt, int* s_pfx) {
  __shared__ int s_total;
  constexpr int TPL = GROUP / 32;  // tiles per lane in a group
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int run = 0;
#pragma unroll 8
    for (int i = 0; i < TPL; ++i) {
      const int t = i * 32 + lane;
      const int c = t < (int)nt ? tile_cnt[g0 + t] : 0;
      const int inc = warp_inclusive(c, OpAdd());
      s_pfx[t] = run + inc - c;
      run += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) s_total = run;
  }
  __syncthreads();
  return s_total;
}

template <int GROUP>
__global__ void __launch_bounds__(512) k_group_agg(const int* __restrict__ tile_cnt,
                                                   const int* __restrict__ fwd_agg,
                                                   const int* __restrict__ bwd_agg, size_t ntiles,
                                                   int nthr, long long* __restrict__ g_cnt,
                                                   long long* __restrict__ g_fwd,
                                                   long long* __restrict__ g_bwd) {
  __shared__ int s_pfx[GROUP];
  const size_t g0 = blockIdx.x * (size_t)GROUP;
  const size_t nt = min((size_t)GROUP, ntiles - g0);
  constexpr int TPL = GROUP / 32;
  const int total = group_tile_prefix<GROUP>(tile_cnt, g0, nt, s_pfx);
  const int j = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (j >= nthr) return;
  int f = -1, b = INT_MAX;
#pragma unroll 8
  for (int i = 0; i < TPL; ++i) {
    const int t = i * 32 + lane;
    if (t < (int)nt) {
      const int fv = fwd_agg[(g0 + t) * kThrPerChunk + j], bv = bwd_agg[(g0 + t) * kThrPerChunk + j];
      if (fv >= 0) f = max(f, fv + s_pfx[t]);
      if (bv >= 0) b = min(b, bv + s_pfx[t]);
    }
  }
  f = __reduce_max_sync(0xffffffffu, f);
  b = __reduce_min_sync(0xffffffffu, b);
  if (lane == 0) {
    g_fwd[blockIdx.x * kThrPerChunk + j] = f;
    g_bwd[blockIdx.x * kThrPerChunk + j] = b == INT_MAX ? LLONG_MAX : (long long)b;
    if (j == 0) g_cnt[blockIdx.x] = total;
  }
}

// Single block over groups (<= kMaxGroups groups = 2^28 terms).
__global__ void __launch_bounds__(512) k_group_scan(size_t ngroups, int nthr,
                                                    long long* __restrict__ g_cnt,
                                                    long long* __restrict__ g_fwd,
                                                    long long* __restrict__ g_bwd,
                                                    long long* __restrict__ a_total) {
  __shared__ long long s_pfx[kMaxGroups];
  __shared__ long long s_total;
  const int ng = (int)ngroups;
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    long long run = 0;
#pragma unroll 8
    for (int i = 0; i * 32 < ng; ++i) {
      const int g = i * 32 + lane;
      const long long c = g < ng ? g_cnt[g] : 0;
      const long long inc = warp_inclusive(c, OpAdd());
      if (g < ng) s_pfx[g] = run + inc - c;
      run += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) s_total = run;
  }
  __syncthreads();
  const int j = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (j < nthr) {
    // forward: exclusive max over the groups before (carry into the group)
    long long run = -1;
#pragma unroll 8
    for (int i = 0; i * 32 < ng; ++i) {
      const int g = i * 32 + lane;
      long long f = -1;
      if (g < ng) {
        const long long fv = g_fwd[g * kThrPerChunk + j];
        if (fv >= 0) f = fv + s_pfx[g];
      }
      const long long inc = warp_inclusive(f, OpMax());
      long long ex = __shfl_up_sync(0xffffffffu, inc, 1);
      if (lane == 0) ex = -1;
      if (g < ng) g_fwd[g * kThrPerChunk + j] = max(run, ex);
      run = max(run, __shfl_sync(0xffffffffu, inc, 31));
    }
    // backward: exclusive min over the groups after
    run = LLONG_MAX;
    const int nchunk = (ng + 31) / 32;
#pragma unroll 8
    for (int i = nchunk - 1; i >= 0; --i) {
      const int g = i * 32 + lane;
      long long b = LLONG_MAX;
      if (g < ng) {
        const long long bv = g_bwd[g * kThrPerChunk + j];
        if (bv != LLONG_MAX) b = bv + s_pfx[g];
      }
      const long long inc = warp_inclusive_rev(b, OpMin());
      long long ex = __shfl_down_sync(0xffffffffu, inc, 1);
      if (lane == 31) ex = LLONG_MAX;
      if (g < ng) g_bwd[g * kThrPerChunk + j] = min(run, ex);
      run = min(run, __shfl_sync(0xffffffffu, inc, 0));
    }
  }
  __syncthreads();
  for (int g = threadIdx.x; g < ng; g += blockDim.x) g_cnt[g] = s_pfx[g];  // group exclusive prefix
  if (threadIdx.x == 0) *a_total = s_total;
}

template <int GROUP>
__global__ void __launch_bounds__(512) k_tile_carry(const int* __restrict__ tile_cnt,
                                                    const int* __restrict__ fwd_agg,
                                                    const int* __restrict__ bwd_agg,
                                                    size_t ntiles, int nthr,
                                                    const long long* __restrict__ g_pfx,
                                                    const long long* __restrict__ g_fwd,
                                                    const long long* __restrict__ g_bwd,
                                                    const long long* __restrict__ a_total,
                                                    int* __restrict__ tile_pfx,
                                                    int* __restrict__ fwd_carry,
                                                    int* __restrict__ bwd_carry) {
  __shared__ int s_pfx[GROUP];
  const size_t g0 = blockIdx.x * (size_t)GROUP;
  const size_t nt = min((size_t)GROUP, ntiles - g0);
  constexpr int TPL = GROUP / 32;
  group_tile_prefix<GROUP>(tile_cnt, g0, nt, s_pfx);
  const long long gp = g_pfx[blockIdx.x];
  for (int t = threadIdx.x; t < (int)nt; t += blockDim.x) tile_pfx[g0 + t] = (int)(gp + s_pfx[t]);
  const int j = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (j >= nthr) return;
  const long long A = *a_total;
  long long run = g_fwd[blockIdx.x * kThrPerChunk + j];  // carry into the group
#pragma unroll 8
  for (int i = 0; i < TPL; ++i) {
    const int t = i * 32 + lane;
    long long f = -1;
    if (t < (int)nt) {
      const int fv = fwd_agg[(g0 + t) * kThrPerChunk + j];
      if (fv >= 0) f = gp + s_pfx[t] + fv;
    }
    const long long inc = warp_inclusive(f, OpMax());
    long long ex = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 0) ex = -1;
    if (t < (int)nt) fwd_carry[(g0 + t) * kThrPerChunk + j] = (int)max(run, ex);
    run = max(run, __shfl_sync(0xffffffffu, inc, 31));
  }
  run = g_bwd[blockIdx.x * kThrPerChunk + j];  // first boundary after the group
#pragma unroll 8
  for (int i = TPL - 1; i >= 0; --i) {
    const int t = i * 32 + lane;
    long long b = LLONG_MAX;
    if (t < (int)nt) {
      const int bv = bwd_agg[(g0 + t) * kThrPerChunk + j];
      if (bv >= 0) b = gp + s_pfx[t] + bv;
    }
    const long long inc = warp_inclusive_rev(b, OpMin());
    long long ex = __shfl_down_sync(0xffffffffu, inc, 1);
    if (lane == 31) ex = LLONG_MAX;
    const long long be = min(run, ex);
    if (t < (int)nt) bwd_carry[(g0 + t) * kThrPerChunk + j] = (int)(be == LLONG_MAX ? A : be);
    run = min(run, __shfl_sync(0xffffffffu, inc, 0));
  }
}

// ------------------------------------------------- warp-tile rank kernels
// One warp owns a tile of WT = 32*WI consecutive terms (lane l: terms
// [WI*l, WI*l+WI)); all scans are warp shuffles, no shared memory or block
// barriers.  NTHR thresholds per chunk (rounded up to a multiple of 4).
#ifndef IQCC_WI
#define IQCC_WI 8
#endif
constexpr int WI = IQCC_WI;  // terms per lane
static_assert(WI % 8 == 0 && WI <= 32, "lcp rows load as int4 (8 shorts)");
constexpr int WT = 32 * WI;

struct WarpItems {
  int l[WI];
  unsigned bits;
};

__device__ __forceinline__ WarpItems load_witems(const short* __restrict__ lcp,
                                                 const unsigned* __restrict__ fmask, size_t M,
                                                 size_t first) {
  WarpItems it;
  if (first + WI <= M) {
    const int4* p = reinterpret_cast<const int4*>(lcp + first);
#pragma unroll
    for (int h = 0; h < WI / 8; ++h) {
      const int4 v = __ldg(p + h);
      const short* s = reinterpret_cast<const short*>(&v);
#pragma unroll
      for (int k = 0; k < 8; ++k) it.l[8 * h + k] = s[k];
    }
  } else {
#pragma unroll
    for (int k = 0; k < WI; ++k) it.l[k] = first + k < M ? (int)lcp[first + k] : INT_MAX;
  }
  it.bits = fmask && first < M ? (fmask[first >> 5] >> (first & 31)) & ((1u << WI) - 1u) : 0u;
  return it;
}

/// Present / anticommuting bits from the merge's next-step metadata (the
/// classify pass of a dress_sequence step): present = filter_keep (dead
/// slots and the pending compress filter are absent), anticommuting from
/// the merge's bits.
struct MaskArgs {
  const double* coef;
  const unsigned* amask;
  const ull* keys;
  int W;  // key words (identity check of slot 0)
  Filter filt;
  SlotRule rule;
  unsigned* fmask;  // out: present and anticommuting
  unsigned* pmask;  // out: survivor owns an output slot
  unsigned* qmask;  // out: its product owns an output slot
};

__device__ __forceinline__ unsigned lane_masks(const MaskArgs& ma, size_t M, size_t first, int lane) {
  unsigned pb = 0, fb = 0, qb = 0;
  if (first < M) {
    const unsigned aw = (ma.amask[first >> 5] >> (first & 31)) & ((1u << WI) - 1u);
    bool id0 = false;
    if (first == 0) {
      id0 = true;
      for (int w = 0; w < ma.W; ++w) id0 = id0 && ma.keys[w] == 0ull;
    }
#pragma unroll
    for (int k = 0; k < WI; ++k) {
      const size_t i = first + k;
      if (i < M) {
        const double c = __ldg(ma.coef + i);
        const bool id = k == 0 && id0;
        const bool pr = filter_keep(ma.filt, i, c, id);
        const bool an = pr && ((aw >> k) & 1u);
        pb |= (unsigned)survivor_slot(ma.rule, pr, id, an, c) << k;
        fb |= (unsigned)an << k;
        qb |= (unsigned)product_slot(ma.rule, an, c) << k;
      }
    }
  }
  // lanes 4j..4j+3 (WI = 8) share one 32-bit mask word
  constexpr int LPW = 32 / WI;
  const int sh = WI * (lane % LPW);
  unsigned xp = pb << sh, xf = fb << sh, xq = qb << sh;
#pragma unroll
  for (int o = 1; o < LPW; o <<= 1) {
    xp |= __shfl_xor_sync(0xffffffffu, xp, o);
    xf |= __shfl_xor_sync(0xffffffffu, xf, o);
    xq |= __shfl_xor_sync(0xffffffffu, xq, o);
  }
  if (lane % LPW == 0 && first < M) {
    ma.pmask[first >> 5] = xp;
    ma.fmask[first >> 5] = xf;
    ma.qmask[first >> 5] = xq;
  }
  return fb;
}

template <int NTHR, bool MASKS>
__global__ void __launch_bounds__(256) k_tile_agg_w(const short* __restrict__ lcp,
                                                    const unsigned* __restrict__ fmask, size_t M,
                                                    size_t ntiles, Thr thr,
                                                    int* __restrict__ tile_cnt,
                                                    int* __restrict__ fwd_agg,
                                                    int* __restrict__ bwd_agg, MaskArgs ma) {
  const size_t wt = blockIdx.x * (size_t)8 + (threadIdx.x >> 5);
  if (wt >= ntiles) return;
  const int lane = threadIdx.x & 31;
  const size_t first = wt * WT + (size_t)lane * WI;
  WarpItems it = load_witems(lcp, MASKS ? nullptr : fmask, M, first);
  if (MASKS) it.bits = lane_masks(ma, M, first, lane);
  const int cnt = __popc(it.bits);
  const int inc = warp_inclusive(cnt, OpAdd());
  const int cl = inc - cnt;
  int lmax = INT_MIN;
#pragma unroll
  for (int k = 0; k < WI; ++k) lmax = max(lmax, it.l[k]);
  lmax = __reduce_max_sync(0xffffffffu, lmax);
  int lmin = INT_MAX;
#pragma unroll
  for (int k = 0; k < WI; ++k) lmin = min(lmin, it.l[k]);
  lmin = __reduce_min_sync(0xffffffffu, lmin);
  const int c_last = __shfl_sync(0xffffffffu, inc, 31) - (int)(__shfl_sync(0xffffffffu, it.bits, 31) >> (WI - 1));
#pragma unroll
  for (int j = 0; j < NTHR; ++j) {
    const int T = thr.t[j];
    int fa = -1, ba = INT_MAX;
    if (lmax <= T) {  // every term is a boundary (warp-uniform fast path)
      fa = c_last;
      ba = 0;
    } else if (T < lmin) {  // no boundary in the tile: fa = -1, ba = none
    } else {
#pragma unroll
      for (int k = 0; k < WI; ++k)
        if (it.l[k] <= T) fa = cl + __popc(it.bits & ((1u << k) - 1u));
#pragma unroll
      for (int k = WI - 1; k >= 0; --k)
        if (it.l[k] <= T) ba = cl + __popc(it.bits & ((1u << k) - 1u));
      fa = __reduce_max_sync(0xffffffffu, fa);
      ba = __reduce_min_sync(0xffffffffu, ba);
    }
    if (lane == 0) {
      fwd_agg[wt * kThrPerChunk + j] = fa;
      bwd_agg[wt * kThrPerChunk + j] = ba == INT_MAX ? -1 : ba;
    }
  }
  if (lane == 31) tile_cnt[wt] = inc;
}

// A term's side of the split at level l need not be stored: inside its node
// a split boundary (lcp == b_l) precedes the term iff its bit b_l is 1 and
// the node's 0-child is non-empty, i.e. iff D = st[le] - st[lt] > 0 in the
// forward scan.  When the bit is 1 but the 0-child is empty both formulas
// give 0, so  delta_l = D > 0 ? -D : (bwd[lt] - bwd[le]).
template <int NTHR, bool FINAL>
__global__ void __launch_bounds__(256, IQCC_RANK_MINB) k_rank_w(const short* __restrict__ lcp,
                                                const unsigned* __restrict__ fmask, size_t M,
                                                size_t ntiles, Thr thr,
                                                const int* __restrict__ tile_pfx,
                                                const int* __restrict__ fwd_carry,
                                                const int* __restrict__ bwd_carry,
                                                int* __restrict__ rdelta, int has_rdelta,
                                                unsigned* __restrict__ inv_perm,
                                                const long long* __restrict__ a_total,
                                                ull* __restrict__ dbg,
                                                const unsigned* __restrict__ qmask,
                                                unsigned char* __restrict__ qflag) {
  const size_t wt = blockIdx.x * (size_t)8 + (threadIdx.x >> 5);
  if (wt >= ntiles) return;
  const int lane = threadIdx.x & 31;
  const size_t first = wt * WT + (size_t)lane * WI;
  const WarpItems it = load_witems(lcp, fmask, M, first);
  const int cnt = __popc(it.bits);
  const int inc = warp_inclusive(cnt, OpAdd());
  const int cl = inc - cnt + tile_pfx[wt];
  // C(k) = anticommuting terms before item k (recomputed, not stored)
  auto Cof = [&](int k) { return cl + __popc(it.bits & ((1u << k) - 1u)); };
  int delta[WI];
#pragma unroll
  for (int k = 0; k < WI; ++k) delta[k] = 0;
  // a threshold below every LCP of the warp tile has no boundary in it: its
  // scans reduce to the carries (warp-uniform skip; common for shallow
  // levels inside runs of equal x planes)
  int lmin = INT_MAX;
#pragma unroll
  for (int k = 0; k < WI; ++k) lmin = min(lmin, it.l[k]);
  lmin = __reduce_min_sync(0xffffffffu, lmin);
  // forward scan of one threshold: last boundary at or before each item
  auto fwd = [&](int j) {
    const int fc = fwd_carry[wt * kThrPerChunk + j];
    if (thr.t[j] < lmin) return fc;
    int a = -1;
#pragma unroll
    for (int k = 0; k < WI; ++k)
      if (it.l[k] <= thr.t[j]) a = Cof(k);
    a = warp_inclusive(a, OpMax());
    int ex = __shfl_up_sync(0xffffffffu, a, 1);
    if (lane == 0) ex = -1;
    return max(ex, fc);
  };
  // backward scan: first boundary strictly after each item
  auto bwd = [&](int j) {
    const int bc = bwd_carry[wt * kThrPerChunk + j];
    if (thr.t[j] < lmin) return bc;
    int b = INT_MAX;
#pragma unroll
    for (int k = WI - 1; k >= 0; --k)
      if (it.l[k] <= thr.t[j]) b = Cof(k);
    b = warp_inclusive_rev(b, OpMin());
    int ex = __shfl_down_sync(0xffffffffu, b, 1);
    if (lane == 31) ex = INT_MAX;
    return min(ex, bc);
  };
  // levels one at a time (thresholds 2lv: node start, 2lv+1: child split):
  // only that level's scans and one bit per item ("D > 0 seen") stay live,
  // so the kernel fits 40 registers; a level without any boundary in the
  // tile (both thresholds below lmin) costs no compares
  const int nlev = thr.nlev;
#pragma unroll 1
  for (int lv = 0; lv < NTHR / 2; ++lv) {
    if (lv >= nlev) break;  // padded levels: D == 0 everywhere
    unsigned used = 0;
    int a = fwd(2 * lv), b = fwd(2 * lv + 1);
    const bool flat = thr.t[2 * lv + 1] < lmin;
    if (flat) {
      const int D = b - a;
      if (D > 0) {
#pragma unroll
        for (int k = 0; k < WI; ++k)
          if ((it.bits >> k) & 1u) delta[k] -= D;
        used = it.bits;
      }
    } else {
#pragma unroll
      for (int k = 0; k < WI; ++k) {
        if (it.l[k] <= thr.t[2 * lv]) a = Cof(k);
        if (it.l[k] <= thr.t[2 * lv + 1]) b = Cof(k);
        const int D = b - a;
        if (((it.bits >> k) & 1u) && D > 0) {
          delta[k] -= D;
          used |= 1u << k;
        }
      }
    }
    a = bwd(2 * lv);
    b = bwd(2 * lv + 1);
    const unsigned rest = it.bits & ~used;
    if (flat) {
      const int E = a - b;
#pragma unroll
      for (int k = 0; k < WI; ++k)
        if ((rest >> k) & 1u) delta[k] += E;
    } else {
#pragma unroll
      for (int k = WI - 1; k >= 0; --k) {
        if ((rest >> k) & 1u) delta[k] += a - b;
        if (it.l[k] <= thr.t[2 * lv]) a = Cof(k);
        if (it.l[k] <= thr.t[2 * lv + 1]) b = Cof(k);
      }
    }
  }
  const unsigned qm = FINAL && qflag && first < M ? (qmask[first >> 5] >> (first & 31)) : 0u;
#pragma unroll
  for (int k = 0; k < WI; ++k) {
    if (!((it.bits >> k) & 1u)) continue;
    const size_t g = first + k;
    const int d = delta[k] + (has_rdelta ? rdelta[g] : 0);
    const int Ck = Cof(k);
    if (FINAL) {
      if (dbg_ok(dbg, 1, (ull)(long long)(Ck + d), (ull)*a_total)) {
        inv_perm[Ck + d] = (unsigned)g;
        if (qflag) qflag[Ck + d] = (unsigned char)((qm >> k) & 1u);
      }
    } else {
      rdelta[g] = d;
    }
  }
}

/// Product slot flags (one byte per product, rank order) -> bit words.
__global__ void k_pack_flags(const unsigned char* __restrict__ flag, size_t A,
                             unsigned* __restrict__ bits) {
  // one word per thread from two 16-byte loads (flag bytes are 0 or 1; the
  // buffer is padded past A, bits past A are masked off)
  const size_t w = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (w * 32 >= A) return;
  const uint4* p = reinterpret_cast<const uint4*>(flag + w * 32);
  const uint4 a = __ldg(p), b = __ldg(p + 1);
  const unsigned q[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  unsigned x = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const unsigned v = q[k] & 0x01010101u;  // bytes -> bits 0, 8, 16, 24
    x |= ((v | (v >> 7) | (v >> 14) | (v >> 21)) & 0xFu) << (4 * k);
  }
  const size_t n = A - w * 32;
  bits[w] = n >= 32 ? x : x & ((1u << n) - 1u);
}

// Debug: inv_perm must be a bijection onto the present anticommuting terms.
__global__ void k_check_perm(const unsigned* __restrict__ inv_perm, size_t A, size_t M,
                             const unsigned* __restrict__ fmask, unsigned* __restrict__ seen,
                             ull* __restrict__ dbg) {
  const size_t r = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (r >= A) return;
  const unsigned g = inv_perm[r];
  if (!dbg_ok(dbg, 10, g, M)) return;
  if (!((fmask[g >> 5] >> (g & 31)) & 1u)) {
    dbg_ok(dbg, 11, r, 0);
    return;
  }
  if (atomicAdd(seen + g, 1u) != 0) dbg_ok(dbg, 12, r, 0);
}

// ------------------------------------------------------------- partition
/// Product j in sorted order: gathered through inv_perm (local products) or
/// read from a materialized buffer q_keys (products received from a peer).
template <int B>
__device__ __forceinline__ Key<B> q_key(const ull* __restrict__ keys,
                                        const unsigned* __restrict__ inv_perm,
                                        const ull* __restrict__ q_keys, size_t j, const Key<B>& P) {
  if (q_keys) return load_key<B>(q_keys, j);
  return key_xor<B>(load_key<B>(keys, inv_perm[j]), P);
}

constexpr int kPartShift = 5;  // coarse merge-path splits every 32 output tiles

template <int B>
__global__ void k_partition(const ull* __restrict__ keys, const unsigned* __restrict__ inv_perm,
                            const ull* __restrict__ q_keys,
                            size_t nS, size_t nQ, Key<B> P, size_t tile_items, size_t ntiles,
                            ull* __restrict__ part_a, ull* __restrict__ part_b,
                            ull* __restrict__ part_o, const unsigned* __restrict__ pmask,
                            const unsigned* __restrict__ ppre, size_t W,
                            const unsigned* __restrict__ ptotal, const unsigned* __restrict__ qbits,
                            const unsigned* __restrict__ qpre, size_t Wq,
                            const unsigned* __restrict__ qtotal, int coarse_shift,
                            ull* __restrict__ raw_a, size_t a_base = 0, size_t b_base = 0) {
  // two passes: coarse_shift > 0 searches every 2^shift-th boundary over the
  // whole range and records the raw split; coarse_shift == 0 searches every
  // boundary inside the window between its two coarse neighbours.  A chunk
  // of a chunked merge is the sub-merge of S[a_base, a_base + nS) and
  // Q[b_base, b_base + nQ) (outputs absolute)
  const size_t t = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) << coarse_shift;
  if (t > ntiles) return;
  const size_t d = min(t * tile_items, nS + nQ);
  size_t lo = d > nQ ? d - nQ : 0, hi = min(d, nS);
  if (coarse_shift == 0 && raw_a) {  // the raw split is monotone in the diagonal
    const size_t c0 = t >> kPartShift;
    lo = max(lo, (size_t)raw_a[c0]);
    if (((c0 + 1) << kPartShift) <= ntiles) hi = min(hi, (size_t)raw_a[c0 + 1]);
  }
  while (lo < hi) {
    size_t mid = (lo + hi) >> 1;
    if (key_cmp<B>(load_key<B>(keys, a_base + mid),
                   q_key<B>(keys, inv_perm, q_keys, b_base + d - 1 - mid, P)) <= 0)
      lo = mid + 1;
    else
      hi = mid;
  }
  size_t a = lo, b = d - lo;
  if (coarse_shift) {
    raw_a[t >> coarse_shift] = a;
    return;
  }
  // never split a run of equal survivors (live + dead slot) from its product
  if (b < nQ) {
    const Key<B> q = q_key<B>(keys, inv_perm, q_keys, b_base + b, P);
    while (a > 0 && key_cmp<B>(load_key<B>(keys, a_base + a - 1), q) == 0) --a;
  }
  a += a_base;
  b += b_base;
  part_a[t] = a;
  part_b[t] = b;
  // output slots before this tile: survivors and products that own a slot
  // (see SlotRule; with theta = 0 every present survivor and every product)
  part_o[t] = present_before(pmask, ppre, W, *ptotal, a) +
              (qbits ? present_before(qbits, qpre, Wq, *qtotal, b) : b);
}

/// Coarse merge-path splits (every 2^kPartShift-th tile boundary), one warp
/// per boundary with a 32-ary search: each round the lanes probe 32
/// positions at once, so a search over 1e8 survivors takes 6 dependent
/// probe rounds instead of 27 (the coarse pass is pure latency).
template <int B>
__global__ void k_partition_coarse(const ull* __restrict__ keys, const unsigned* __restrict__ inv_perm,
                                   const ull* __restrict__ q_keys, size_t nS, size_t nQ, Key<B> P,
                                   size_t tile_items, size_t ntiles, ull* __restrict__ raw_a,
                                   size_t a_base = 0, size_t b_base = 0) {
  const size_t c = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const size_t t = c << kPartShift;
  if (t > ntiles) return;  // warp-uniform
  const size_t d = min(t * tile_items, nS + nQ);
  size_t lo = d > nQ ? d - nQ : 0, hi = min(d, nS);
  // invariant: the split a is in [lo, hi]; pred(m) = key(m) <= qkey(d-1-m) holds below a
  while (hi > lo) {
    const size_t span = hi - lo;
    const size_t step = (span + 31) / 32;  // probe lo + step*(lane+1) - 1
    const size_t m = lo + step * (lane + 1) - 1;
    bool pr = true;
    if (m < hi)
      pr = key_cmp<B>(load_key<B>(keys, a_base + m), q_key<B>(keys, inv_perm, q_keys, b_base + d - 1 - m, P)) <= 0;
    const unsigned fails = __ballot_sync(0xffffffffu, !pr);
    if (fails == 0) {
      // every probe below hi held: the split lies past the last of them
      // (a tail shorter than `step` may remain unprobed)
      lo += step * min((size_t)32, span / step);
    } else {
      const int f = __ffs(fails) - 1;  // first probe where the predicate fails
      const size_t mf = lo + step * (f + 1) - 1;
      lo += step * f;  // probes < f held: the split is past them
      hi = mf;         // and at or before the failing probe
    }
  }
  if (lane == 0) raw_a[c] = lo;
}

template <int B>
__device__ __forceinline__ Key<B> sm_key(const ull* sk, int e) {
  Key<B> k;
#pragma unroll
  for (int w = 0; w < 2 * B; ++w) k.w[w] = sk[(size_t)e * 2 * B + w];
  return k;
}

// ----------------------------------------------------------------- merge
// One output tile per CTA (dynamic tile id for the look-back).  The
// survivor range S[a0,a1) is contiguous: it is staged into shared memory by
// the TMA engine (cp.async.bulk, one elected thread, completion on an
// mbarrier).  The product range Q[b0,b1) is a gather through inv_perm: each
// row/coefficient is fetched with cp.async (LDGSTS) so every thread keeps
// many requests in flight without staging through registers.  Outputs are
// written to a shared staging list in merged order and stored coalesced.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async8(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_init(unsigned long long* mb, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(mb)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* mb, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(mb)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* s, const void* g, unsigned bytes,
                                         unsigned long long* mb) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(s)),
      "l"(g), "r"(bytes), "r"(smem_u32(mb))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* mb, unsigned phase) {
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(mb)), "r"(phase)
        : "memory");
  }
}

template <int B, int NT, int IPT>
struct MergeCfg {
  static constexpr int TILE = NT * IPT;
  static constexpr int CAP = TILE + 8;  // tiles absorb short runs of equal survivors
  static constexpr size_t KEYB = (size_t)CAP * 16 * B;
  // one input stage: survivor rows [0,nS) then product rows [nS, nS+nQ);
  // S coefs [coff, coff+nS), Q coefs [nS+4, ...); then the tile's plan bit
  // words (pmask, fmask, product slots; BW words each) fetched with the rows
  static constexpr int BW = (CAP + 31) / 32 + 3;
  static constexpr size_t OFF_SBITS = KEYB + (size_t)(CAP + 4) * 8;
  static constexpr size_t STAGE = (OFF_SBITS + (size_t)3 * BW * 4 + 127) & ~(size_t)127;
  static constexpr size_t OFF_OUTV = 2 * STAGE;
  static constexpr size_t OFF_OUTE = OFF_OUTV + (size_t)CAP * 8;
  static constexpr size_t OFF_TA = (OFF_OUTE + (size_t)CAP * 2 + 15) & ~(size_t)15;
  static constexpr size_t OFF_PM = OFF_TA + (size_t)2 * NT * 4;  // present bits of S
  static constexpr int PMW = (CAP + 31) / 32;
  static constexpr size_t OFF_SM = OFF_PM + (size_t)PMW * 4;     // slot bits of S
  static constexpr size_t OFF_PP = OFF_SM + (size_t)PMW * 4;     // their prefix
  static constexpr size_t OFF_QM = OFF_PP + (size_t)PMW * 4;     // slot bits of Q
  static constexpr size_t OFF_QP = OFF_QM + (size_t)PMW * 4;     // their prefix
  static constexpr size_t OFF_AM = OFF_QP + (size_t)PMW * 4;     // anticommute bits of S
  static constexpr size_t OFF_HIST = (OFF_AM + (size_t)PMW * 4 + 15) & ~(size_t)15;
  static constexpr int HBINS = kHistBins + kSubBins;  // |c| histograms (u32, per CTA) for compress
  static constexpr size_t bytes(bool hist, int stages) {
    return OFF_HIST - (2 - stages) * STAGE + (hist ? HBINS * 4 : 0);
  }
};

// Staged key rows in shared memory: row-major (default; survivors land by
// one TMA bulk copy), or with IQCC_SPLIT_SMEM=1 split into 16-byte chunks
// (chunk h of element e at chunk index h*CAPR + e), which makes a warp's
// reads of consecutive elements bank-conflict free (row-major 32-byte rows
// are 2-way conflicted: 76% of the merge's excess shared wavefronts under
// ncu) but needs per-thread cp.async for the survivors: measured 1.6 ms per
// bench step slower (profiles/r2_summary.md), so row-major stays.
#ifndef IQCC_SPLIT_SMEM
#define IQCC_SPLIT_SMEM 0
#endif
template <int B, int CAPR>
__device__ __forceinline__ Key<B> sm_key16(const ull* sk, int e) {
  Key<B> k;
  const ulonglong2* p = reinterpret_cast<const ulonglong2*>(sk);
#pragma unroll
  for (int h = 0; h < B; ++h) {
    const ulonglong2 v = IQCC_SPLIT_SMEM ? p[h * CAPR + e] : p[(size_t)e * B + h];
    k.w[2 * h] = v.x;
    k.w[2 * h + 1] = v.y;
  }
  return k;
}
/// 16-byte chunk h of staged element e (see sm_key16).
template <int B, int CAPR>
__device__ __forceinline__ ull* sm_chunk(ull* sk, int e, int h) {
  return IQCC_SPLIT_SMEM ? sk + 2 * ((size_t)h * CAPR + e) : sk + (size_t)e * 2 * B + 2 * h;
}

struct MergeArgs {
  const ull* keys;
  const double* coef;
  Filter filt;
  const unsigned* inv_perm;
  const ull* q_keys;    // non-null: products already materialized (key ^ P, value)
  const double* q_vals;
  const ull* part_a;
  const ull* part_b;
  const ull* part_o;
  size_t ntiles;
  double cs, sn, drop, eps;
  ull* out_keys;
  double* out_coef;
  ull* counters;
  unsigned* hist;
  int want_hist;
  ull* dbg;
  // next-step metadata (nullptr: none): LCP with the predecessor slot and
  // anticommute bits against the next entangler pn
  short* out_lcp;
  unsigned* out_amask;
  ull pn[8];
  SlotRule rule;
  const unsigned* qbits;  // product slot bits in product order (nullptr: all)
  // the plan's per-slot bits of the store: survivor owns an output slot
  // (pmask) and present & anticommuting (fmask); a present survivor without
  // a slot commutes and is dropped by the compress, so it acts as absent
  const unsigned* pmask;
  const unsigned* fmask;
  double theta;           // count emitted non-identity |c| >= theta (0: off)
  int sub_b0;             // first exponent bin of the fine histogram (< 0: none)
};

/// Issue the loads of one tile into one stage: survivors by the TMA bulk
/// engine (thread 0, completion on *mb), products by per-thread cp.async
/// gathers (one commit group).
__device__ __forceinline__ void cp_async4(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(s)), "l"(g) : "memory");
}

/// Survivor rows [a0, a1) and their coefficients into a stage: split
/// 16-byte chunks by per-thread cp.async (IQCC_SPLIT_SMEM), else one TMA
/// bulk copy each (thread 0, completion on *mb).
template <int B, int NT, int CAPR>
__device__ __forceinline__ void stage_survivors(const MergeArgs& g, size_t a0, size_t a1, ull* sk, double* sc,
                                                unsigned long long* mb) {
  const int nS = (int)(a1 - a0);
  if (nS <= 0) return;
  const size_t c0 = a0 & ~(size_t)1, c1 = (a1 + 1) & ~(size_t)1;
  if (IQCC_SPLIT_SMEM) {
    for (int i = threadIdx.x; i < nS; i += NT) {
      const ull* gk = g.keys + (a0 + i) * 2 * B;
#pragma unroll
      for (int h = 0; h < B; ++h) cp_async16(sm_chunk<B, CAPR>(sk, i, h), gk + 2 * h);
    }
    for (int i = threadIdx.x; i < (int)((c1 - c0) >> 1); i += NT) cp_async16(sc + 2 * i, g.coef + c0 + 2 * i);
  } else if (threadIdx.x == 0) {
    const unsigned kb = (unsigned)nS * 16u * B;
    const unsigned cb = (unsigned)((c1 - c0) * 8);
    mbar_expect_tx(mb, kb + cb);
    bulk_g2s(sk, g.keys + a0 * 2 * B, kb, mb);
    bulk_g2s(sc, g.coef + c0, cb, mb);
  }
}

template <int B, int NT, int CAPR>
__device__ __forceinline__ void merge_issue(const MergeArgs& g, size_t tile, ull* sk, double* sc,
                                            unsigned long long* mb, unsigned* sbits = nullptr, int BW = 0) {
  const size_t a0 = g.part_a[tile], a1 = g.part_a[tile + 1];
  const size_t b0 = g.part_b[tile], b1 = g.part_b[tile + 1];
  const int nS = (int)(a1 - a0), nQ = (int)(b1 - b0);
  stage_survivors<B, NT, CAPR>(g, a0, a1, sk, sc, mb);
  const int qc0 = nS + 4;
  if (g.q_keys) {  // contiguous received products
    for (int j = threadIdx.x; j < nQ; j += NT) {
      const ull* gk = g.q_keys + (b0 + j) * 2 * B;
#pragma unroll
      for (int h = 0; h < B; ++h) cp_async16(sm_chunk<B, CAPR>(sk, nS + j, h), gk + 2 * h);
      cp_async8(sc + qc0 + j, g.q_vals + b0 + j);
    }
  } else {
    for (int j = threadIdx.x; j < nQ; j += NT) {
      const size_t src = __ldg(g.inv_perm + b0 + j);
      const ull* gk = g.keys + src * 2 * B;
#pragma unroll
      for (int h = 0; h < B; ++h) cp_async16(sm_chunk<B, CAPR>(sk, nS + j, h), gk + 2 * h);
      cp_async8(sc + qc0 + j, g.coef + src);
    }
  }
  if (sbits) {  // the tile's plan bit words ride along (no dependent load after the wait)
    const size_t pw0 = a0 >> 5, qw0 = b0 >> 5;
    const int npw = (int)(((a1 + 31) >> 5) - pw0) + 1, nqw = (int)(((b1 + 31) >> 5) - qw0) + 1;
    for (int w = threadIdx.x; w < npw; w += NT) {
      cp_async4(sbits + w, g.pmask + pw0 + w);
      cp_async4(sbits + BW + w, g.fmask + pw0 + w);
    }
    if (g.qbits)
      for (int w = threadIdx.x; w < nqw; w += NT) cp_async4(sbits + 2 * BW + w, g.qbits + qw0 + w);
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

// Output slot rule (no look-back needed): every present survivor and every
// product owns one slot, in merged order.  A survivor/product pair writes
// the combined value into the survivor's slot and a dead slot after it;
// a value failing keep_term leaves a dead slot.  So the tile's output
// offset is present_before(a0) + b0, known before the tile runs.
struct TileBounds {
  size_t a0, a1, b0, b1, o0, o1;
};
/// Plan bits of one tile staged in shared memory by the pipelined merge:
/// pm/fm hold pmask/fmask words from word pw0 on, qb the product slot words
/// from qw0 on.
struct StagedBits {
  const unsigned* pm;
  const unsigned* fm;
  const unsigned* qb;
  size_t pw0, qw0;
};

template <int B, int NT, int IPT>
__device__ __forceinline__ void merge_compute(const MergeArgs& g, size_t tile, const Key<B>& P,
                                              ull* sk, double* sc, unsigned char* smem_raw,
                                              int& n_eps, int& n_dead, int& n_coll, int& n_ge,
                                              const TileBounds* tbp = nullptr,
                                              const StagedBits* sb = nullptr) {
  using Cfg = MergeCfg<B, NT, IPT>;
  double* outv = reinterpret_cast<double*>(smem_raw + Cfg::OFF_OUTV);
  unsigned short* oute = reinterpret_cast<unsigned short*>(smem_raw + Cfg::OFF_OUTE);
  int* s_ta = reinterpret_cast<int*>(smem_raw + Cfg::OFF_TA);
  int* s_tb = s_ta + NT;
  unsigned* spm = reinterpret_cast<unsigned*>(smem_raw + Cfg::OFF_PM);
  unsigned* ssm = reinterpret_cast<unsigned*>(smem_raw + Cfg::OFF_SM);
  unsigned* spp = reinterpret_cast<unsigned*>(smem_raw + Cfg::OFF_PP);
  unsigned* sqm = reinterpret_cast<unsigned*>(smem_raw + Cfg::OFF_QM);
  unsigned* sqp = reinterpret_cast<unsigned*>(smem_raw + Cfg::OFF_QP);
  unsigned* sam = reinterpret_cast<unsigned*>(smem_raw + Cfg::OFF_AM);
  unsigned* shist = reinterpret_cast<unsigned*>(smem_raw + Cfg::OFF_HIST);
  const TileBounds tb = tbp ? *tbp
                            : TileBounds{g.part_a[tile], g.part_a[tile + 1], g.part_b[tile],
                                         g.part_b[tile + 1], g.part_o[tile], g.part_o[tile + 1]};
  const size_t a0 = tb.a0, a1 = tb.a1, b0 = tb.b0, b1 = tb.b1, o0 = tb.o0, o1 = tb.o1;
  const int nS = (int)(a1 - a0), nQ = (int)(b1 - b0), n = nS + nQ;
  const int nslots = (int)(o1 - o0);
  const int coff = (int)(a0 & 1);
  const int qc0 = nS + 4;
  // plan bits: global, or the tile's words staged in shared memory (indexed
  // through a base shifted by the first staged word)
  const unsigned* PMASK = sb ? sb->pm - sb->pw0 : g.pmask;
  const unsigned* FMASK = sb ? sb->fm - sb->pw0 : g.fmask;
  const unsigned* QBITS = g.qbits ? (sb ? sb->qb - sb->qw0 : g.qbits) : nullptr;

  // survivor bits from the plan: slot (pmask, also "present": see MergeArgs)
  // and present & anticommuting (fmask); slot bits of the products
  {
    auto bits_at = [&](const unsigned* m, size_t gb, int rem) {
      const unsigned sh = (unsigned)(gb & 31);
      unsigned x = m[gb >> 5] >> sh;
      if (sh) x |= m[(gb >> 5) + 1] << (32 - sh);
      return rem < 32 ? x & ((1u << rem) - 1u) : x;
    };
    for (int w = threadIdx.x; w < (nS + 31) >> 5; w += NT) {
      const size_t gb = a0 + (size_t)w * 32;
      const int rem = nS - w * 32;
      const unsigned sl = bits_at(PMASK, gb, rem);
      spm[w] = sl;
      ssm[w] = sl;
      sam[w] = bits_at(FMASK, gb, rem);
    }
    if (QBITS)
      for (int w = threadIdx.x; w < (nQ + 31) >> 5; w += NT) {
        const size_t gb = b0 + (size_t)w * 32;
        const unsigned sh = (unsigned)(gb & 31);
        unsigned x = QBITS[gb >> 5] >> sh;
        if (sh) x |= QBITS[(gb >> 5) + 1] << (32 - sh);
        const int rem = nQ - w * 32;
        if (rem < 32) x &= (1u << rem) - 1u;
        sqm[w] = x;
      }
  }
  // local products stay raw in shared memory (key = row ^ P on the fly);
  // received products arrive as final keys and values
  const bool qdirect = g.q_keys != nullptr;
  const Key<B> PX = qdirect ? Key<B>{} : P;
  auto qkey = [&](int j) { return key_xor<B>(sm_key16<B, Cfg::CAP>(sk, nS + j), PX); };
  auto qval = [&](int j, const Key<B>& kq) {
    if (qdirect) return sc[qc0 + j];
    const double pr = __dmul_rn(sc[qc0 + j], g.sn);
    return product_phase<B>(key_xor<B>(kq, P), P) == 1 ? pr : -pr;
  };
  {  // per-thread merge-path split (runs of equal survivors stay with their product)
    const int d = min((int)threadIdx.x * IPT, n);
    int lo = max(0, d - nQ), hi = min(d, nS);
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (key_cmp<B>(sm_key16<B, Cfg::CAP>(sk, mid), qkey(d - 1 - mid)) <= 0)
        lo = mid + 1;
      else
        hi = mid;
    }
    int a = lo;
    const int b = d - lo;
    if (b < nQ) {
      const Key<B> q = qkey(b);
      while (a > 0 && key_cmp<B>(sm_key16<B, Cfg::CAP>(sk, a - 1), q) == 0) --a;
    }
    s_ta[threadIdx.x] = a;
    s_tb[threadIdx.x] = b;
  }
  __syncthreads();
  if (threadIdx.x < 64) {  // exclusive prefixes of the slot-bit words (warp 0: S, warp 1: Q)
    const bool isq = threadIdx.x >= 32;
    if (!isq || g.qbits) {
      const unsigned* m = isq ? sqm : ssm;
      unsigned* pf = isq ? sqp : spp;
      const int nw = ((isq ? nQ : nS) + 31) >> 5;
      const int lane = threadIdx.x & 31;
      unsigned carry = 0;
      for (int w0 = 0; w0 < nw; w0 += 32) {
        const int w = w0 + lane;
        const unsigned c = w < nw ? __popc(m[w]) : 0u;
        const unsigned inc = warp_inclusive(c, OpAdd());
        if (w < nw) pf[w] = carry + inc - c;
        carry += __shfl_sync(0xffffffffu, inc, 31);
      }
    }
  }
  __syncthreads();
  const int ia0 = s_ta[threadIdx.x], ib0 = s_tb[threadIdx.x];
  const int ia1 = threadIdx.x + 1 < NT ? s_ta[threadIdx.x + 1] : nS;
  const int ib1 = threadIdx.x + 1 < NT ? s_tb[threadIdx.x + 1] : nQ;
  auto present = [&](int e) { return (spm[e >> 5] >> (e & 31)) & 1u; };
  auto sslot = [&](int e) { return (ssm[e >> 5] >> (e & 31)) & 1u; };
  auto qslot = [&](int j) { return g.qbits ? (sqm[j >> 5] >> (j & 31)) & 1u : 1u; };
  // slots before a position in a (prefixed) bit list of n entries
  auto before = [&](const unsigned* m, const unsigned* pf, int n, int x) -> int {
    if (n <= 0) return 0;
    const int w = min(x, n - 1) >> 5;
    const unsigned msk = x >= n ? (0xffffffffu >> (31 - ((n - 1) & 31))) : ((1u << (x & 31)) - 1u);
    return (int)(pf[w] + __popc(m[w] & msk));
  };
  int slot = before(ssm, spp, nS, ia0) + (g.qbits ? before(sqm, sqp, nQ, ib0) : ib0);

  // single walk; every slot value goes straight to the staging list
  {
    int i = ia0, j = ib0;
    Key<B> ks, kq;
    if (i < ia1) ks = sm_key16<B, Cfg::CAP>(sk, i);
    if (j < ib1) kq = qkey(j);
    auto put = [&](double v, int e) {
      if (dbg_ok(g.dbg, 2, (ull)slot, (ull)nslots)) {
        outv[slot] = v;
        oute[slot] = (unsigned short)e;
      }
      ++slot;
    };
#pragma unroll 1
    while (i < ia1 || j < ib1) {
      const int c = j >= ib1 ? -1 : (i >= ia1 ? 1 : key_cmp<B>(ks, kq));
      if (c <= 0) {
        const bool pres = present(i);
        const bool sl = sslot(i);
        const bool id = a0 + i == 0 && key_is_identity<B>(ks);
        double v = 0.0;
        if (pres) {
          const double cv = sc[coff + i];
          v = ((sam[i >> 5] >> (i & 31)) & 1u) ? __dmul_rn(cv, g.cs) : cv;
        }
        if (c == 0) {
          const double qv = qval(j, kq);
          const bool qs = qslot(j);
          if (pres) {
            ++n_coll;
            // the sum goes to the survivor's slot, else to the product's;
            // without either slot |sum| < theta (SlotRule)
            const double sum = __dadd_rn(v, qv);
            if (sl) {
              put(keep_term(sum, id, g.drop) ? sum : dead_value(), i);
              if (qs) put(dead_value(), nS + j);  // the product's slot
            } else if (qs) {
              put(keep_term(sum, id, g.drop) ? sum : dead_value(), nS + j);
            }
          } else if (qs) {
            put(keep_term(qv, b0 + j == 0 && key_is_identity<B>(kq), g.drop) ? qv : dead_value(), nS + j);
          }
        } else if (sl) {
          put(keep_term(v, id, g.drop) ? v : dead_value(), i);
        }
      } else if (qslot(j)) {
        // a dressing product is never the identity (T^P = 0 needs T = P,
        // which commutes); merge_sums' second operand may start with it
        const double qv = qval(j, kq);
        put(keep_term(qv, b0 + j == 0 && key_is_identity<B>(kq), g.drop) ? qv : dead_value(), nS + j);
      }
      if (c <= 0 && ++i < ia1) ks = sm_key16<B, Cfg::CAP>(sk, i);
      if (c >= 0 && ++j < ib1) kq = qkey(j);
    }
  }
  __syncthreads();
  const bool meta = g.out_lcp != nullptr;
  Key<B> PN;
#pragma unroll
  for (int w = 0; w < 2 * B; ++w) PN.w[w] = g.pn[w];
  for (int q0 = 0; q0 < nslots; q0 += NT) {  // block-uniform trip count
    const int q = q0 + (int)threadIdx.x;
    bool anti = false;
    if (q < nslots) {
      const int e = oute[q];
      const double v = outv[q];
      const Key<B> k = e < nS ? sm_key16<B, Cfg::CAP>(sk, e) : qkey(e - nS);
      store_key<B>(g.out_keys, o0 + q, k);
      g.out_coef[o0 + q] = v;
      if (is_dead(v)) {
        ++n_dead;
      } else if (g.want_hist) {
        const double a = fabs(v);
        const bool id = o0 + q == 0 && key_is_identity<B>(k);
        if (id || a >= g.eps) ++n_eps;
        if (!id && a >= g.eps) {
          const unsigned hb = hist_bin(a);
          atomicAdd(shist + hb, 1u);
          const unsigned sb = hb - (unsigned)g.sub_b0;
          if (sb < (unsigned)kSubWindow)
            atomicAdd(shist + kHistBins + sb * kSubBinsPer +
                          (unsigned)(((ull)__double_as_longlong(a) >> (52 - kSubBits)) & (kSubBinsPer - 1)),
                      1u);
        }
        if (!id && g.theta != 0.0 && a >= g.theta) ++n_ge;
      }
      if (meta) {
        short l = -1;  // tile-first slot: fixed up by k_meta_fix
        if (q > 0) {
          const int ep = oute[q - 1];
          l = (short)key_lcp<B>(ep < nS ? sm_key16<B, Cfg::CAP>(sk, ep) : qkey(ep - nS), k);
        }
        g.out_lcp[o0 + q] = l;
        anti = anticommutes<B>(k, PN);
      }
    }
    if (meta) {
      const unsigned bal = __ballot_sync(0xffffffffu, anti);
      if ((threadIdx.x & 31) == 0 && bal) {
        const size_t ob = o0 + q0 + (threadIdx.x & ~31u);
        const unsigned sh = (unsigned)(ob & 31);
        atomicOr(g.out_amask + (ob >> 5), bal << sh);
        if (sh) atomicOr(g.out_amask + (ob >> 5) + 1, bal >> (32 - sh));
      }
    }
  }
}

/// LCP of every tile's first output slot with its predecessor (the merge
/// only sees predecessors inside its own tile).
template <int B>
__global__ void k_meta_fix(const ull* __restrict__ keys, const ull* __restrict__ part_o, size_t ntiles,
                           short* __restrict__ lcp) {
  const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (t >= ntiles) return;
  const size_t Mout = part_o[ntiles];
  const size_t o = part_o[t];
  if (o == 0 || o >= Mout) return;
  lcp[o] = (short)key_lcp<B>(load_key<B>(keys, o - 1), load_key<B>(keys, o));
}

template <int B, int NT>
__device__ __forceinline__ void merge_flush(const MergeArgs& g, unsigned* shist, int n_eps,
                                            int n_dead, int n_coll, int n_ge, int* s_cnt) {
  n_dead = __reduce_add_sync(0xffffffffu, n_dead);
  n_eps = __reduce_add_sync(0xffffffffu, n_eps);
  n_coll = __reduce_add_sync(0xffffffffu, n_coll);
  n_ge = __reduce_add_sync(0xffffffffu, n_ge);
  if ((threadIdx.x & 31) == 0) {
    if (n_dead) atomicAdd(&s_cnt[0], n_dead);
    if (n_eps) atomicAdd(&s_cnt[1], n_eps);
    if (n_coll) atomicAdd(&s_cnt[2], n_coll);
    if (n_ge) atomicAdd(&s_cnt[3], n_ge);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_cnt[0]) atomicAdd(g.counters + 2, (ull)s_cnt[0]);
    if (s_cnt[1]) atomicAdd(g.counters + 1, (ull)s_cnt[1]);
    if (s_cnt[2]) atomicAdd(g.counters + 5, (ull)s_cnt[2]);
    if (s_cnt[3]) atomicAdd(g.counters + 6, (ull)s_cnt[3]);
  }
  if (g.want_hist)
    for (int b = threadIdx.x; b < kHistBins + kSubBins; b += NT)
      if (shist[b]) atomicAdd(g.hist + b, shist[b]);
}

/// One tile per CTA (single input stage): the default; enough CTAs stay
/// resident that load latency of one hides behind the merge of others.
template <int B, int NT, int IPT>
__global__ void __launch_bounds__(NT, merge_minb(B, NT)) k_merge1(MergeArgs g, Key<B> P) {
  using Cfg = MergeCfg<B, NT, IPT>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned* shist = reinterpret_cast<unsigned*>(smem_raw + Cfg::OFF_HIST - Cfg::STAGE);
  __shared__ __align__(8) unsigned long long mbar;
  __shared__ int s_cnt[4];
  const size_t tile = blockIdx.x;
  if (threadIdx.x == 0) {
    mbar_init(&mbar, 1);
    s_cnt[0] = s_cnt[1] = s_cnt[2] = s_cnt[3] = 0;
  }
  if (g.want_hist)
    for (int b = threadIdx.x; b < Cfg::HBINS; b += NT) shist[b] = 0;
  __syncthreads();
  ull* sk = reinterpret_cast<ull*>(smem_raw);
  double* sc = reinterpret_cast<double*>(smem_raw + Cfg::KEYB);
  unsigned* sbits = reinterpret_cast<unsigned*>(smem_raw + Cfg::OFF_SBITS);
  const TileBounds tb{g.part_a[tile], g.part_a[tile + 1], g.part_b[tile],
                      g.part_b[tile + 1], g.part_o[tile], g.part_o[tile + 1]};
  merge_issue<B, NT, Cfg::CAP>(g, tile, sk, sc, &mbar, sbits, Cfg::BW);
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  if (!IQCC_SPLIT_SMEM && tb.a1 > tb.a0) mbar_wait(&mbar, 0);
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&mbar)) : "memory");
  int n_eps = 0, n_dead = 0, n_coll = 0, n_ge = 0;
  const StagedBits sb{sbits, sbits + Cfg::BW, sbits + 2 * Cfg::BW, tb.a0 >> 5, tb.b0 >> 5};
  // shared layout past the single stage is shifted down by one STAGE
  merge_compute<B, NT, IPT>(g, tile, P, sk, sc, smem_raw - Cfg::STAGE, n_eps, n_dead, n_coll, n_ge, &tb, &sb);
  merge_flush<B, NT>(g, shist, n_eps, n_dead, n_coll, n_ge, s_cnt);
}

/// Persistent merge: each CTA walks tiles blockIdx.x, +gridDim.x, ... with a
/// two-stage pipeline: the next tile's TMA bulk copy and cp.async gathers
/// are in flight while the current tile is merged and stored.
#ifndef IQCC_PMERGE_MINB
#define IQCC_PMERGE_MINB 4
#endif
template <int B, int NT, int IPT>
__global__ void __launch_bounds__(NT, (B >= 4 ? 2 : IQCC_PMERGE_MINB) * 256 / NT) k_merge(MergeArgs g, Key<B> P) {
  using Cfg = MergeCfg<B, NT, IPT>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned* shist = reinterpret_cast<unsigned*>(smem_raw + Cfg::OFF_HIST);
  __shared__ __align__(8) unsigned long long mbar[2];
  __shared__ int s_cnt[4];
  if (threadIdx.x == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    s_cnt[0] = s_cnt[1] = s_cnt[2] = s_cnt[3] = 0;
  }
  if (g.want_hist)
    for (int b = threadIdx.x; b < Cfg::HBINS; b += NT) shist[b] = 0;
  __syncthreads();
  auto stage_k = [&](int st) { return reinterpret_cast<ull*>(smem_raw + st * Cfg::STAGE); };
  auto stage_c = [&](int st) {
    return reinterpret_cast<double*>(smem_raw + st * Cfg::STAGE + Cfg::KEYB);
  };
  size_t tile = blockIdx.x;
  if (tile < g.ntiles) merge_issue<B, NT, Cfg::CAP>(g, tile, stage_k(0), stage_c(0), &mbar[0]);
  unsigned phase[2] = {0u, 0u};
  int n_eps = 0, n_dead = 0, n_coll = 0, n_ge = 0;
  for (int it = 0; tile < g.ntiles; ++it, tile += gridDim.x) {
    const int cur = it & 1;
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    if (!IQCC_SPLIT_SMEM && g.part_a[tile + 1] > g.part_a[tile]) {
      mbar_wait(&mbar[cur], phase[cur]);
      phase[cur] ^= 1u;
    }
    __syncthreads();
    const size_t next = tile + gridDim.x;
    if (next < g.ntiles) merge_issue<B, NT, Cfg::CAP>(g, next, stage_k(cur ^ 1), stage_c(cur ^ 1), &mbar[cur ^ 1]);
    merge_compute<B, NT, IPT>(g, tile, P, stage_k(cur), stage_c(cur), smem_raw, n_eps, n_dead, n_coll, n_ge);
    __syncthreads();  // stage `cur` and the staging list are free again
  }
  merge_flush<B, NT>(g, shist, n_eps, n_dead, n_coll, n_ge, s_cnt);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&mbar[0])) : "memory");
    asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&mbar[1])) : "memory");
  }
}

// ---------------------------------------------------------- pipelined merge
// Persistent CTAs walk tiles blockIdx.x, +gridDim.x, ... with every global
// dependency of a tile issued ahead of its merge, so a CTA never waits on
// memory between tiles:
//   tile k+3: merge-path bounds loaded into registers (parked in a 3-slot
//             shared ring after the merge of tile k)
//   tile k+2: inv_perm slice fetched into shared memory by cp.async
//   tile k+1: survivors by TMA bulk copy (mbarrier), products gathered by
//             cp.async through the staged inv_perm, plan bit words by cp.async
//   tile k  : merged from shared memory (merge_compute)
// The |c| histogram and the counters are flushed once per CTA.
template <int B, int NT, int IPT>
struct PipeCfg {
  using M = MergeCfg<B, NT, IPT>;
  static constexpr int BW = M::PMW + 3;  // staged plan words per mask (a shifted window + 1)
  static constexpr size_t STAGE = (M::KEYB + (size_t)(M::CAP + 4) * 8 + (size_t)3 * BW * 4 + 127) & ~(size_t)127;
  static constexpr size_t OFF_BITS = M::KEYB + (size_t)(M::CAP + 4) * 8;  // within a stage
  static constexpr int IDXW = M::CAP + 8;  // staged inv_perm words per slot
  static constexpr size_t OFF_IDX = 2 * STAGE;
  static constexpr size_t OFF_REST = (OFF_IDX + (size_t)2 * IDXW * 4 + 127) & ~(size_t)127;
  // merge_compute's layout (outv ...) starts at OFF_REST: it addresses it as
  // smem_raw + M::OFF_OUTV with smem_raw shifted by OFF_REST - M::OFF_OUTV
  static constexpr size_t bytes(bool hist) {
    return OFF_REST + (M::OFF_HIST - M::OFF_OUTV) + (hist ? M::HBINS * 4 : 0);
  }
};

#ifndef IQCC_PIPE_MINB
#define IQCC_PIPE_MINB 4
#endif
template <int B, int NT, int IPT>
__global__ void __launch_bounds__(NT, (B >= 4 ? 2 : IQCC_PIPE_MINB) * 256 / NT) k_merge_pipe(MergeArgs g, Key<B> P) {
  using Cfg = PipeCfg<B, NT, IPT>;
  using M = MergeCfg<B, NT, IPT>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* rest = smem_raw + Cfg::OFF_REST - M::OFF_OUTV;  // merge_compute's base
  unsigned* shist = reinterpret_cast<unsigned*>(rest + M::OFF_HIST);
  __shared__ __align__(8) unsigned long long mbar[2];
  __shared__ int s_cnt[4];
  __shared__ TileBounds s_tb[3];
  auto stage = [&](int st) { return smem_raw + st * Cfg::STAGE; };
  auto idx_slot = [&](int sl) { return reinterpret_cast<unsigned*>(smem_raw + Cfg::OFF_IDX) + sl * Cfg::IDXW; };
  const size_t G = gridDim.x;
  const size_t t0 = blockIdx.x;
  auto tile_of = [&](size_t k) { return t0 + k * G; };
  auto load_bounds = [&](size_t t, ull* r) {  // threads 0..5: one bound each
    const int i = threadIdx.x;
    if (t < g.ntiles && i < 6) {
      const ull* src = i < 2 ? g.part_a : (i < 4 ? g.part_b : g.part_o);
      r[0] = src[t + (i & 1)];
    }
  };
  auto park_bounds = [&](int slot, ull v) {
    if (threadIdx.x < 6) reinterpret_cast<size_t*>(&s_tb[slot])[threadIdx.x] = (size_t)v;
  };
  // inv_perm[b0, b1) -> idx slot (16-byte aligned superset; local products only)
  auto issue_idx = [&](size_t t, int slot) {
    if (t >= g.ntiles || g.q_keys) return;
    const TileBounds& tb = s_tb[(t - t0) / G % 3];
    const size_t e0 = tb.b0 & ~(size_t)3, e1 = (tb.b1 + 3) & ~(size_t)3;
    unsigned* dst = idx_slot(slot);
    for (size_t j = threadIdx.x; j < (e1 - e0) / 4; j += NT) cp_async16(dst + 4 * j, g.inv_perm + e0 + 4 * j);
  };
  // survivors (TMA), products (cp.async gathers through the staged idx), plan bits
  auto issue_data = [&](size_t t, int st, int slot) {
    if (t >= g.ntiles) return;
    const TileBounds& tb = s_tb[(t - t0) / G % 3];
    unsigned char* base = stage(st);
    ull* sk = reinterpret_cast<ull*>(base);
    double* sc = reinterpret_cast<double*>(base + M::KEYB);
    unsigned* bits = reinterpret_cast<unsigned*>(base + Cfg::OFF_BITS);
    const int nS = (int)(tb.a1 - tb.a0), nQ = (int)(tb.b1 - tb.b0);
    stage_survivors<B, NT, M::CAP>(g, tb.a0, tb.a1, sk, sc, &mbar[st]);
    const int qc0 = nS + 4;
    if (g.q_keys) {
      for (int j = threadIdx.x; j < nQ; j += NT) {
        const ull* gk = g.q_keys + (tb.b0 + j) * 2 * B;
#pragma unroll
        for (int h = 0; h < B; ++h) cp_async16(sm_chunk<B, M::CAP>(sk, nS + j, h), gk + 2 * h);
        cp_async8(sc + qc0 + j, g.q_vals + tb.b0 + j);
      }
    } else {
      const unsigned* ix = idx_slot(slot) + (tb.b0 & 3);
      for (int j = threadIdx.x; j < nQ; j += NT) {
        const size_t src = ix[j];
        const ull* gk = g.keys + src * 2 * B;
#pragma unroll
        for (int h = 0; h < B; ++h) cp_async16(sm_chunk<B, M::CAP>(sk, nS + j, h), gk + 2 * h);
        cp_async8(sc + qc0 + j, g.coef + src);
      }
    }
    // plan bit words: pmask/fmask from word a0/32 on, product slot words from b0/32 on
    const size_t pw0 = tb.a0 >> 5, qw0 = tb.b0 >> 5;
    const int npw = (int)(((tb.a1 + 31) >> 5) - pw0) + 1, nqw = (int)(((tb.b1 + 31) >> 5) - qw0) + 1;
    for (int w = threadIdx.x; w < npw; w += NT) {
      cp_async4(bits + w, g.pmask + pw0 + w);
      cp_async4(bits + Cfg::BW + w, g.fmask + pw0 + w);
    }
    if (g.qbits)
      for (int w = threadIdx.x; w < nqw; w += NT) cp_async4(bits + 2 * Cfg::BW + w, g.qbits + qw0 + w);
  };
  auto commit = [] { asm volatile("cp.async.commit_group;\n" ::: "memory"); };

  if (threadIdx.x == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    s_cnt[0] = s_cnt[1] = s_cnt[2] = s_cnt[3] = 0;
  }
  if (g.want_hist)
    for (int b = threadIdx.x; b < M::HBINS; b += NT) shist[b] = 0;
  // prologue: bounds of tiles 0..2 (0, 1 parked, 2 in registers), idx of
  // tile 0 (waited), data of tile 0, idx of tile 1
  ull r0 = 0, r1 = 0, rn = 0;
  load_bounds(tile_of(0), &r0);
  load_bounds(tile_of(1), &r1);
  load_bounds(tile_of(2), &rn);
  park_bounds(0, r0);
  park_bounds(1, r1);
  __syncthreads();
  issue_idx(tile_of(0), 0);
  commit();
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  issue_data(tile_of(0), 0, 0);
  commit();
  issue_idx(tile_of(1), 1);
  commit();
  unsigned phase[2] = {0u, 0u};
  int n_eps = 0, n_dead = 0, n_coll = 0, n_ge = 0;
  for (size_t k = 0; tile_of(k) < g.ntiles; ++k) {
    const int cur = (int)(k & 1);
    const size_t t = tile_of(k);
    // data(k) and idx(k+1) landed; bounds(k+2) parked by the previous iteration
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    const TileBounds tb = s_tb[k % 3];
    if (!IQCC_SPLIT_SMEM && tb.a1 > tb.a0) {
      mbar_wait(&mbar[cur], phase[cur]);
      phase[cur] ^= 1u;
    }
    if (k == 0) park_bounds(2, rn);
    __syncthreads();
    issue_data(tile_of(k + 1), cur ^ 1, (int)((k + 1) & 1));
    commit();
    issue_idx(tile_of(k + 2), cur);  // the slot of idx(k), consumed by data(k)
    commit();
    ull rb = 0;
    load_bounds(tile_of(k + 3), &rb);  // lands while tile k is merged
    unsigned char* base = stage(cur);
    const unsigned* bits = reinterpret_cast<const unsigned*>(base + Cfg::OFF_BITS);
    const StagedBits sb{bits, bits + Cfg::BW, bits + 2 * Cfg::BW, tb.a0 >> 5, tb.b0 >> 5};
    merge_compute<B, NT, IPT>(g, t, P, reinterpret_cast<ull*>(base), reinterpret_cast<double*>(base + M::KEYB),
                              rest, n_eps, n_dead, n_coll, n_ge, &tb, &sb);
    __syncthreads();  // stage cur, the staging list and the ring slot k % 3 are free
    park_bounds((int)(k % 3), rb);
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  merge_flush<B, NT>(g, shist, n_eps, n_dead, n_coll, n_ge, s_cnt);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&mbar[0])) : "memory");
    asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&mbar[1])) : "memory");
  }
}

/// Merge tile shapes (NT threads x IPT items); the default per block count
/// can be overridden for tuning with IQCC_MERGE_CFG=<index>.
struct MergeShape {
  int nt, ipt;
};
constexpr MergeShape kMergeShapes[] = {{256, 4}, {128, 4}, {128, 8}, {256, 2}, {512, 2}, {64, 8}};

// ------------------------------------------------------------- host side
namespace {

template <int B>
Key<B> make_key(const uint64_t* row) {
  Key<B> k;
  row_to_device_key(row, B, k.w);
  return k;
}

template <int B>
std::vector<int> level_positions(const Key<B>& P) {
  // level order: word ascending, then bit index ascending (matches the pext
  // in k_classify); any order works for the rank sum
  std::vector<int> pos;
  for (int w = 0; w < 2 * B; ++w)
    for (int b = 0; b < 64; ++b)
      if ((P.w[w] >> b) & 1ull) pos.push_back(64 * w + (63 - b));
  return pos;
}



/// Device state of one planned step (classify + present prefix + product
/// order), shared by the local dressing step and the partitioned one.
struct PlanState {
  size_t M = 0, A = 0, W = 0;
  unsigned* inv_perm = nullptr;
  unsigned* pmask = nullptr;
  unsigned* fmask = nullptr;
  unsigned* ppre = nullptr;
  unsigned* ptotal = nullptr;
  const long long* a_dev = nullptr;  // device product count (nullptr: none)
  SlotRule rule{1.0, 0.0, 0.0, 0.0, 0.0, 0};
  const unsigned* qbits = nullptr;   // product slot bits in rank order (nullptr: all)
  const unsigned* qpre = nullptr;
  const unsigned* qtotal = nullptr;
  size_t Wq = 0;
};
thread_local PlanState g_plan;  // per host thread (engine context), see capi.cu

template <int B>
void plan_impl(DeviceStore& s, const Key<B>& P, bool products, bool read_A = true,
               SlotRule rule = SlotRule{1.0, 0.0, 0.0, 0.0, 0.0, 0}) {
  Workspace& ws = workspace();
  cudaStream_t st = stream();
  PlanState pl;
  pl.rule = rule;
  const size_t M = s.M;
  pl.M = M;
  const std::vector<int> pos = level_positions<B>(P);
  const int m = (int)pos.size();
  const int nch = (m + kLevelsPerChunk - 1) / kLevelsPerChunk;
  const size_t W = (M + 31) / 32;
  pl.W = W;
  unsigned* fmask = ws.fmask.as<unsigned>(3 * std::max<size_t>(W, 1) + 64);
  pl.fmask = fmask;
  pl.pmask = fmask + std::max<size_t>(W, 1);
  unsigned* qmask = pl.pmask + std::max<size_t>(W, 1);
  pl.ppre = ws.tables.as<unsigned>(std::max<size_t>(W, 1) + (W + PW - 1) / PW + 8);
  unsigned* bsum = pl.ppre + std::max<size_t>(W, 1);
  pl.ptotal = bsum + (W + PW - 1) / PW + 4;
  IQCC_CUDA(cudaMemsetAsync(pl.ptotal, 0, sizeof(unsigned), st));
  short* lcp = nullptr;
  // the previous merge of a dress_sequence already classified the store
  const bool use_meta = products && M > 0 && s.meta_valid &&
                        std::equal(P.w, P.w + 2 * B, s.meta_P);
  const size_t nb = (W + PW - 1) / PW;
  auto run_present = [&]() {
    KernelScope ks("present");
    k_popc_blocks<<<(unsigned)nb, 256, 0, st>>>(pl.pmask, W, bsum);
    k_scan_blocks<<<1, 1024, 0, st>>>(bsum, nb, pl.ptotal);
    k_popc_prefix<<<(unsigned)nb, 256, 0, st>>>(pl.pmask, W, bsum, pl.ppre);
    count_launch("present");
    count_launch("present");
  };
  MaskArgs ma{};
  if (use_meta) {
    lcp = s.meta_lcp.as<short>(M);
    ma.coef = s.coef();
    ma.amask = s.meta_amask.as<unsigned>(W + 2);
    ma.keys = s.keys();
    ma.W = 2 * B;
    ma.filt = s.filt;
    ma.fmask = fmask;
    ma.pmask = pl.pmask;
    ma.qmask = qmask;
    ma.rule = rule;
  } else if (M > 0) {
    lcp = ws.lcp.as<short>(M);
    {
      KernelScope ks("classify");
#ifdef IQCC_CLS_IT
      constexpr int IT = B >= 4 ? 2 : IQCC_CLS_IT;
#else
      constexpr int IT = 2;  // 56 registers: 4 CTAs / SM
#endif
      k_classify<B, IT><<<(unsigned)((M + 256 * IT - 1) / (256 * IT)), 256, 0, st>>>(
          s.keys(), s.coef(), s.filt, M, P, lcp, fmask, pl.pmask, rule, qmask);
    }
    if (getenv("IQCC_DEBUG")) debug_check("classify");
    run_present();
  }
  if (getenv("IQCC_DEBUG") && M > 0) debug_check("present");
  if (products && M > 0) {
    const size_t ntiles = (M + WT - 1) / WT;
    // IQCC_FORCE_GROUP_LARGE (test hook): take the large-shard carry path
    // (1024-tile groups, > 6.7e7 slots in production) at any size
    const int group = ntiles > (size_t)kGroupSmall * 1024 || getenv("IQCC_FORCE_GROUP_LARGE") ? kGroupLarge
                                                                                               : kGroupSmall;
    const size_t ngroups = (ntiles + group - 1) / group;
    if (ngroups > (size_t)kMaxGroups) throw std::runtime_error("dress: more than 2^28 terms per device shard");
    int* tile_cnt = ws.tile_cnt.as<int>(ntiles);
    int* fwd_agg = ws.fwd_agg.as<int>(ntiles * kThrPerChunk);
    int* bwd_agg = ws.bwd_agg.as<int>(ntiles * kThrPerChunk);
    int* tile_pfx = ws.tile_pfx.as<int>(ntiles);
    int* fwd_carry = ws.fwd_carry.as<int>(ntiles * kThrPerChunk);
    int* bwd_carry = ws.bwd_carry.as<int>(ntiles * kThrPerChunk);
    long long* g = ws.misc.as<long long>(ngroups * (1 + 2 * kThrPerChunk) + 8);
    long long* g_cnt = g;
    long long* g_fwd = g + ngroups;
    long long* g_bwd = g_fwd + ngroups * kThrPerChunk;
    long long* a_total = g_bwd + ngroups * kThrPerChunk;
    int* rdelta = nch > 1 ? ws.rdelta.as<int>(M) : nullptr;
    pl.inv_perm = ws.inv_perm.as<unsigned>(M + 8);  // +8: the pipelined merge fetches 16-byte groups
    // product slot flags in rank order (only when some products lose their slot)
    unsigned char* qflag = rule.thq != 0.0 ? ws.qflag.as<unsigned char>(M + 64) : nullptr;
    ull* dbg = debug_buffer();
    const unsigned wblocks = (unsigned)((ntiles + 7) / 8);
    for (int c = 0; c < nch; ++c) {
      Thr thr;
      thr.nlev = std::min(kLevelsPerChunk, m - c * kLevelsPerChunk);
      thr.n = 2 * thr.nlev;
      for (int j = 0; j < kThrPerChunk; ++j) thr.t[j] = -2;  // never a boundary
      for (int lv = 0; lv < thr.nlev; ++lv) {
        const int b = pos[c * kLevelsPerChunk + lv];
        thr.t[2 * lv] = b - 1;  // node start: lcp < b
        thr.t[2 * lv + 1] = b;  // child split: lcp <= b
      }
      const int nthr4 = (thr.n + 3) & ~3;
      thr.n = nthr4;  // padded thresholds (t = -2) flow through every kernel
      const bool last = c == nch - 1;
      {
        KernelScope ks("tile_agg");
#define IQCC_AGG(NT_, MK_) k_tile_agg_w<NT_, MK_><<<wblocks, 256, 0, st>>>(lcp, fmask, M, ntiles, thr, tile_cnt, fwd_agg, bwd_agg, ma)
        if (use_meta && c == 0) {
          switch (nthr4) {
            case 4: IQCC_AGG(4, true); break;
            case 8: IQCC_AGG(8, true); break;
            case 12: IQCC_AGG(12, true); break;
            default: IQCC_AGG(16, true); break;
          }
        } else {
          switch (nthr4) {
            case 4: IQCC_AGG(4, false); break;
            case 8: IQCC_AGG(8, false); break;
            case 12: IQCC_AGG(12, false); break;
            default: IQCC_AGG(16, false); break;
          }
        }
#undef IQCC_AGG
      }
      if (use_meta && c == 0) run_present();
      {
        KernelScope ks("carry");
        const unsigned cthreads = 32u * (unsigned)thr.n;  // one warp per threshold
        if (group == kGroupLarge)
          k_group_agg<kGroupLarge><<<(unsigned)ngroups, cthreads, 0, st>>>(tile_cnt, fwd_agg, bwd_agg, ntiles,
                                                                           thr.n, g_cnt, g_fwd, g_bwd);
        else
          k_group_agg<kGroupSmall><<<(unsigned)ngroups, cthreads, 0, st>>>(tile_cnt, fwd_agg, bwd_agg, ntiles,
                                                                           thr.n, g_cnt, g_fwd, g_bwd);
        k_group_scan<<<1, cthreads, 0, st>>>(ngroups, thr.n, g_cnt, g_fwd, g_bwd, a_total);
        if (group == kGroupLarge)
          k_tile_carry<kGroupLarge><<<(unsigned)ngroups, cthreads, 0, st>>>(tile_cnt, fwd_agg, bwd_agg, ntiles, thr.n,
                                                          g_cnt, g_fwd, g_bwd, a_total, tile_pfx,
                                                          fwd_carry, bwd_carry);
        else
          k_tile_carry<kGroupSmall><<<(unsigned)ngroups, cthreads, 0, st>>>(tile_cnt, fwd_agg, bwd_agg, ntiles, thr.n,
                                                          g_cnt, g_fwd, g_bwd, a_total, tile_pfx,
                                                          fwd_carry, bwd_carry);
        count_launch("carry");
        count_launch("carry");
      }
      {
        KernelScope ks("rank");
#define IQCC_RANK(NT_, F_) k_rank_w<NT_, F_><<<wblocks, 256, 0, st>>>(lcp, fmask, M, ntiles, thr, tile_pfx, fwd_carry, bwd_carry, rdelta, c > 0, pl.inv_perm, a_total, dbg, qmask, qflag)
        if (last) {
          switch (nthr4) {
            case 4: IQCC_RANK(4, true); break;
            case 8: IQCC_RANK(8, true); break;
            case 12: IQCC_RANK(12, true); break;
            default: IQCC_RANK(16, true); break;
          }
        } else {
          switch (nthr4) {
            case 4: IQCC_RANK(4, false); break;
            case 8: IQCC_RANK(8, false); break;
            case 12: IQCC_RANK(12, false); break;
            default: IQCC_RANK(16, false); break;
          }
        }
#undef IQCC_RANK
      }
    }
    if (getenv("IQCC_DEBUG")) debug_check("rank");
    pl.a_dev = a_total;
    if (!read_A) {  // the caller reads the count (with its own round trip)
      g_plan = pl;
      return;
    }
    long long* a_host = static_cast<long long*>(host_pinned(sizeof(long long)));
    d2h_small(a_host, a_total, sizeof(long long), st);
    host_sync(st);
    pl.A = (size_t)*a_host;
    if (qflag) {  // flags -> bits + popcount prefix (like the survivor slot bits)
      const size_t A = pl.A, Wq = (A + 31) / 32, nbq = (Wq + PW - 1) / PW;
      unsigned* qb = ws.qbits.as<unsigned>(2 * std::max<size_t>(Wq, 1) + nbq + 64);
      unsigned* qpre = qb + std::max<size_t>(Wq, 1) + 2;
      unsigned* qbs = qpre + std::max<size_t>(Wq, 1);
      unsigned* qtot = qbs + nbq + 4;
      IQCC_CUDA(cudaMemsetAsync(qb, 0, (std::max<size_t>(Wq, 1) + 2) * sizeof(unsigned), st));
      IQCC_CUDA(cudaMemsetAsync(qtot, 0, sizeof(unsigned), st));
      if (A > 0) {
        KernelScope ks("present");
        k_pack_flags<<<(unsigned)((Wq + 255) / 256), 256, 0, st>>>(qflag, A, qb);
        k_popc_blocks<<<(unsigned)nbq, 256, 0, st>>>(qb, Wq, qbs);
        k_scan_blocks<<<1, 1024, 0, st>>>(qbs, nbq, qtot);
        k_popc_prefix<<<(unsigned)nbq, 256, 0, st>>>(qb, Wq, qbs, qpre);
        count_launch("present");
        count_launch("present");
        count_launch("present");
      }
      pl.qbits = qb;
      pl.qpre = qpre;
      pl.qtotal = qtot;
      pl.Wq = Wq;
    }
    if (getenv("IQCC_DEBUG") && pl.A > 0) {
      unsigned* seen = ws.misc2.as<unsigned>(M);
      IQCC_CUDA(cudaMemsetAsync(seen, 0, M * sizeof(unsigned), st));
      k_check_perm<<<(unsigned)((pl.A + 255) / 256), 256, 0, st>>>(pl.inv_perm, pl.A, M, fmask, seen, dbg);
      debug_check("perm check");
    }
  }
  g_plan = pl;
}

thread_local int g_sub_b0 = -(1 << 20);  // fine-histogram window of the last merge (see kSubBins)

template <int B, int NT, int IPT>
void launch_merge_t(DeviceStore& s, const Key<B>& P, size_t nQ, const ull* q_keys, const double* q_vals,
                    double cs, double sn, double drop, bool want_hist, double eps, const Key<B>* PN,
                    double theta, const ChunkPlan* cp) {
  Workspace& ws = workspace();
  cudaStream_t st = stream();
  const PlanState& pl = g_plan;
  constexpr int TILEM = NT * IPT;
  const size_t M = s.M;
  const size_t total = M + nQ;
  // tiles: one range, or per chunk of a chunked merge (chunk c = S[a_c,
  // a_c+1) with Q[r_c, r_c+1), tiles [T_c, T_c+1) of one global tile list)
  const int C = cp ? cp->C : 1;
  std::vector<size_t> tc(C + 1, 0);
  size_t nco_max = 1;
  for (int c = 0; c < C; ++c) {
    const size_t len = cp ? (cp->a[c + 1] - cp->a[c]) + (cp->r[c + 1] - cp->r[c]) : total;
    const size_t n = cp ? (len + TILEM - 1) / TILEM : std::max<size_t>(1, (total + TILEM - 1) / TILEM);
    tc[c + 1] = tc[c] + n;
    nco_max = std::max(nco_max, (n >> kPartShift) + 1);
  }
  const size_t ntm = tc[C];
  if (cp && (ntm == 0 || cp->a[C] != M || cp->r[C] != nQ))
    throw std::logic_error("chunked merge: chunk bounds do not cover the inputs");
  ull* pa = ws.part_a.as<ull>(3 * (ntm + 1) + nco_max + 8);
  ull* pb = pa + (ntm + 1);
  ull* po = pb + (ntm + 1);
  auto partition = [&](int c, const unsigned* qtotal, size_t Wq) {
    KernelScope ks("partition");
    ull* raw = po + (ntm + 1);
    const size_t a0 = cp ? cp->a[c] : 0, b0 = cp ? cp->r[c] : 0;
    const size_t nS = cp ? cp->a[c + 1] - a0 : M, nq = cp ? cp->r[c + 1] - b0 : nQ;
    const size_t n = tc[c + 1] - tc[c], nco = (n >> kPartShift) + 1;
    k_partition_coarse<B><<<(unsigned)((nco * 32 + 255) / 256), 256, 0, st>>>(
        s.keys(), pl.inv_perm, q_keys, nS, nq, P, TILEM, n, raw, a0, b0);
    k_partition<B><<<(unsigned)((n + 1 + 255) / 256), 256, 0, st>>>(
        s.keys(), pl.inv_perm, q_keys, nS, nq, P, TILEM, n, pa + tc[c], pb + tc[c], po + tc[c], pl.pmask,
        pl.ppre, pl.W, pl.ptotal, pl.qbits, pl.qpre, Wq, qtotal, 0, raw, a0, b0);
    count_launch("partition");
  };
  if (!cp) partition(0, pl.qtotal, pl.Wq);
  ull* out_keys = ws.out_keys.as<ull>(std::max<size_t>(total, 1) * 2 * B);
  double* out_coef = ws.out_coef.as<double>(std::max<size_t>(total, 1));
  ull* ctr = ws.counters.as<ull>(16);
  unsigned* hist = ws.hist.as<unsigned>(kHistBins + kSubBins);
  IQCC_CUDA(cudaMemsetAsync(ctr, 0, 8 * sizeof(ull), st));
  if (want_hist) IQCC_CUDA(cudaMemsetAsync(hist, 0, (kHistBins + kSubBins) * sizeof(unsigned), st));
  using Cfg = MergeCfg<B, NT, IPT>;
  MergeArgs g;
  g.keys = s.keys();
  g.coef = s.coef();
  g.filt = s.filt;
  g.inv_perm = pl.inv_perm;
  g.q_keys = q_keys;
  g.q_vals = q_vals;
  g.part_a = pa;
  g.part_b = pb;
  g.part_o = po;
  g.ntiles = ntm;
  g.cs = cs;
  g.sn = sn;
  g.drop = drop;
  g.eps = eps;
  g.out_keys = out_keys;
  g.out_coef = out_coef;
  g.counters = ctr;
  g.hist = hist;
  g.want_hist = want_hist ? 1 : 0;
  g.dbg = debug_buffer();
  g.rule = pl.rule;
  g.theta = want_hist ? theta : 0.0;
  // the cut lies at or above the (verified) floor theta: a fine histogram of
  // the exponent bins from theta's up lets the select skip ~6 bits
  g.sub_b0 = want_hist && theta > 0.0 ? hist_bin_of(theta) : -(1 << 20);
  g_sub_b0 = g.sub_b0;
  g.qbits = pl.qbits;
  g.pmask = pl.pmask;
  g.fmask = pl.fmask;
  g.out_lcp = nullptr;
  g.out_amask = nullptr;
  for (int w = 0; w < 8; ++w) g.pn[w] = 0;
  if (PN) {
    g.out_lcp = s.meta_lcp.as<short>(std::max<size_t>(total, 1));
    const size_t wn = total / 32 + 2;
    g.out_amask = s.meta_amask.as<unsigned>(wn);
    IQCC_CUDA(cudaMemsetAsync(g.out_amask, 0, wn * sizeof(unsigned), st));
    for (int w = 0; w < 2 * B; ++w) g.pn[w] = PN->w[w];
  }
  static const bool persistent = getenv("IQCC_MERGE_PERSIST") != nullptr;
  static const bool pipelined = getenv("IQCC_MERGE_PIPE") != nullptr && atoi(getenv("IQCC_MERGE_PIPE")) != 0;
  if (pipelined && !cp) {
    using PC = PipeCfg<B, NT, IPT>;
    static int ctas_per_sm = 0, n_sm = 0;
    const int dev = ctx_device(ctx_current());
    if (func_attr_once((const void*)k_merge_pipe<B, NT, IPT>, dev)) {
      IQCC_CUDA(cudaFuncSetAttribute(k_merge_pipe<B, NT, IPT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)PC::bytes(true)));
      IQCC_CUDA(cudaFuncSetAttribute(k_merge_pipe<B, NT, IPT>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     (int)cudaSharedmemCarveoutMaxShared));
    }
    if (!ctas_per_sm) {
      IQCC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas_per_sm, k_merge_pipe<B, NT, IPT>, NT,
                                                              PC::bytes(true)));
      IQCC_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
      ctas_per_sm = std::max(ctas_per_sm, 1);
    }
    KernelScope ks("merge");
    const unsigned grid = (unsigned)std::min<size_t>(ntm, (size_t)n_sm * ctas_per_sm);
    k_merge_pipe<B, NT, IPT><<<grid, NT, PC::bytes(want_hist), st>>>(g, P);
  } else if (persistent && !cp) {
    static int ctas_per_sm = 0, n_sm = 0;
    if (func_attr_once((const void*)k_merge<B, NT, IPT>, ctx_device(ctx_current())))
      IQCC_CUDA(cudaFuncSetAttribute(k_merge<B, NT, IPT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)Cfg::bytes(true, 2)));
    if (!ctas_per_sm) {
      IQCC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas_per_sm, k_merge<B, NT, IPT>, NT,
                                                              Cfg::bytes(true, 2)));
      IQCC_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, 0));
      ctas_per_sm = std::max(ctas_per_sm, 1);
    }
    KernelScope ks("merge");
    const unsigned grid = (unsigned)std::min<size_t>(ntm, (size_t)n_sm * ctas_per_sm);
    k_merge<B, NT, IPT><<<grid, NT, Cfg::bytes(want_hist, 2), st>>>(g, P);
  } else {
    if (func_attr_once((const void*)k_merge1<B, NT, IPT>, ctx_device(ctx_current()))) {
      IQCC_CUDA(cudaFuncSetAttribute(k_merge1<B, NT, IPT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)Cfg::bytes(true, 1)));
      IQCC_CUDA(cudaFuncSetAttribute(k_merge1<B, NT, IPT>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     (int)cudaSharedmemCarveoutMaxShared));
    }
    if (!cp) {
      KernelScope ks("merge");
      k_merge1<B, NT, IPT><<<(unsigned)ntm, NT, Cfg::bytes(want_hist, 1), st>>>(g, P);
    } else {
      // chunk by chunk as the products land: the wait for chunk c (and its
      // slot bits) is enqueued by the caller, then its partition and merge
      for (int c = 0; c < C; ++c) {
        const unsigned* qtotal = pl.qtotal;
        size_t Wq = pl.Wq;
        cp->arrive(c, &qtotal, &Wq);
        const size_t n = tc[c + 1] - tc[c];
        if (n == 0) continue;
        partition(c, qtotal, Wq);
        MergeArgs gc = g;
        gc.part_a = pa + tc[c];
        gc.part_b = pb + tc[c];
        gc.part_o = po + tc[c];
        gc.ntiles = n;
        KernelScope ks("merge");
        k_merge1<B, NT, IPT><<<(unsigned)n, NT, Cfg::bytes(want_hist, 1), st>>>(gc, P);
      }
    }
  }
  if (PN) {
    KernelScope ks("meta_fix");
    k_meta_fix<B><<<(unsigned)((ntm + 255) / 256), 256, 0, st>>>(out_keys, po, ntm, g.out_lcp);
  }
  IQCC_CUDA(cudaMemcpyAsync(ctr + 3, po + ntm, sizeof(ull), cudaMemcpyDeviceToDevice, st));
  if (getenv("IQCC_DEBUG")) debug_check("merge");
}

thread_local Reducer* g_merge_red = nullptr;

__global__ void k_pack_glob(ull* ctr, ull identity) {
  if (threadIdx.x == 0) {
    ctr[8] = ctr[1];
    ctr[9] = ctr[6];
    ctr[10] = identity;
  }
}

template <int B>
DressOutcome merge_impl(DeviceStore& s, const Key<B>& P, size_t nQ, const ull* q_keys,
                        const double* q_vals, double cs, double sn, double drop, bool want_hist,
                        double eps, const Key<B>* PN = nullptr, double theta = 0.0,
                        const ChunkPlan* cp = nullptr) {
  static int shape = -1;
  if (shape < 0) {
    const char* env = getenv("IQCC_MERGE_CFG");
    shape = env ? atoi(env) : 3;
    if (shape < 0 || shape >= (int)(sizeof(kMergeShapes) / sizeof(kMergeShapes[0]))) shape = 3;
  }
#define IQCC_MERGE(NT_, IPT_) launch_merge_t<B, NT_, IPT_>(s, P, nQ, q_keys, q_vals, cs, sn, drop, want_hist, eps, PN, theta, cp)
  switch (shape) {
    case 0: IQCC_MERGE(256, 4); break;
    case 1: IQCC_MERGE(128, 4); break;
    case 2: IQCC_MERGE(128, 8); break;
    case 3: IQCC_MERGE(256, 2); break;
    case 4: IQCC_MERGE(512, 2); break;
    default: IQCC_MERGE(64, 8); break;
  }
#undef IQCC_MERGE
  Workspace& ws = workspace();
  cudaStream_t st = stream();
  ull* ctr = ws.counters.as<ull>(16);
  ull* hc = static_cast<ull*>(host_pinned(16 * sizeof(ull)));
  if (g_merge_red) {
    k_pack_glob<<<1, 32, 0, st>>>(ctr, s.has_identity ? 1ull : 0ull);
    g_merge_red->sum_device(ctr + 8, 3);
  }
  d2h_small(hc, ctr, (g_merge_red ? 11 : 8) * sizeof(ull), st);
  host_sync(st);
  std::swap(s.kbuf, ws.out_keys);
  std::swap(s.cbuf, ws.out_coef);
  // algorithmic bytes of the step: (M_in + M_out) * (16B + 8),
  // M_out = the dressed sum's size (present survivors + products - partner
  // pairs) whether or not every term got an output slot
  const size_t logical_in = s.logical;
  const size_t m_out = logical_in + nQ - hc[5];
  s.M = hc[3];                // physical slots (live + dead)
  s.filt = Filter{};
  s.logical = hc[3] - hc[2];  // minus dead slots
  s.meta_valid = PN != nullptr;
  if (PN)
    for (int w = 0; w < 2 * B; ++w) s.meta_P[w] = PN->w[w];
  add_alg_bytes("merge", (double)(logical_in + m_out) * (16.0 * B + 8.0));
  DressOutcome out;
  out.count_eps = hc[1];
  out.n_anticommuting = g_plan.A;
  out.n_ge_theta = hc[6];
  out.n_pairs = hc[5];
  if (g_merge_red) {
    out.has_glob = true;
    for (int k = 0; k < 3; ++k) out.glob[k] = hc[8 + k];
  }
  return out;
}

template <int B>
DressOutcome dress_impl(DeviceStore& s, const uint64_t* gen_row, double cs, double sn, double drop,
                        bool want_hist, double eps, const uint64_t* next_row, double theta,
                        bool anti_only) {
  const Key<B> P = make_key<B>(gen_row);
  SlotRule rule = make_slot_rule(cs, sn, theta);
  rule.anti_only = anti_only ? 1 : 0;
  plan_impl<B>(s, P, sn != 0.0, true, rule);
  Key<B> PN;
  if (next_row) PN = make_key<B>(next_row);
  return merge_impl<B>(s, P, g_plan.A, nullptr, nullptr, cs, sn, drop, want_hist, eps,
                       next_row ? &PN : nullptr, theta);
}

// Sorted products as a contiguous buffer (keys ^ P, +-fl(c*sin)) for a peer.
template <int B>
__global__ void k_materialize(const ull* __restrict__ keys, const double* __restrict__ coef,
                              const unsigned* __restrict__ inv_perm, size_t r0, size_t A, Key<B> P,
                              double sn, ull* __restrict__ okeys, double* __restrict__ ovals,
                              double thq, unsigned* __restrict__ obits) {
  const size_t r = r0 + blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  double v = 0.0;
  if (r < A) {
    const unsigned src = inv_perm[r];
    const Key<B> k = load_key<B>(keys, src);
    const double pr = __dmul_rn(coef[src], sn);
    store_key<B>(okeys, r, key_xor<B>(k, P));
    v = product_phase<B>(k, P) == 1 ? pr : -pr;
    ovals[r] = v;
  }
  if (obits) {  // the receiver's slot bits (SlotRule: |v| >= thq), r0 % 32 == 0
    const unsigned b = __ballot_sync(0xffffffffu, r < A && fabs(v) >= thq);
    if ((threadIdx.x & 31) == 0 && r < A) obits[r >> 5] = b;
  }
}

/// Products pushed straight into a peer's receive buffer over NVLink (CUDA
/// IPC mapping): each CTA gathers a tile of 256 products into shared memory,
/// then writes it with fully coalesced 16-byte stores, so the remote writes
/// leave as full lines (per-thread scattered row stores halve NVLink
/// throughput).  Grid-stride over tiles; one CTA per SM slot.
template <int B>
__global__ void __launch_bounds__(256) k_push(const ull* __restrict__ keys, const double* __restrict__ coef,
                                              const unsigned* __restrict__ inv_perm, size_t A, Key<B> P,
                                              double sn, ull* __restrict__ okeys, double* __restrict__ ovals,
                                              size_t r_begin = 0) {
  __shared__ __align__(16) ull sk[256 * 2 * B];
  __shared__ __align__(16) double sv[256];
  for (size_t t = blockIdx.x; r_begin + t * 256 < A; t += gridDim.x) {
    const size_t r0 = r_begin + t * 256;
    const int n = (int)min((size_t)256, A - r0);
    if ((int)threadIdx.x < n) {
      const unsigned src = inv_perm[r0 + threadIdx.x];
      const Key<B> k = load_key<B>(keys, src);
      const double pr = __dmul_rn(coef[src], sn);
      const Key<B> q = key_xor<B>(k, P);
#pragma unroll
      for (int w = 0; w < 2 * B; ++w) sk[threadIdx.x * 2 * B + w] = q.w[w];
      sv[threadIdx.x] = product_phase<B>(k, P) == 1 ? pr : -pr;
    }
    __syncthreads();
    ulonglong2* dk = reinterpret_cast<ulonglong2*>(okeys + r0 * 2 * B);
    const ulonglong2* s2 = reinterpret_cast<const ulonglong2*>(sk);
    for (int j = threadIdx.x; j < n * B; j += 256) dk[j] = s2[j];
    if (n == 256 && (r0 & 1) == 0) {
      if (threadIdx.x < 128)
        reinterpret_cast<double2*>(ovals + r0)[threadIdx.x] = reinterpret_cast<const double2*>(sv)[threadIdx.x];
    } else if ((int)threadIdx.x < n) {
      ovals[r0 + threadIdx.x] = sv[threadIdx.x];
    }
    __syncthreads();
  }
  __threadfence_system();  // the remote stores land before a ready flag raised after this kernel
}

}  // namespace

void push_products(DeviceStore& s, const uint64_t* gen_row, double sn, ull* okeys, double* ovals,
                   size_t r0, size_t r1, cudaStream_t on, unsigned max_grid) {
  const size_t A = std::min(r1, g_plan.A);
  if (A <= r0) return;
  cudaStream_t st = on ? on : stream();
  std::optional<KernelScope> ks;
  if (!on) ks.emplace("exchange");
  const unsigned grid = (unsigned)std::min<size_t>((A - r0 + 255) / 256, max_grid ? max_grid : 148 * 8);
  switch (s.B) {
    case 1: k_push<1><<<grid, 256, 0, st>>>(s.keys(), s.coef(), g_plan.inv_perm, A, make_key<1>(gen_row), sn, okeys, ovals, r0); break;
    case 2: k_push<2><<<grid, 256, 0, st>>>(s.keys(), s.coef(), g_plan.inv_perm, A, make_key<2>(gen_row), sn, okeys, ovals, r0); break;
    default: k_push<4><<<grid, 256, 0, st>>>(s.keys(), s.coef(), g_plan.inv_perm, A, make_key<4>(gen_row), sn, okeys, ovals, r0); break;
  }
}

const long long* plan_products_async(DeviceStore& s, const uint64_t* gen_row, double cs,
                                     double sn, double theta) {
  // survivor slots by the rule; the products leave for the peer, whose
  // slot bits the receiver derives from the values (recv_slot_bits)
  const SlotRule r{cs, sn, theta, 0.0, 0.0, 0};
  switch (s.B) {
    case 1: plan_impl<1>(s, make_key<1>(gen_row), true, false, r); break;
    case 2: plan_impl<2>(s, make_key<2>(gen_row), true, false, r); break;
    default: plan_impl<4>(s, make_key<4>(gen_row), true, false, r); break;
  }
  return g_plan.a_dev;
}

void plan_survivors(DeviceStore& s, const uint64_t* gen_row, double cs, double sn, double theta) {
  const SlotRule r{cs, sn, theta, 0.0, 0.0, 0};
  switch (s.B) {
    case 1: plan_impl<1>(s, make_key<1>(gen_row), false, true, r); break;
    case 2: plan_impl<2>(s, make_key<2>(gen_row), false, true, r); break;
    default: plan_impl<4>(s, make_key<4>(gen_row), false, true, r); break;
  }
}

/// Slot bits of received products (final values, rank order): a product
/// without a partner keeps its value, so slot iff |v| >= thq (SlotRule).
__global__ void k_value_slots(const double* __restrict__ v, size_t n, double thq,
                              unsigned* __restrict__ bits) {
  const size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const bool f = j < n && fabs(v[j]) >= thq;
  const unsigned b = __ballot_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0 && j < n) bits[j >> 5] = b;
}

void recv_slot_bits(const double* rv, size_t n, double thq) {
  g_plan.qbits = g_plan.qpre = g_plan.qtotal = nullptr;
  g_plan.Wq = 0;
  if (thq == 0.0) return;  // every received product owns a slot
  Workspace& ws = workspace();
  cudaStream_t st = stream();
  const size_t Wq = (n + 31) / 32, nbq = (Wq + PW - 1) / PW;
  unsigned* qb = ws.qbits.as<unsigned>(2 * std::max<size_t>(Wq, 1) + nbq + 64);
  unsigned* qpre = qb + std::max<size_t>(Wq, 1) + 2;
  unsigned* qbs = qpre + std::max<size_t>(Wq, 1);
  unsigned* qtot = qbs + nbq + 4;
  IQCC_CUDA(cudaMemsetAsync(qb, 0, (std::max<size_t>(Wq, 1) + 2) * sizeof(unsigned), st));
  IQCC_CUDA(cudaMemsetAsync(qtot, 0, sizeof(unsigned), st));
  if (n > 0) {
    KernelScope ks("present");
    k_value_slots<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(rv, n, thq, qb);
    k_popc_blocks<<<(unsigned)nbq, 256, 0, st>>>(qb, Wq, qbs);
    k_scan_blocks<<<1, 1024, 0, st>>>(qbs, nbq, qtot);
    k_popc_prefix<<<(unsigned)nbq, 256, 0, st>>>(qb, Wq, qbs, qpre);
    count_launch("present");
    count_launch("present");
    count_launch("present");
  }
  g_plan.qbits = qb;
  g_plan.qpre = qpre;
  g_plan.qtotal = qtot;
  g_plan.Wq = Wq;
}

thread_local double g_rs_thq = 0.0;
thread_local unsigned* g_qtc = nullptr;  // running slot totals through each chunk

void recv_slot_bits_begin(size_t n, double thq, int chunks) {
  g_plan.qbits = g_plan.qpre = g_plan.qtotal = nullptr;
  g_plan.Wq = 0;
  g_rs_thq = thq;
  if (thq == 0.0) return;  // every received product owns a slot
  Workspace& ws = workspace();
  cudaStream_t st = stream();
  const size_t Wq = (n + 31) / 32, nbq = (Wq + PW - 1) / PW;
  unsigned* qb = ws.qbits.as<unsigned>(2 * std::max<size_t>(Wq, 1) + nbq + 64 + chunks);
  unsigned* qpre = qb + std::max<size_t>(Wq, 1) + 2;
  unsigned* qbs = qpre + std::max<size_t>(Wq, 1);
  g_qtc = qbs + nbq + 8;
  IQCC_CUDA(cudaMemsetAsync(qb, 0, (std::max<size_t>(Wq, 1) + 2) * sizeof(unsigned), st));
  g_plan.qbits = qb;
  g_plan.qpre = qpre;
  g_plan.qtotal = g_qtc + (chunks - 1);
  g_plan.Wq = Wq;
}

void recv_slot_bits_chunk(const double* rv, size_t r0, size_t r1, size_t n, int c,
                          const unsigned** qtotal, size_t* Wq) {
  if (!g_plan.qbits) return;
  if (r0 % (32 * (size_t)PW)) throw std::logic_error("recv_slot_bits_chunk: unaligned chunk");
  cudaStream_t st = stream();
  const size_t Wall = (n + 31) / 32, nbq = (Wall + PW - 1) / PW;
  unsigned* qb = const_cast<unsigned*>(g_plan.qbits);  // this context's workspace arrays
  unsigned* qpre = const_cast<unsigned*>(g_plan.qpre);
  unsigned* qbs = qpre + std::max<size_t>(Wall, 1);
  const size_t w0 = r0 / 32, w1 = (r1 + 31) / 32;
  if (r1 > r0) {
    KernelScope ks("present");
    const size_t b0 = w0 / PW, b1 = std::min(nbq, (w1 + PW - 1) / PW);
    k_value_slots<<<(unsigned)((r1 - r0 + 255) / 256), 256, 0, st>>>(rv + r0, r1 - r0, g_rs_thq, qb + w0);
    k_popc_blocks<<<(unsigned)(b1 - b0), 256, 0, st>>>(qb + w0, w1 - w0, qbs + b0);
    k_scan_blocks<<<1, 1024, 0, st>>>(qbs + b0, b1 - b0, g_qtc + c, c ? g_qtc + c - 1 : nullptr);
    k_popc_prefix<<<(unsigned)(b1 - b0), 256, 0, st>>>(qb + w0, w1 - w0, qbs + b0, qpre + w0);
    count_launch("present");
    count_launch("present");
    count_launch("present");
  } else if (c == 0) {
    IQCC_CUDA(cudaMemsetAsync(g_qtc, 0, sizeof(unsigned), st));
  } else {
    IQCC_CUDA(cudaMemcpyAsync(g_qtc + c, g_qtc + c - 1, sizeof(unsigned), cudaMemcpyDeviceToDevice, st));
  }
  *qtotal = g_qtc + c;
  *Wq = std::max(w0, w1);
}

void plan_set_products(size_t A) { g_plan.A = A; }

const unsigned* plan_inv_perm() { return g_plan.inv_perm; }

void set_merge_reducer(Reducer* red) { g_merge_red = red; }

int merge_sub_window() { return g_sub_b0; }

size_t plan_products(DeviceStore& s, const uint64_t* gen_row, bool products) {
  switch (s.B) {
    case 1: plan_impl<1>(s, make_key<1>(gen_row), products); break;
    case 2: plan_impl<2>(s, make_key<2>(gen_row), products); break;
    default: plan_impl<4>(s, make_key<4>(gen_row), products); break;
  }
  return g_plan.A;
}

void materialize_products(DeviceStore& s, const uint64_t* gen_row, double sn, ull* okeys,
                          double* ovals, size_t r0, size_t r1, const char* family, double thq,
                          unsigned* obits) {
  r1 = std::min(r1, g_plan.A);
  if (r1 <= r0) return;
  cudaStream_t st = stream();
  KernelScope ks(family);
  const unsigned grid = (unsigned)((r1 - r0 + 255) / 256);
  switch (s.B) {
    case 1: k_materialize<1><<<grid, 256, 0, st>>>(s.keys(), s.coef(), g_plan.inv_perm, r0, r1, make_key<1>(gen_row), sn, okeys, ovals, thq, obits); break;
    case 2: k_materialize<2><<<grid, 256, 0, st>>>(s.keys(), s.coef(), g_plan.inv_perm, r0, r1, make_key<2>(gen_row), sn, okeys, ovals, thq, obits); break;
    default: k_materialize<4><<<grid, 256, 0, st>>>(s.keys(), s.coef(), g_plan.inv_perm, r0, r1, make_key<4>(gen_row), sn, okeys, ovals, thq, obits); break;
  }
}

/// Slot bits of n received products already packed by the sender (bits
/// words, possibly in a peer's memory): the local prefix for the merge.
void recv_slot_bits_packed(const unsigned* bits, size_t n, double thq) {
  g_plan.qbits = g_plan.qpre = g_plan.qtotal = nullptr;
  g_plan.Wq = 0;
  if (thq == 0.0) return;
  Workspace& ws = workspace();
  cudaStream_t st = stream();
  const size_t Wq = (n + 31) / 32, nbq = (Wq + PW - 1) / PW;
  unsigned* qpre = ws.qbits.as<unsigned>(std::max<size_t>(Wq, 1) + nbq + 64);
  unsigned* qbs = qpre + std::max<size_t>(Wq, 1);
  unsigned* qtot = qbs + nbq + 4;
  IQCC_CUDA(cudaMemsetAsync(qtot, 0, sizeof(unsigned), st));
  if (n > 0) {
    KernelScope ks("present");
    k_popc_blocks<<<(unsigned)nbq, 256, 0, st>>>(bits, Wq, qbs);
    k_scan_blocks<<<1, 1024, 0, st>>>(qbs, nbq, qtot);
    k_popc_prefix<<<(unsigned)nbq, 256, 0, st>>>(bits, Wq, qbs, qpre);
    count_launch("present");
    count_launch("present");
  }
  g_plan.qbits = bits;
  g_plan.qpre = qpre;
  g_plan.qtotal = qtot;
  g_plan.Wq = Wq;
}

template <int B>
DressOutcome merge_products_t(DeviceStore& s, const uint64_t* gen_row, double cs, double sn,
                              double drop, bool want_hist, double eps, size_t nQ, const ull* q_keys,
                              const double* q_vals, const uint64_t* next_row, double theta,
                              const ChunkPlan* cp) {
  Key<B> PN;
  if (next_row) PN = make_key<B>(next_row);
  return merge_impl<B>(s, make_key<B>(gen_row), nQ, q_keys, q_vals, cs, sn, drop, want_hist, eps,
                       next_row ? &PN : nullptr, theta, cp);
}

DressOutcome merge_products(DeviceStore& s, const uint64_t* gen_row, double cs, double sn,
                            double drop, bool want_hist, double eps, size_t nQ, const ull* q_keys,
                            const double* q_vals, const uint64_t* next_row, double theta,
                            const ChunkPlan* cp) {
  switch (s.B) {
    case 1: return merge_products_t<1>(s, gen_row, cs, sn, drop, want_hist, eps, nQ, q_keys, q_vals, next_row, theta, cp);
    case 2: return merge_products_t<2>(s, gen_row, cs, sn, drop, want_hist, eps, nQ, q_keys, q_vals, next_row, theta, cp);
    default: return merge_products_t<4>(s, gen_row, cs, sn, drop, want_hist, eps, nQ, q_keys, q_vals, next_row, theta, cp);
  }
}

/// merge_sums (iqcc/pauli.hpp:383-415): out = a's terms merged with b's
/// through the merge kernel with an all-zero "entangler" (it commutes with
/// every word, so a's values pass unchanged and b enters as received,
/// final products): a + b (a first) on shared words, keep_term(drop) on
/// every output, identity always kept.
void merge_sums_store(DeviceStore& a, DeviceStore& b, double drop, DeviceStore& out) {
  if (a.n_qubits != b.n_qubits) throw std::invalid_argument("merge_sums: mismatched qubit counts");
  store_materialize(b);  // plain sorted live terms (same logical content)
  store_clone(a, out);
  const std::vector<uint64_t> zero(2 * out.B, 0);
  plan_survivors(out, zero.data(), 1.0, 0.0, 0.0);
  recv_slot_bits(b.coef(), b.M, 0.0);
  merge_products(out, zero.data(), 1.0, 0.0, drop, false, 0.0, b.M, b.keys(), b.coef());
  out.has_identity = a.has_identity || b.has_identity;
}

void dress_undo(DeviceStore& s, size_t M, size_t logical, const Filter& filt) {
  Workspace& ws = workspace();
  std::swap(s.kbuf, ws.out_keys);
  std::swap(s.cbuf, ws.out_coef);
  s.M = M;
  s.logical = logical;
  s.filt = filt;
  s.meta_valid = false;  // the failed merge overwrote the metadata
}

DressOutcome dress_step(DeviceStore& s, const uint64_t* gen_row, double cs, double sn, double drop,
                        bool want_hist, double eps, const uint64_t* next_row, double theta,
                        bool anti_only) {
  switch (s.B) {
    case 1: return dress_impl<1>(s, gen_row, cs, sn, drop, want_hist, eps, next_row, theta, anti_only);
    case 2: return dress_impl<2>(s, gen_row, cs, sn, drop, want_hist, eps, next_row, theta, anti_only);
    case 4: return dress_impl<4>(s, gen_row, cs, sn, drop, want_hist, eps, next_row, theta, anti_only);
    default: throw std::runtime_error("dress: unsupported block count");
  }
}

// ------------------------------------------------------------ growth split
template <int B>
__global__ void k_growth(const ull* __restrict__ keys, size_t M, Filter filt,
                         const double* __restrict__ coef, Key<B> P, ull* __restrict__ ctr) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  int a = 0, c = 0;
  if (i < M) {
    Key<B> k = load_key<B>(keys, i);
    if (filter_keep(filt, i, coef[i], key_is_identity<B>(k))) {
      a = anticommutes<B>(k, P);
      c = 1 - a;
    }
  }
  a = __reduce_add_sync(0xffffffffu, a);
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0) {
    if (a) atomicAdd(ctr, (ull)a);
    if (c) atomicAdd(ctr + 1, (ull)c);
  }
}

void growth_split(DeviceStore& s, const uint64_t* gen_row, size_t* nc, size_t* na) {
  Workspace& ws = workspace();
  cudaStream_t st = stream();
  ull* ctr = ws.counters.as<ull>(16);
  IQCC_CUDA(cudaMemsetAsync(ctr, 0, 2 * sizeof(ull), st));
  const unsigned grid = (unsigned)std::max<size_t>(1, (s.M + 255) / 256);
  {
    KernelScope ks("growth");
    switch (s.B) {
      case 1: k_growth<1><<<grid, 256, 0, st>>>(s.keys(), s.M, s.filt, s.coef(), make_key<1>(gen_row), ctr); break;
      case 2: k_growth<2><<<grid, 256, 0, st>>>(s.keys(), s.M, s.filt, s.coef(), make_key<2>(gen_row), ctr); break;
      default: k_growth<4><<<grid, 256, 0, st>>>(s.keys(), s.M, s.filt, s.coef(), make_key<4>(gen_row), ctr); break;
    }
  }
  ull h[2];
  d2h_small(h, ctr, sizeof(h), st);
  host_sync(st);
  *na = h[0];
  *nc = h[1];
}

// ---------------------------------------------------------- sortless stats
// SortlessStats of sortless_dress (iqcc/dressing.hpp:182-189, 248-305): the
// support buckets (bucket_by_support, :159-177) are the distinct bit
// patterns of the terms on the entangler's support positions (x and z bit
// of every qubit P touches, key bit i = position i, :115-147); a bucket
// anticommutes iff its pattern does (commutation only sees the support), and
// every anticommuting bucket yields one new-term stream when sin != 0.
// Distinct patterns: a device bitmap over all 2^(2w) patterns for w <= 11
// support qubits, else an open-addressing hash set of 64-bit patterns.
struct SupportSpec {
  int npos;
  short word[64];  // device key word of position i
  short bit[64];   // bit index in that word (LSB 0)
};

template <int B>
__device__ __forceinline__ ull support_key(const Key<B>& k, const SupportSpec& sp) {
  ull key = 0;
  for (int i = 0; i < sp.npos; ++i) {
    ull v = 0;
#pragma unroll
    for (int j = 0; j < 2 * B; ++j) v = (j == sp.word[i]) ? k.w[j] : v;
    key |= ((v >> sp.bit[i]) & 1ull) << i;
  }
  return key;
}

template <int B>
__global__ void k_support_bitmap(const ull* __restrict__ keys, const double* __restrict__ coef, size_t M,
                                 Filter filt, SupportSpec sp, unsigned* __restrict__ bitmap) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= M) return;
  const Key<B> k = load_key<B>(keys, i);
  if (!filter_keep(filt, i, coef[i], i == 0 && key_is_identity<B>(k))) return;
  const ull key = support_key<B>(k, sp);
  atomicOr(bitmap + (key >> 5), 1u << (key & 31));
}

template <int B>
__global__ void k_support_hash(const ull* __restrict__ keys, const double* __restrict__ coef, size_t M,
                               Filter filt, SupportSpec sp, ull* __restrict__ table, ull mask,
                               ull anti_mask, ull* __restrict__ ctr) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= M) return;
  const Key<B> k = load_key<B>(keys, i);
  if (!filter_keep(filt, i, coef[i], i == 0 && key_is_identity<B>(k))) return;
  const ull key = support_key<B>(k, sp);
  const ull stored = key + 1;  // 0 marks an empty slot
  ull h = (key * 0x9E3779B97F4A7C15ull) & mask;
  for (;;) {
    const ull prev = atomicCAS(table + h, 0ull, stored);
    if (prev == 0ull) {  // first occurrence of the pattern
      atomicAdd(ctr, 1ull);
      if (__popcll(key & anti_mask) & 1) atomicAdd(ctr + 1, 1ull);
      return;
    }
    if (prev == stored) return;
    h = (h + 1) & mask;
  }
}

__global__ void k_bitmap_count(const unsigned* __restrict__ bitmap, size_t words, ull anti_mask,
                               ull* __restrict__ ctr) {
  const size_t w = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  unsigned n = 0, a = 0;
  if (w < words) {
    unsigned v = bitmap[w];
    n = __popc(v);
    while (v) {
      const int b = __ffs(v) - 1;
      v &= v - 1;
      a += __popcll(((ull)w * 32 + b) & anti_mask) & 1;
    }
  }
  n = __reduce_add_sync(0xffffffffu, n);
  a = __reduce_add_sync(0xffffffffu, a);
  if ((threadIdx.x & 31) == 0 && n) {
    atomicAdd(ctr, (ull)n);
    if (a) atomicAdd(ctr + 1, (ull)a);
  }
}

void sortless_stats(DeviceStore& s, const uint64_t* gen_row, size_t* n_buckets, size_t* n_anti_buckets) {
  // support positions in the reference's order (:115-128): for every qubit j
  // of supp(P) ascending, x bit (position j) then z bit (position n + j)
  const uint32_t B = s.B;
  SupportSpec sp{};
  ull anti = 0;
  std::vector<int> qubits;
  for (uint32_t blk = 0; blk < B; ++blk) {
    const uint64_t b = gen_row[blk] | gen_row[B + blk];
    for (int t = 0; t < 64; ++t)
      if ((b >> t) & 1ull) qubits.push_back((int)(blk * 64 + t));
  }
  if (2 * qubits.size() > 64) throw std::runtime_error("entangler support exceeds 64 bits; not supported");
  sp.npos = (int)(2 * qubits.size());
  for (size_t k = 0; k < qubits.size(); ++k) {
    const int j = qubits[k];
    // device keys are bit-reversed words: qubit j of block j/64 sits at bit 63 - j%64
    sp.word[2 * k] = (short)(j / 64);
    sp.bit[2 * k] = (short)(63 - j % 64);
    sp.word[2 * k + 1] = (short)(B + j / 64);
    sp.bit[2 * k + 1] = (short)(63 - j % 64);
    const bool px = (gen_row[j / 64] >> (j % 64)) & 1ull, pz = (gen_row[B + j / 64] >> (j % 64)) & 1ull;
    // T anticommutes iff sum_j (tx_j pz_j + tz_j px_j) is odd
    if (pz) anti |= 1ull << (2 * k);
    if (px) anti |= 1ull << (2 * k + 1);
  }
  Workspace& ws = workspace();
  cudaStream_t st = stream();
  ull* ctr = ws.counters.as<ull>(16);
  IQCC_CUDA(cudaMemsetAsync(ctr, 0, 2 * sizeof(ull), st));
  const unsigned grid = (unsigned)std::max<size_t>(1, (s.M + 255) / 256);
  KernelScope ks("sortless_stats");
  if (sp.npos <= 22) {
    const size_t words = std::max<size_t>(1, ((size_t)1 << sp.npos) / 32);
    unsigned* bm = ws.misc2.as<unsigned>(words);
    IQCC_CUDA(cudaMemsetAsync(bm, 0, words * sizeof(unsigned), st));
    if (s.M) {
      switch (B) {
        case 1: k_support_bitmap<1><<<grid, 256, 0, st>>>(s.keys(), s.coef(), s.M, s.filt, sp, bm); break;
        case 2: k_support_bitmap<2><<<grid, 256, 0, st>>>(s.keys(), s.coef(), s.M, s.filt, sp, bm); break;
        default: k_support_bitmap<4><<<grid, 256, 0, st>>>(s.keys(), s.coef(), s.M, s.filt, sp, bm); break;
      }
    }
    k_bitmap_count<<<(unsigned)((words + 255) / 256), 256, 0, st>>>(bm, words, anti, ctr);
  } else {
    size_t cap = 1024;
    while (cap < 2 * s.M) cap <<= 1;
    ull* table = ws.misc3.as<ull>(cap);
    IQCC_CUDA(cudaMemsetAsync(table, 0, cap * sizeof(ull), st));
    if (s.M) {
      switch (B) {
        case 1: k_support_hash<1><<<grid, 256, 0, st>>>(s.keys(), s.coef(), s.M, s.filt, sp, table, cap - 1, anti, ctr); break;
        case 2: k_support_hash<2><<<grid, 256, 0, st>>>(s.keys(), s.coef(), s.M, s.filt, sp, table, cap - 1, anti, ctr); break;
        default: k_support_hash<4><<<grid, 256, 0, st>>>(s.keys(), s.coef(), s.M, s.filt, sp, table, cap - 1, anti, ctr); break;
      }
    }
  }
  ull h[2];
  d2h_small(h, ctr, sizeof(h), st);
  host_sync(st);
  *n_buckets = h[0];
  *n_anti_buckets = h[1];
}

}  // namespace iqcc_b200
