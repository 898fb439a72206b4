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
#include <climits>
#include <stdexcept>

#include "engine.cuh"

namespace iqcc_b200 {

constexpr int TT = 256;  // threads per scan tile
constexpr int TI = 8;    // terms per thread
constexpr int TILE = TT * TI;
constexpr int GROUP = 1024;  // tiles per carry group

struct Thr {
  int t[kThrPerChunk];
  int n;     // thresholds in use (2 * levels)
  int nlev;  // levels in this chunk
};

// ---------------------------------------------------------------- classify
template <int B>
__global__ void __launch_bounds__(256) k_classify(const ull* __restrict__ keys, size_t M, Key<B> P,
                                                  const int* __restrict__ lvl, int m,
                                                  short* __restrict__ lcp,
                                                  unsigned char* __restrict__ mbits,
                                                  unsigned* __restrict__ fmask) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  int f = 0;
  if (i < M) {
    Key<B> k = load_key<B>(keys, i);
    int l = -1;
    if (i > 0) l = key_lcp<B>(load_key<B>(keys, i - 1), k);
    lcp[i] = (short)l;
    f = anticommutes<B>(k, P);
    for (int c = 0; c * kLevelsPerChunk < m; ++c) {
      unsigned byte = 0;
      for (int j = 0; j < kLevelsPerChunk && c * kLevelsPerChunk + j < m; ++j)
        byte |= key_bit<B>(k, __ldg(lvl + c * kLevelsPerChunk + j)) << j;
      mbits[(size_t)c * M + i] = (unsigned char)byte;
    }
  }
  unsigned bal = __ballot_sync(0xffffffffu, f);
  const size_t i0 = i - (threadIdx.x & 31);
  if ((threadIdx.x & 31) == 0 && i0 < M) fmask[i0 >> 5] = bal;
}

// ------------------------------------------------------------ tile helpers
struct TileItems {
  int l[TI];
  unsigned bits;  // anticommute bits of the thread's TI terms
};

__device__ __forceinline__ TileItems load_items(const short* __restrict__ lcp,
                                                const unsigned* __restrict__ fmask, size_t M,
                                                size_t first) {
  TileItems it;
#pragma unroll
  for (int k = 0; k < TI; ++k) it.l[k] = (first + k < M) ? (int)lcp[first + k] : INT_MAX;
  it.bits = 0;
  if (first < M) it.bits = (fmask[first >> 5] >> (first & 31)) & 0xFFu;
  return it;
}

template <int NV>
__device__ __forceinline__ void block_excl_max_vec(int (&v)[NV], int* sm /*[TT/32][NV]*/) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int inc[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) inc[j] = warp_inclusive(v[j], OpMax());
  if (lane == 31)
#pragma unroll
    for (int j = 0; j < NV; ++j) sm[warp * NV + j] = inc[j];
  __syncthreads();
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    int base = -1;
    for (int w = 0; w < warp; ++w) base = max(base, sm[w * NV + j]);
    int ex = __shfl_up_sync(0xffffffffu, inc[j], 1);
    if (lane == 0) ex = -1;
    v[j] = max(base, ex);
  }
  __syncthreads();
}

template <int NV>
__device__ __forceinline__ void block_excl_min_rev_vec(int (&v)[NV], int* sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = TT / 32;
  int inc[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) inc[j] = warp_inclusive_rev(v[j], OpMin());
  if (lane == 0)
#pragma unroll
    for (int j = 0; j < NV; ++j) sm[warp * NV + j] = inc[j];
  __syncthreads();
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    int base = INT_MAX;
    for (int w = warp + 1; w < NW; ++w) base = min(base, sm[w * NV + j]);
    int ex = __shfl_down_sync(0xffffffffu, inc[j], 1);
    if (lane == 31) ex = INT_MAX;
    v[j] = min(base, ex);
  }
  __syncthreads();
}

// -------------------------------------------------------- tile aggregates
// fwd_agg[tile][j]: tile-local C of the LAST term with lcp <= thr j (or -1);
// bwd_agg[tile][j]: tile-local C of the FIRST such term (or -1).
__global__ void __launch_bounds__(TT) k_tile_agg(const short* __restrict__ lcp,
                                                 const unsigned* __restrict__ fmask, size_t M,
                                                 Thr thr, int* __restrict__ tile_cnt,
                                                 int* __restrict__ fwd_agg,
                                                 int* __restrict__ bwd_agg) {
  __shared__ int sm[TT / 32 * kThrPerChunk + 8];
  __shared__ int s_total;
  const size_t tile = blockIdx.x;
  const size_t first = tile * TILE + (size_t)threadIdx.x * TI;
  TileItems it = load_items(lcp, fmask, M, first);
  int total;
  int cl = block_exclusive<TT>((int)__popc(it.bits), 0, OpAdd(), sm, &total);
  if (threadIdx.x == 0) s_total = total;
  int fa[kThrPerChunk], ba[kThrPerChunk];
#pragma unroll
  for (int j = 0; j < kThrPerChunk; ++j) {
    fa[j] = -1;
    ba[j] = INT_MAX;
  }
#pragma unroll
  for (int k = 0; k < TI; ++k) {
    int ck = cl + __popc(it.bits & ((1u << k) - 1u));
#pragma unroll
    for (int j = 0; j < kThrPerChunk; ++j)
      if (j < thr.n && it.l[k] <= thr.t[j]) {
        fa[j] = ck;
        ba[j] = min(ba[j], ck);
      }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < kThrPerChunk; ++j) {
    int a = fa[j], b = ba[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a = max(a, __shfl_xor_sync(0xffffffffu, a, o));
      b = min(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    fa[j] = a;
    ba[j] = b;
  }
  __shared__ int sf[TT / 32][kThrPerChunk], sb[TT / 32][kThrPerChunk];
  if (lane == 0)
#pragma unroll
    for (int j = 0; j < kThrPerChunk; ++j) {
      sf[warp][j] = fa[j];
      sb[warp][j] = ba[j];
    }
  __syncthreads();
  if (threadIdx.x < kThrPerChunk) {
    int j = threadIdx.x, a = -1, b = INT_MAX;
    for (int w = 0; w < TT / 32; ++w) {
      a = max(a, sf[w][j]);
      b = min(b, sb[w][j]);
    }
    fwd_agg[tile * kThrPerChunk + j] = a;
    bwd_agg[tile * kThrPerChunk + j] = b == INT_MAX ? -1 : b;
  }
  if (threadIdx.x == 0) tile_cnt[tile] = s_total;
}

// ---------------------------------------------------------- carry scans
// Group level: values relative to the group start.
__global__ void __launch_bounds__(GROUP) k_group_agg(const int* __restrict__ tile_cnt,
                                                     const int* __restrict__ fwd_agg,
                                                     const int* __restrict__ bwd_agg, size_t ntiles,
                                                     int nthr, long long* __restrict__ g_cnt,
                                                     long long* __restrict__ g_fwd,
                                                     long long* __restrict__ g_bwd) {
  __shared__ long long sm[GROUP / 32 + 2];
  const size_t tile = blockIdx.x * (size_t)GROUP + threadIdx.x;
  const bool in = tile < ntiles;
  long long cnt = in ? tile_cnt[tile] : 0;
  long long total;
  long long pfx = block_exclusive<GROUP>(cnt, 0LL, OpAdd(), sm, &total);
  if (threadIdx.x == 0) g_cnt[blockIdx.x] = total;
  for (int j = 0; j < nthr; ++j) {
    long long f = -1, b = LLONG_MAX;
    if (in) {
      int fv = fwd_agg[tile * kThrPerChunk + j], bv = bwd_agg[tile * kThrPerChunk + j];
      if (fv >= 0) f = fv + pfx;
      if (bv >= 0) b = bv + pfx;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      f = max(f, __shfl_xor_sync(0xffffffffu, f, o));
      b = min(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    __shared__ long long rf[GROUP / 32], rb[GROUP / 32];
    if ((threadIdx.x & 31) == 0) {
      rf[threadIdx.x >> 5] = f;
      rb[threadIdx.x >> 5] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      long long a = -1, c = LLONG_MAX;
      for (int w = 0; w < GROUP / 32; ++w) {
        a = max(a, rf[w]);
        c = min(c, rb[w]);
      }
      g_fwd[blockIdx.x * kThrPerChunk + j] = a;
      g_bwd[blockIdx.x * kThrPerChunk + j] = c;
    }
    __syncthreads();
  }
}

// Single block over groups (<= 1024 groups = 2^31 terms).
__global__ void __launch_bounds__(1024) k_group_scan(size_t ngroups, int nthr,
                                                     long long* __restrict__ g_cnt,
                                                     long long* __restrict__ g_fwd,
                                                     long long* __restrict__ g_bwd,
                                                     long long* __restrict__ a_total) {
  __shared__ long long sm[1024 / 32 + 2];
  const int g = threadIdx.x;
  const bool in = g < (int)ngroups;
  long long cnt = in ? g_cnt[g] : 0;
  long long total;
  long long pfx = block_exclusive<1024>(cnt, 0LL, OpAdd(), sm, &total);
  for (int j = 0; j < nthr; ++j) {
    long long f = -1, b = LLONG_MAX;
    if (in) {
      long long fv = g_fwd[g * kThrPerChunk + j], bv = g_bwd[g * kThrPerChunk + j];
      if (fv >= 0) f = fv + pfx;
      if (bv != LLONG_MAX) b = bv + pfx;
    }
    long long fe = block_exclusive<1024>(f, -1LL, OpMax(), sm, (long long*)nullptr);
    long long be = block_exclusive_rev<1024>(b, LLONG_MAX, OpMin(), sm);
    if (in) {
      g_fwd[g * kThrPerChunk + j] = fe;  // carry INTO the group (global C)
      g_bwd[g * kThrPerChunk + j] = be;
    }
  }
  if (in) g_cnt[g] = pfx;  // group exclusive prefix
  if (g == 0) *a_total = total;
}

__global__ void __launch_bounds__(GROUP) k_tile_carry(const int* __restrict__ tile_cnt,
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
  __shared__ long long sm[GROUP / 32 + 2];
  const size_t tile = blockIdx.x * (size_t)GROUP + threadIdx.x;
  const bool in = tile < ntiles;
  long long cnt = in ? tile_cnt[tile] : 0;
  long long pfx = block_exclusive<GROUP>(cnt, 0LL, OpAdd(), sm, (long long*)nullptr) + g_pfx[blockIdx.x];
  const long long A = *a_total;
  if (in) tile_pfx[tile] = (int)pfx;
  for (int j = 0; j < nthr; ++j) {
    long long f = -1, b = LLONG_MAX;
    if (in) {
      int fv = fwd_agg[tile * kThrPerChunk + j], bv = bwd_agg[tile * kThrPerChunk + j];
      if (fv >= 0) f = fv + pfx;
      if (bv >= 0) b = bv + pfx;
    }
    long long fe = block_exclusive<GROUP>(f, -1LL, OpMax(), sm, (long long*)nullptr);
    long long be = block_exclusive_rev<GROUP>(b, LLONG_MAX, OpMin(), sm);
    fe = max(fe, g_fwd[blockIdx.x * kThrPerChunk + j]);
    be = min(be, g_bwd[blockIdx.x * kThrPerChunk + j]);
    if (in) {
      fwd_carry[tile * kThrPerChunk + j] = (int)fe;
      bwd_carry[tile * kThrPerChunk + j] = (int)(be == LLONG_MAX ? A : be);
    }
  }
}

// ----------------------------------------------------------------- rank
template <bool FINAL>
__global__ void __launch_bounds__(TT) k_rank(const short* __restrict__ lcp,
                                             const unsigned char* __restrict__ mb,
                                             const unsigned* __restrict__ fmask, size_t M, Thr thr,
                                             const int* __restrict__ tile_pfx,
                                             const int* __restrict__ fwd_carry,
                                             const int* __restrict__ bwd_carry,
                                             int* __restrict__ rdelta, int has_rdelta,
                                             unsigned* __restrict__ inv_perm) {
  __shared__ int sm[(TT / 32) * kThrPerChunk + 8];
  const size_t tile = blockIdx.x;
  const size_t first = tile * TILE + (size_t)threadIdx.x * TI;
  TileItems it = load_items(lcp, fmask, M, first);
  unsigned char mbk[TI];
#pragma unroll
  for (int k = 0; k < TI; ++k) mbk[k] = (first + k < M) ? mb[first + k] : 0;
  int cl = block_exclusive<TT>((int)__popc(it.bits), 0, OpAdd(), sm, (int*)nullptr) + tile_pfx[tile];
  int C[TI], delta[TI];
#pragma unroll
  for (int k = 0; k < TI; ++k) {
    C[k] = cl + __popc(it.bits & ((1u << k) - 1u));
    delta[k] = 0;
  }
  // forward: last boundary at or before the term
  int st[kThrPerChunk];
#pragma unroll
  for (int j = 0; j < kThrPerChunk; ++j) {
    int a = -1;
#pragma unroll
    for (int k = 0; k < TI; ++k)
      if (it.l[k] <= thr.t[j]) a = C[k];
    st[j] = a;
  }
  block_excl_max_vec<kThrPerChunk>(st, sm);
#pragma unroll
  for (int j = 0; j < kThrPerChunk; ++j) st[j] = max(st[j], fwd_carry[tile * kThrPerChunk + j]);
#pragma unroll
  for (int k = 0; k < TI; ++k) {
#pragma unroll
    for (int j = 0; j < kThrPerChunk; ++j)
      if (it.l[k] <= thr.t[j]) st[j] = C[k];
    if ((it.bits >> k) & 1u) {
#pragma unroll
      for (int lv = 0; lv < kLevelsPerChunk; ++lv)
        if (lv < thr.nlev && ((mbk[k] >> lv) & 1u)) delta[k] -= st[2 * lv + 1] - st[2 * lv];
    }
  }
  // backward: first boundary strictly after the term
#pragma unroll
  for (int j = 0; j < kThrPerChunk; ++j) {
    int b = INT_MAX;
#pragma unroll
    for (int k = TI - 1; k >= 0; --k)
      if (it.l[k] <= thr.t[j]) b = C[k];
    st[j] = b;
  }
  block_excl_min_rev_vec<kThrPerChunk>(st, sm);
#pragma unroll
  for (int j = 0; j < kThrPerChunk; ++j) st[j] = min(st[j], bwd_carry[tile * kThrPerChunk + j]);
#pragma unroll
  for (int k = TI - 1; k >= 0; --k) {
    if ((it.bits >> k) & 1u) {
#pragma unroll
      for (int lv = 0; lv < kLevelsPerChunk; ++lv)
        if (lv < thr.nlev && !((mbk[k] >> lv) & 1u)) delta[k] += st[2 * lv] - st[2 * lv + 1];
    }
#pragma unroll
    for (int j = 0; j < kThrPerChunk; ++j)
      if (it.l[k] <= thr.t[j]) st[j] = C[k];
  }
#pragma unroll
  for (int k = 0; k < TI; ++k) {
    if (!((it.bits >> k) & 1u)) continue;
    const size_t g = first + k;
    int d = delta[k] + (has_rdelta ? rdelta[g] : 0);
    if (FINAL)
      inv_perm[C[k] + d] = (unsigned)g;
    else
      rdelta[g] = d;
  }
}

// ------------------------------------------------------------- partition
template <int B>
__device__ __forceinline__ Key<B> q_key(const ull* __restrict__ keys,
                                        const unsigned* __restrict__ inv_perm, size_t j,
                                        const Key<B>& P) {
  return key_xor<B>(load_key<B>(keys, inv_perm[j]), P);
}

template <int B>
__global__ void k_partition(const ull* __restrict__ keys, const unsigned* __restrict__ inv_perm,
                            size_t nS, size_t nQ, Key<B> P, size_t tile_items, size_t ntiles,
                            ull* __restrict__ part_a, ull* __restrict__ part_b) {
  const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (t > ntiles) return;
  const size_t d = min(t * tile_items, nS + nQ);
  size_t lo = d > nQ ? d - nQ : 0, hi = min(d, nS);
  while (lo < hi) {
    size_t mid = (lo + hi) >> 1;
    if (key_cmp<B>(load_key<B>(keys, mid), q_key<B>(keys, inv_perm, d - 1 - mid, P)) <= 0)
      lo = mid + 1;
    else
      hi = mid;
  }
  size_t a = lo, b = d - lo;
  // never split an equal (survivor, product) pair across tiles
  if (a > 0 && b < nQ && key_cmp<B>(load_key<B>(keys, a - 1), q_key<B>(keys, inv_perm, b, P)) == 0)
    --a;
  part_a[t] = a;
  part_b[t] = b;
}

// ----------------------------------------------------------------- merge
template <int B>
struct MergeSmem {
  static constexpr size_t bytes(int cap, int nt) {
    return (size_t)cap * (16 * B + 8 + 1) + 2 * nt * sizeof(int) + 4096 * sizeof(unsigned) + 64;
  }
};

template <int B>
__device__ __forceinline__ Key<B> sm_key(const ull* sk, int e) {
  Key<B> k;
#pragma unroll
  for (int w = 0; w < 2 * B; ++w) k.w[w] = sk[(size_t)e * 2 * B + w];
  return k;
}

template <int B, int NT, int IPT>
__global__ void __launch_bounds__(NT) k_merge(
    const ull* __restrict__ keys, const double* __restrict__ coef, Filter filt,
    const unsigned* __restrict__ inv_perm, const ull* __restrict__ part_a,
    const ull* __restrict__ part_b, size_t ntiles, Key<B> P, double cs, double sn, double drop,
    ull* __restrict__ out_keys, double* __restrict__ out_coef, ull* __restrict__ tile_status,
    unsigned* __restrict__ tile_counter, ull* __restrict__ counters, int want_hist, double eps,
    unsigned* __restrict__ hist) {
  constexpr int CAP = NT * IPT + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ull* sk = reinterpret_cast<ull*>(smem_raw);
  double* sv = reinterpret_cast<double*>(sk + (size_t)CAP * 2 * B);
  int* s_ta = reinterpret_cast<int*>(sv + CAP);
  int* s_tb = s_ta + NT;
  unsigned* shist = reinterpret_cast<unsigned*>(s_tb + NT);
  unsigned char* sf = reinterpret_cast<unsigned char*>(shist + 4096);
  __shared__ ull s_tile, s_base;
  __shared__ int scratch[NT / 32 + 2];

  if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
  if (want_hist)
    for (int b = threadIdx.x; b < 4096; b += NT) shist[b] = 0;
  __syncthreads();
  const ull tile = s_tile;
  if (tile >= ntiles) return;
  const size_t a0 = part_a[tile], a1 = part_a[tile + 1];
  const size_t b0 = part_b[tile], b1 = part_b[tile + 1];
  const int nS = (int)(a1 - a0), nQ = (int)(b1 - b0), n = nS + nQ;

  for (int e = threadIdx.x; e < nS; e += NT) {
    const size_t i = a0 + e;
    Key<B> k = load_key<B>(keys, i);
    const double c = __ldg(coef + i);
    const bool id = key_is_identity<B>(k);
    const double v = anticommutes<B>(k, P) ? __dmul_rn(c, cs) : c;
#pragma unroll
    for (int w = 0; w < 2 * B; ++w) sk[(size_t)e * 2 * B + w] = k.w[w];
    sv[e] = v;
    sf[e] = (unsigned char)((filter_keep(filt, i, c, id) ? 1 : 0) | (id ? 2 : 0));
  }
  for (int e = threadIdx.x; e < nQ; e += NT) {
    const size_t src = __ldg(inv_perm + b0 + e);
    Key<B> k = load_key<B>(keys, src);
    const double c = __ldg(coef + src);
    const double pr = __dmul_rn(c, sn);
    const double v = product_phase<B>(k, P) == 1 ? pr : -pr;
    Key<B> q = key_xor<B>(k, P);
    const int e2 = nS + e;
#pragma unroll
    for (int w = 0; w < 2 * B; ++w) sk[(size_t)e2 * 2 * B + w] = q.w[w];
    sv[e2] = v;
    sf[e2] = (unsigned char)(filter_keep(filt, src, c, false) ? 1 : 0);
  }
  __syncthreads();

  // per-thread merge-path split inside the tile (pairs never split)
  {
    const int d = min((int)threadIdx.x * IPT, n);
    int lo = max(0, d - nQ), hi = min(d, nS);
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (key_cmp<B>(sm_key<B>(sk, mid), sm_key<B>(sk, nS + d - 1 - mid)) <= 0)
        lo = mid + 1;
      else
        hi = mid;
    }
    int a = lo, b = d - lo;
    if (a > 0 && b < nQ && key_cmp<B>(sm_key<B>(sk, a - 1), sm_key<B>(sk, nS + b)) == 0) --a;
    s_ta[threadIdx.x] = a;
    s_tb[threadIdx.x] = b;
  }
  __syncthreads();
  const int ia0 = s_ta[threadIdx.x], ib0 = s_tb[threadIdx.x];
  const int ia1 = threadIdx.x + 1 < NT ? s_ta[threadIdx.x + 1] : nS;
  const int ib1 = threadIdx.x + 1 < NT ? s_tb[threadIdx.x + 1] : nQ;

  // walk: calls emit(entry index for the key, value) for every surviving output
  auto walk = [&](auto&& emit) {
    int i = ia0, j = ib0;
    while (i < ia1 || j < ib1) {
      int c;
      if (j >= ib1)
        c = -1;
      else if (i >= ia1)
        c = 1;
      else
        c = key_cmp<B>(sm_key<B>(sk, i), sm_key<B>(sk, nS + j));
      if (c < 0) {
        const unsigned char f = sf[i];
        if ((f & 1) && keep_term(sv[i], f & 2, drop)) emit(i, sv[i], (f & 2) != 0);
        ++i;
      } else if (c > 0) {
        const unsigned char f = sf[nS + j];
        if ((f & 1) && keep_term(sv[nS + j], false, drop)) emit(nS + j, sv[nS + j], false);
        ++j;
      } else {
        const unsigned char fs = sf[i], fq = sf[nS + j];
        const bool ps = fs & 1, pq = fq & 1;
        if (ps || pq) {
          double v = ps && pq ? __dadd_rn(sv[i], sv[nS + j]) : (ps ? sv[i] : sv[nS + j]);
          if (keep_term(v, fs & 2, drop)) emit(i, v, (fs & 2) != 0);
        }
        ++i;
        ++j;
      }
    }
  };

  int cnt = 0;
  walk([&](int, double, bool) { ++cnt; });
  int total;
  const int excl = block_exclusive<NT>(cnt, 0, OpAdd(), scratch, &total);
  if (threadIdx.x == 0) {
    s_base = lookback_exclusive(tile_status, tile, (ull)total);
    if (tile == ntiles - 1) counters[0] = s_base + total;
  }
  __syncthreads();
  size_t pos = s_base + excl;
  int n_eps = 0;
  walk([&](int e, double v, bool id) {
    Key<B> k = sm_key<B>(sk, e);
    store_key<B>(out_keys, pos, k);
    out_coef[pos] = v;
    ++pos;
    if (want_hist) {
      const double a = fabs(v);
      if (id || a >= eps) ++n_eps;
      if (!id && a >= eps) atomicAdd(shist + (unsigned)(__double_as_longlong(a) >> 51), 1u);
    }
  });
  if (want_hist) {
    int tot_eps;
    block_exclusive<NT>(n_eps, 0, OpAdd(), scratch, &tot_eps);
    if (threadIdx.x == 0 && tot_eps) atomicAdd(counters + 1, (ull)tot_eps);
    __syncthreads();
    for (int b = threadIdx.x; b < 4096; b += NT)
      if (shist[b]) atomicAdd(hist + b, shist[b]);
  }
}

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
  std::vector<int> pos;
  for (int w = 0; w < 2 * B; ++w)
    for (int b = 63; b >= 0; --b)
      if ((P.w[w] >> b) & 1ull) pos.push_back(64 * w + (63 - b));
  return pos;  // ascending canonical positions
}

template <int B>
constexpr int merge_threads() { return B >= 4 ? 128 : 256; }

template <int B>
DressOutcome dress_impl(DeviceStore& s, const uint64_t* gen_row, double cs, double sn, double drop,
                        bool want_hist, double eps) {
  Workspace& ws = workspace();
  cudaStream_t st = stream();
  const size_t M = s.M;
  const Key<B> P = make_key<B>(gen_row);
  DressOutcome out;
  size_t A = 0;
  unsigned* inv_perm = nullptr;
  if (sn != 0.0 && M > 0) {
    const std::vector<int> pos = level_positions<B>(P);
    const int m = (int)pos.size();
    const int nch = (m + kLevelsPerChunk - 1) / kLevelsPerChunk;
    int* d_lvl = ws.levels.as<int>(m);
    IQCC_CUDA(cudaMemcpyAsync(d_lvl, pos.data(), m * sizeof(int), cudaMemcpyHostToDevice, st));
    short* lcp = ws.lcp.as<short>(M);
    unsigned char* mb = ws.mbits.as<unsigned char>((size_t)nch * M);
    unsigned* fmask = ws.fmask.as<unsigned>((M + 31) / 32);
    {
      KernelScope ks("classify");
      k_classify<B><<<(unsigned)((M + 255) / 256), 256, 0, st>>>(s.keys(), M, P, d_lvl, m, lcp, mb,
                                                                  fmask);
    }
    const size_t ntiles = (M + TILE - 1) / TILE;
    const size_t ngroups = (ntiles + GROUP - 1) / GROUP;
    if (ngroups > 1024) throw std::runtime_error("dress: more than 2^31 terms on one device");
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
    inv_perm = ws.inv_perm.as<unsigned>(M);
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
      {
        KernelScope ks("rank");
        k_tile_agg<<<(unsigned)ntiles, TT, 0, st>>>(lcp, fmask, M, thr, tile_cnt, fwd_agg, bwd_agg);
        k_group_agg<<<(unsigned)ngroups, GROUP, 0, st>>>(tile_cnt, fwd_agg, bwd_agg, ntiles, thr.n,
                                                         g_cnt, g_fwd, g_bwd);
        k_group_scan<<<1, 1024, 0, st>>>(ngroups, thr.n, g_cnt, g_fwd, g_bwd, a_total);
        k_tile_carry<<<(unsigned)ngroups, GROUP, 0, st>>>(tile_cnt, fwd_agg, bwd_agg, ntiles, thr.n,
                                                          g_cnt, g_fwd, g_bwd, a_total, tile_pfx,
                                                          fwd_carry, bwd_carry);
        if (c == nch - 1)
          k_rank<true><<<(unsigned)ntiles, TT, 0, st>>>(lcp, mb + (size_t)c * M, fmask, M, thr,
                                                        tile_pfx, fwd_carry, bwd_carry, rdelta,
                                                        c > 0, inv_perm);
        else
          k_rank<false><<<(unsigned)ntiles, TT, 0, st>>>(lcp, mb + (size_t)c * M, fmask, M, thr,
                                                         tile_pfx, fwd_carry, bwd_carry, rdelta,
                                                         c > 0, inv_perm);
        count_launch("rank");
        count_launch("rank");
        count_launch("rank");
        count_launch("rank");
      }
    }
    long long a_host = 0;
    IQCC_CUDA(cudaMemcpyAsync(&a_host, a_total, sizeof(long long), cudaMemcpyDeviceToHost, st));
    IQCC_CUDA(cudaStreamSynchronize(st));
    A = (size_t)a_host;
  }
  out.n_anticommuting = A;

  constexpr int NT = merge_threads<B>(), IPT = 8, TILEM = NT * IPT;
  const size_t total = M + A;
  const size_t ntm = std::max<size_t>(1, (total + TILEM - 1) / TILEM);
  ull* pa = ws.part_a.as<ull>(ntm + 1);
  ull* pb = ws.part_b.as<ull>(ntm + 1);
  {
    KernelScope ks("partition");
    k_partition<B><<<(unsigned)((ntm + 1 + 255) / 256), 256, 0, st>>>(s.keys(), inv_perm, M, A, P,
                                                                      TILEM, ntm, pa, pb);
  }
  ull* out_keys = ws.out_keys.as<ull>(std::max<size_t>(total, 1) * 2 * B);
  double* out_coef = ws.out_coef.as<double>(std::max<size_t>(total, 1));
  ull* tstat = ws.tile_status.as<ull>(ntm + 1);
  ull* ctr = ws.counters.as<ull>(8);
  unsigned* hist = ws.hist.as<unsigned>(4096);
  IQCC_CUDA(cudaMemsetAsync(tstat, 0, (ntm + 1) * sizeof(ull), st));
  IQCC_CUDA(cudaMemsetAsync(ctr, 0, 8 * sizeof(ull), st));
  if (want_hist) IQCC_CUDA(cudaMemsetAsync(hist, 0, 4096 * sizeof(unsigned), st));
  unsigned* tile_counter = reinterpret_cast<unsigned*>(ctr + 4);
  const size_t smem = MergeSmem<B>::bytes(TILEM + 1, NT);
  static bool attr = false;
  if (!attr) {
    IQCC_CUDA(cudaFuncSetAttribute(k_merge<B, NT, IPT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    attr = true;
  }
  {
    KernelScope ks("merge");
    k_merge<B, NT, IPT><<<(unsigned)ntm, NT, smem, st>>>(
        s.keys(), s.coef(), s.filt, inv_perm, pa, pb, ntm, P, cs, sn, drop, out_keys, out_coef,
        tstat, tile_counter, ctr, want_hist ? 1 : 0, eps, hist);
  }
  ull hc[2] = {0, 0};
  IQCC_CUDA(cudaMemcpyAsync(hc, ctr, 2 * sizeof(ull), cudaMemcpyDeviceToHost, st));
  IQCC_CUDA(cudaStreamSynchronize(st));
  std::swap(s.kbuf, ws.out_keys);
  std::swap(s.cbuf, ws.out_coef);
  s.M = hc[0];
  s.filt = Filter{};
  s.logical = s.M;
  out.count_eps = hc[1];
  return out;
}

}  // namespace

DressOutcome dress_step(DeviceStore& s, const uint64_t* gen_row, double cs, double sn, double drop,
                        bool want_hist, double eps) {
  switch (s.B) {
    case 1: return dress_impl<1>(s, gen_row, cs, sn, drop, want_hist, eps);
    case 2: return dress_impl<2>(s, gen_row, cs, sn, drop, want_hist, eps);
    case 4: return dress_impl<4>(s, gen_row, cs, sn, drop, want_hist, eps);
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
  ull* ctr = ws.counters.as<ull>(8);
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
  IQCC_CUDA(cudaMemcpyAsync(h, ctr, sizeof(h), cudaMemcpyDeviceToHost, st));
  IQCC_CUDA(cudaStreamSynchronize(st));
  *na = h[0];
  *nc = h[1];
}

}  // namespace iqcc_b200
