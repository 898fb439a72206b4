// qmf.cu — QMF energy / gradient, DIS screening, partition-bit selection.
//
// * expect (iqcc/qmf.hpp:67-90): one term per thread; the Bloch factor
//   product runs over the support in ascending qubit order exactly as
//   expect_word, so every per-term value c*<W> is bit-identical to the
//   reference; only the summation order differs (compensated, fixed tree).
// * qmf_energy_gradient (iqcc/qmf.hpp:94-148): one term per warp, lanes own
//   qubit ranges; prefix/suffix factor products by warp scans; each warp
//   accumulates into its own shared gradient (deterministic order).
// * gradient / group_gradient (iqcc/dis.hpp:39-52, 121-132): one candidate
//   per thread summing its terms sequentially in canonical order, so the
//   value is bit-identical to the reference (ranking ties resolve alike).
// * dis_candidates (iqcc/dis.hpp:140-191): flip groups = runs of equal x
//   planes of the sorted store; odd-Y enumeration per group on the device.
// * choose_partition_bits (iqcc/partition.hpp:52-108): per round, counts of
//   set bits per (position, class) by shared-memory atomics.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "engine.cuh"

namespace iqcc_b200 {

// ------------------------------------------------------------------ expect
// factor table layout in shared memory: [q][3] = (X, Z, Y)
__device__ __forceinline__ int letter_index(unsigned x, unsigned z) { return x ? (z ? 2 : 0) : 1; }

template <int B>
__device__ __forceinline__ double word_expect(const Key<B>& k, const double* __restrict__ tab) {
  double val = 1.0;
#pragma unroll
  for (int w = 0; w < B; ++w) {
    ull s = k.w[w] | k.w[B + w];
    while (s) {  // ascending qubit = descending bit of the reversed word
      const int lz = __clzll((long long)s);
      const int bit = 63 - lz;
      const int q = 64 * w + lz;
      const unsigned x = (unsigned)(k.w[w] >> bit) & 1u, z = (unsigned)(k.w[B + w] >> bit) & 1u;
      val = __dmul_rn(val, tab[3 * q + letter_index(x, z)]);
      s &= ~(1ull << bit);
    }
  }
  return val;
}

struct TwoSum {  // Neumaier compensated accumulator
  double s = 0.0, c = 0.0;
  __device__ __forceinline__ void add(double x) {
    const double t = __dadd_rn(s, x);
    if (fabs(s) >= fabs(x))
      c = __dadd_rn(c, __dadd_rn(__dsub_rn(s, t), x));
    else
      c = __dadd_rn(c, __dadd_rn(__dsub_rn(x, t), s));
    s = t;
  }
  __device__ __forceinline__ void merge(const TwoSum& o) {
    add(o.s);
    c = __dadd_rn(c, o.c);
  }
};

template <int B>
__global__ void __launch_bounds__(256) k_expect(const ull* __restrict__ keys,
                                                const double* __restrict__ coef, size_t M,
                                                Filter filt, const double* __restrict__ tab_g,
                                                int nq, double* __restrict__ partial) {
  extern __shared__ double tab[];
  __shared__ double rs[256], rc[256];
  for (int i = threadIdx.x; i < 3 * nq; i += blockDim.x) tab[i] = tab_g[i];
  __syncthreads();
  TwoSum acc;
  const size_t per = (M + gridDim.x - 1) / gridDim.x;
  const size_t lo = blockIdx.x * per, hi = min(M, lo + per);
  for (size_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const Key<B> k = load_key<B>(keys, i);
    const double c = coef[i];
    if (!filter_keep(filt, i, c, i == 0 && key_is_identity<B>(k))) continue;
    acc.add(__dmul_rn(c, word_expect<B>(k, tab)));
  }
  rs[threadIdx.x] = acc.s;
  rc[threadIdx.x] = acc.c;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {  // fixed tree: deterministic
    if (threadIdx.x < o) {
      TwoSum a{rs[threadIdx.x], rc[threadIdx.x]}, b{rs[threadIdx.x + o], rc[threadIdx.x + o]};
      a.merge(b);
      rs[threadIdx.x] = a.s;
      rc[threadIdx.x] = a.c;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    partial[2 * blockIdx.x] = rs[0];
    partial[2 * blockIdx.x + 1] = rc[0];
  }
}

static std::vector<double> fetch(const double* d, size_t n) {
  std::vector<double> h(n);
  IQCC_CUDA(cudaMemcpyAsync(h.data(), d, n * sizeof(double), cudaMemcpyDeviceToHost, stream()));
  IQCC_CUDA(cudaStreamSynchronize(stream()));
  return h;
}

static double host_sum_pairs(const std::vector<double>& p) {
  double s = 0.0, c = 0.0;
  for (size_t i = 0; i < p.size(); i += 2) {
    const double x = p[i];
    const double t = s + x;
    c += std::fabs(s) >= std::fabs(x) ? (s - t) + x : (x - t) + s;
    s = t;
    c += p[i + 1];
  }
  return s + c;
}

double expect_store(DeviceStore& s, const double* factors) {
  Workspace& ws = workspace();
  cudaStream_t st = stream();
  if (s.logical == 0) return 0.0;
  const int nq = (int)s.n_qubits;
  double* tab = ws.tables.as<double>(3 * (size_t)std::max(nq, 1));
  IQCC_CUDA(cudaMemcpyAsync(tab, factors, 3 * nq * sizeof(double), cudaMemcpyHostToDevice, st));
  const unsigned grid = (unsigned)std::min<size_t>(1184, std::max<size_t>(1, (s.M + 1023) / 1024));
  double* part = ws.partials.as<double>(2 * grid);
  const size_t smem = 3 * (size_t)std::max(nq, 1) * sizeof(double);
  {
    KernelScope ks("expect");
    switch (s.B) {
      case 1: k_expect<1><<<grid, 256, smem, st>>>(s.keys(), s.coef(), s.M, s.filt, tab, nq, part); break;
      case 2: k_expect<2><<<grid, 256, smem, st>>>(s.keys(), s.coef(), s.M, s.filt, tab, nq, part); break;
      default: k_expect<4><<<grid, 256, smem, st>>>(s.keys(), s.coef(), s.M, s.filt, tab, nq, part); break;
    }
  }
  return host_sum_pairs(fetch(part, 2 * grid));
}

// -------------------------------------------------------- QMF gradient
// One term per warp.  Lane L owns qubits [QPL*L, QPL*L+QPL).  Factors of
// identity positions are 1.0 (exact), so the products equal the support-only
// products up to association; rest_k = prefix_k * suffix_k.
template <int B>
__global__ void __launch_bounds__(256) k_qmf_grad(const ull* __restrict__ keys,
                                                  const double* __restrict__ coef, size_t M,
                                                  Filter filt, const double* __restrict__ tab_g,
                                                  const double* __restrict__ der_g, int nq,
                                                  double* __restrict__ partial) {
  constexpr int QPL = 2 * B;  // qubits per lane: 64*B / 32
  extern __shared__ double sm[];
  double* tab = sm;                  // [nq][3]
  double* der = tab + 3 * nq;        // [nq][6]
  double* wgrad = der + 6 * nq;      // [8 warps][2 nq]
  __shared__ double es[8], ec[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 3 * nq; i += blockDim.x) tab[i] = tab_g[i];
  for (int i = threadIdx.x; i < 6 * nq; i += blockDim.x) der[i] = der_g[i];
  for (int i = threadIdx.x; i < 16 * nq; i += blockDim.x) wgrad[i] = 0.0;
  __syncthreads();
  double* mg = wgrad + (size_t)warp * 2 * nq;
  TwoSum e;
  const size_t nw = (size_t)gridDim.x * 8;
  for (size_t i = blockIdx.x * (size_t)8 + warp; i < M; i += nw) {
    const Key<B> k = load_key<B>(keys, i);
    const double c = coef[i];
    if (!filter_keep(filt, i, c, i == 0 && key_is_identity<B>(k))) continue;
    double f[QPL];
    int li[QPL];
    double lp = 1.0;
#pragma unroll
    for (int t = 0; t < QPL; ++t) {
      const int q = QPL * lane + t;
      const int w = q >> 6, bit = 63 - (q & 63);
      ull xw = 0, zw = 0;
#pragma unroll
      for (int j = 0; j < B; ++j) {
        xw = (j == w) ? k.w[j] : xw;
        zw = (j == w) ? k.w[B + j] : zw;
      }
      const unsigned x = (unsigned)(xw >> bit) & 1u, z = (unsigned)(zw >> bit) & 1u;
      li[t] = (x | z) && q < nq ? letter_index(x, z) : -1;
      f[t] = li[t] >= 0 ? tab[3 * q + li[t]] : 1.0;
      lp = __dmul_rn(lp, f[t]);
    }
    // exclusive prefix / suffix of the lane products across the warp
    double pre = lp, suf = lp;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double a = __shfl_up_sync(0xffffffffu, pre, o);
      if (lane >= o) pre = __dmul_rn(a, pre);
      const double b = __shfl_down_sync(0xffffffffu, suf, o);
      if (lane + o < 32) suf = __dmul_rn(suf, b);
    }
    const double total = __shfl_sync(0xffffffffu, pre, 31);
    double pex = __shfl_up_sync(0xffffffffu, pre, 1);
    double sex = __shfl_down_sync(0xffffffffu, suf, 1);
    if (lane == 0) pex = 1.0;
    if (lane == 31) sex = 1.0;
    if (lane == 0) e.add(__dmul_rn(c, total));
    double run = pex;  // product of factors before position t
#pragma unroll
    for (int t = 0; t < QPL; ++t) {
      double after = sex;  // product of factors after position t
#pragma unroll
      for (int u = QPL - 1; u > t; --u) after = __dmul_rn(f[u], after);
      if (li[t] >= 0) {
        const int q = QPL * lane + t;
        const double rest = __dmul_rn(run, after);
        const double cr = __dmul_rn(c, rest);
        mg[q] = __dadd_rn(mg[q], __dmul_rn(cr, der[6 * q + 2 * li[t]]));
        mg[nq + q] = __dadd_rn(mg[nq + q], __dmul_rn(cr, der[6 * q + 2 * li[t] + 1]));
      }
      run = __dmul_rn(run, f[t]);
    }
  }
  if (lane == 0) {
    es[warp] = e.s;
    ec[warp] = e.c;
  }
  __syncthreads();
  double* out = partial + (size_t)blockIdx.x * (2 * nq + 2);
  for (int j = threadIdx.x; j < 2 * nq; j += blockDim.x) {
    double acc = 0.0;
    for (int w = 0; w < 8; ++w) acc = __dadd_rn(acc, wgrad[(size_t)w * 2 * nq + j]);
    out[j] = acc;
  }
  if (threadIdx.x == 0) {
    TwoSum t;
    for (int w = 0; w < 8; ++w) t.merge(TwoSum{es[w], ec[w]});
    out[2 * nq] = t.s;
    out[2 * nq + 1] = t.c;
  }
}

double qmf_grad_store(DeviceStore& s, const double* factors, const double* derivs, double* grad) {
  Workspace& ws = workspace();
  cudaStream_t st = stream();
  const int nq = (int)s.n_qubits;
  std::fill(grad, grad + 2 * nq, 0.0);
  if (s.logical == 0) return 0.0;
  double* tab = ws.tables.as<double>(9 * (size_t)nq);
  IQCC_CUDA(cudaMemcpyAsync(tab, factors, 3 * nq * sizeof(double), cudaMemcpyHostToDevice, st));
  IQCC_CUDA(cudaMemcpyAsync(tab + 3 * nq, derivs, 6 * nq * sizeof(double), cudaMemcpyHostToDevice, st));
  const unsigned grid = (unsigned)std::min<size_t>(592, std::max<size_t>(1, (s.M + 63) / 64));
  double* part = ws.grad_part.as<double>((size_t)grid * (2 * nq + 2));
  const size_t smem = (size_t)(3 + 6 + 16) * nq * sizeof(double);
  {
    KernelScope ks("qmf_grad");
    switch (s.B) {
      case 1:
        IQCC_CUDA(cudaFuncSetAttribute(k_qmf_grad<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_qmf_grad<1><<<grid, 256, smem, st>>>(s.keys(), s.coef(), s.M, s.filt, tab, tab + 3 * nq, nq, part);
        break;
      case 2:
        IQCC_CUDA(cudaFuncSetAttribute(k_qmf_grad<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_qmf_grad<2><<<grid, 256, smem, st>>>(s.keys(), s.coef(), s.M, s.filt, tab, tab + 3 * nq, nq, part);
        break;
      default:
        IQCC_CUDA(cudaFuncSetAttribute(k_qmf_grad<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_qmf_grad<4><<<grid, 256, smem, st>>>(s.keys(), s.coef(), s.M, s.filt, tab, tab + 3 * nq, nq, part);
        break;
    }
  }
  std::vector<double> h = fetch(part, (size_t)grid * (2 * nq + 2));
  double es = 0.0, ec = 0.0;
  for (unsigned b = 0; b < grid; ++b) {
    const double* p = h.data() + (size_t)b * (2 * nq + 2);
    for (int j = 0; j < 2 * nq; ++j) grad[j] += p[j];
    const double x = p[2 * nq];
    const double t = es + x;
    ec += std::fabs(es) >= std::fabs(x) ? (es - t) + x : (x - t) + es;
    es = t;
    ec += p[2 * nq + 1];
  }
  return es + ec;
}

// --------------------------------------------------------------- DIS
// g(P) = sum_k Im(c_k i^t) <omega|T_k P|omega>, skipping Im == 0; for real
// c_k, Im(c i^t) = c (t=1), -c (t=3), 0 otherwise (even t: commuting).
// One candidate per thread; the term range [lo, hi) is streamed through
// shared memory tiles shared by the whole block.
template <int B>
__global__ void __launch_bounds__(128) k_dis_full(const ull* __restrict__ keys,
                                                  const double* __restrict__ coef, size_t M,
                                                  Filter filt, const double* __restrict__ tab_g,
                                                  int nq, const ull* __restrict__ cands, size_t K,
                                                  double* __restrict__ g_out) {
  constexpr int TT = 128;
  extern __shared__ double dsm[];
  double* tab = dsm;
  ull* tk = reinterpret_cast<ull*>(tab + 3 * nq);
  double* tc = reinterpret_cast<double*>(tk + (size_t)TT * 2 * B);
  for (int i = threadIdx.x; i < 3 * nq; i += blockDim.x) tab[i] = tab_g[i];
  const size_t cid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  Key<B> P;
  if (cid < K) P = load_key<B>(cands, cid);
  double g = 0.0;
  for (size_t base = 0; base < M; base += TT) {
    __syncthreads();
    const size_t i = base + threadIdx.x;
    if (i < M) {
      const Key<B> k = load_key<B>(keys, i);
      double c = coef[i];
      if (!filter_keep(filt, i, c, i == 0 && key_is_identity<B>(k))) c = 0.0;  // Im(0) == 0: skipped
#pragma unroll
      for (int w = 0; w < 2 * B; ++w) tk[(size_t)threadIdx.x * 2 * B + w] = k.w[w];
      tc[threadIdx.x] = c;
    }
    __syncthreads();
    if (cid >= K) continue;
    const int n = (int)min((size_t)TT, M - base);
    for (int j = 0; j < n; ++j) {
      Key<B> k;
#pragma unroll
      for (int w = 0; w < 2 * B; ++w) k.w[w] = tk[(size_t)j * 2 * B + w];
      const double c = tc[j];
      if (c == 0.0 || !anticommutes<B>(k, P)) continue;
      const double im = product_phase<B>(k, P) == 1 ? c : -c;
      g = __dadd_rn(g, __dmul_rn(im, word_expect<B>(key_xor<B>(k, P), tab)));
    }
  }
  if (cid < K) g_out[cid] = g;
}

// Candidate restricted to its flip group [lo, hi) (group_gradient).
template <int B>
__global__ void k_dis_group(const ull* __restrict__ keys, const double* __restrict__ coef,
                            Filter filt, const double* __restrict__ tab_g, int nq,
                            const ull* __restrict__ cands, const ull* __restrict__ range,
                            size_t K, double* __restrict__ g_out) {
  extern __shared__ double tab[];
  for (int i = threadIdx.x; i < 3 * nq; i += blockDim.x) tab[i] = tab_g[i];
  __syncthreads();
  const size_t cid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (cid >= K) return;
  const Key<B> P = load_key<B>(cands, cid);
  const size_t lo = range[2 * cid], hi = range[2 * cid + 1];
  double g = 0.0;
  for (size_t i = lo; i < hi; ++i) {
    const Key<B> k = load_key<B>(keys, i);
    const double c = coef[i];
    if (!filter_keep(filt, i, c, i == 0 && key_is_identity<B>(k)) || c == 0.0) continue;
    if (!anticommutes<B>(k, P)) continue;
    const double im = product_phase<B>(k, P) == 1 ? c : -c;
    g = __dadd_rn(g, __dmul_rn(im, word_expect<B>(key_xor<B>(k, P), tab)));
  }
  g_out[cid] = g;
}

// Flip-group range of each candidate: keys with the candidate's x plane form
// one contiguous run [lower_bound(x,0), lower_bound(x+1 ...)) of the sorted store.
template <int B>
__device__ __forceinline__ int cmp_x(const Key<B>& a, const Key<B>& b) {
#pragma unroll
  for (int w = 0; w < B; ++w)
    if (a.w[w] != b.w[w]) return a.w[w] < b.w[w] ? -1 : 1;
  return 0;
}

template <int B>
__global__ void k_group_range(const ull* __restrict__ keys, size_t M, const ull* __restrict__ cands,
                              size_t K, ull* __restrict__ range) {
  const size_t cid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (cid >= K) return;
  const Key<B> P = load_key<B>(cands, cid);
  size_t lo = 0, hi = M;
  while (lo < hi) {  // first key with x >= P.x
    const size_t mid = (lo + hi) >> 1;
    if (cmp_x<B>(load_key<B>(keys, mid), P) < 0) lo = mid + 1; else hi = mid;
  }
  size_t a = lo;
  hi = M;
  while (lo < hi) {  // first key with x > P.x
    const size_t mid = (lo + hi) >> 1;
    if (cmp_x<B>(load_key<B>(keys, mid), P) <= 0) lo = mid + 1; else hi = mid;
  }
  range[2 * cid] = a;
  range[2 * cid + 1] = lo;
}

template <int B>
static void gradients_impl(DeviceStore& s, const double* factors, const uint64_t* cands_rows,
                           size_t K, bool flip_group_only, double* g) {
  Workspace& ws = workspace();
  cudaStream_t st = stream();
  const int nq = (int)s.n_qubits;
  std::vector<ull> ck(K * 2 * B);
  for (size_t k = 0; k < K; ++k) row_to_device_key(cands_rows + k * 2 * B, B, ck.data() + k * 2 * B);
  ull* dc = ws.misc3.as<ull>(std::max<size_t>(K, 1) * 2 * B + 2 * std::max<size_t>(K, 1));
  ull* rng = dc + std::max<size_t>(K, 1) * 2 * B;
  double* tab = ws.tables.as<double>(3 * (size_t)std::max(nq, 1));
  double* dg = ws.partials.as<double>(std::max<size_t>(K, 1));
  IQCC_CUDA(cudaMemcpyAsync(dc, ck.data(), ck.size() * sizeof(ull), cudaMemcpyHostToDevice, st));
  IQCC_CUDA(cudaMemcpyAsync(tab, factors, 3 * nq * sizeof(double), cudaMemcpyHostToDevice, st));
  if (K == 0) return;
  if (flip_group_only) {
    KernelScope ks("dis_gradient");
    k_group_range<B><<<(unsigned)((K + 127) / 128), 128, 0, st>>>(s.keys(), s.M, dc, K, rng);
    k_dis_group<B><<<(unsigned)((K + 127) / 128), 128, 3 * nq * sizeof(double), st>>>(
        s.keys(), s.coef(), s.filt, tab, nq, dc, rng, K, dg);
    count_launch("dis_gradient");
  } else {
    KernelScope ks("dis_gradient");
    const size_t smem = 3 * nq * sizeof(double) + 128 * (16 * B + 8);
    k_dis_full<B><<<(unsigned)((K + 127) / 128), 128, smem, st>>>(s.keys(), s.coef(), s.M, s.filt, tab,
                                                                    nq, dc, K, dg);
  }
  IQCC_CUDA(cudaMemcpyAsync(g, dg, K * sizeof(double), cudaMemcpyDeviceToHost, st));
  IQCC_CUDA(cudaStreamSynchronize(st));
}

void gradients_store(DeviceStore& s, const double* factors, const uint64_t* cands, size_t K,
                     bool flip_group_only, double* g) {
  switch (s.B) {
    case 1: gradients_impl<1>(s, factors, cands, K, flip_group_only, g); break;
    case 2: gradients_impl<2>(s, factors, cands, K, flip_group_only, g); break;
    default: gradients_impl<4>(s, factors, cands, K, flip_group_only, g); break;
  }
}

// ------------------------------------------------------ DIS screening
// Flip groups (group_by_flip, iqcc/dis.hpp:23-35) are the runs of equal x
// planes of the (materialized) store.
template <int B>
__global__ void k_group_starts(const ull* __restrict__ keys, size_t M, unsigned* __restrict__ flag) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= M) return;
  flag[i] = (i == 0 || cmp_x<B>(load_key<B>(keys, i - 1), load_key<B>(keys, i)) != 0) ? 1u : 0u;
}

// odd_y_candidates (iqcc/dis.hpp:89-116): exhaustive odd-popcount masks in
// increasing order (the j-th is 2j or 2j+1, whichever has odd parity) when
// 2^(w-1) fits the cap, else one single-Y word per flip position.
__host__ __device__ __forceinline__ ull nth_odd_mask(ull j) {
  const ull a = 2 * j;
#if defined(__CUDA_ARCH__)
  return (__popcll((long long)a) & 1) ? a : a + 1;
#else
  return (__builtin_popcountll(a) & 1) ? a : a + 1;
#endif
}

__host__ __device__ __forceinline__ ull odd_y_count(int w, ull cap) {
  if (w == 0) return 0;
  const bool exhaustive = w < 2 || (w <= 63 && (1ull << (w - 1)) <= cap);
  if (exhaustive) {
    const ull all = 1ull << (w - 1);
    return all < cap ? all : cap;
  }
  return (ull)w < cap ? (ull)w : cap;
}

template <int B>
__global__ void k_make_cands(const ull* __restrict__ keys, const ull* __restrict__ gstart,
                             const ull* __restrict__ cstart, size_t ngroups, ull cap,
                             ull* __restrict__ cands, ull* __restrict__ cgroup) {
  const size_t gi = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (gi >= ngroups) return;
  const Key<B> k0 = load_key<B>(keys, gstart[gi]);
  int pos[64 * B];
  int w = 0;
  for (int b = 0; b < B; ++b) {  // flip positions in ascending qubit order
    ull s = k0.w[b];
    while (s) {
      const int lz = __clzll((long long)s);
      pos[w++] = 64 * b + lz;
      s &= ~(1ull << (63 - lz));
    }
  }
  const ull nc = cstart[gi + 1] - cstart[gi];
  const bool exhaustive = w < 2 || (w <= 63 && (1ull << (w - 1)) <= cap);
  for (ull j = 0; j < nc; ++j) {
    const ull ymask = exhaustive ? nth_odd_mask(j) : (1ull << j);
    Key<B> c;
#pragma unroll
    for (int t = 0; t < 2 * B; ++t) c.w[t] = 0;
#pragma unroll
    for (int t = 0; t < B; ++t) c.w[t] = k0.w[t];
    for (int i = 0; i < w; ++i)
      if ((ymask >> i) & 1ull) {
        const int q = pos[i];
        c.w[B + (q >> 6)] |= 1ull << (63 - (q & 63));
      }
    store_key<B>(cands, cstart[gi] + j, c);
    cgroup[cstart[gi] + j] = gi;
  }
}

template <int B>
static size_t dis_impl(DeviceStore& s, const double* factors, bool poles, size_t top_k, double thr,
                       size_t cap, std::vector<uint64_t>& rows_out, std::vector<double>& g_out) {
  store_materialize(s);  // groups are runs of the live terms
  Workspace& ws = workspace();
  cudaStream_t st = stream();
  const size_t M = s.M;
  rows_out.clear();
  g_out.clear();
  if (M == 0) return 0;
  unsigned* flag = ws.fmask.as<unsigned>(M);
  {
    KernelScope ks("dis_groups");
    k_group_starts<B><<<(unsigned)((M + 255) / 256), 256, 0, st>>>(s.keys(), M, flag);
  }
  std::vector<unsigned> hf(M);
  IQCC_CUDA(cudaMemcpyAsync(hf.data(), flag, M * sizeof(unsigned), cudaMemcpyDeviceToHost, st));
  std::vector<ull> hk(M * 2 * B);  // x planes of group heads (host bookkeeping)
  IQCC_CUDA(cudaMemcpyAsync(hk.data(), s.keys(), M * 2 * B * sizeof(ull), cudaMemcpyDeviceToHost, st));
  IQCC_CUDA(cudaStreamSynchronize(st));
  std::vector<ull> gstart, cstart{0};
  for (size_t i = 0; i < M; ++i)
    if (hf[i]) {
      int w = 0;
      for (int b = 0; b < B; ++b) w += __builtin_popcountll(hk[i * 2 * B + b]);
      gstart.push_back(i);
      cstart.push_back(cstart.back() + odd_y_count(w, cap));
    }
  const size_t ng = gstart.size(), K = cstart.back();
  gstart.push_back(M);
  if (K == 0) return 0;
  ull* dgs = ws.misc.as<ull>(2 * (ng + 2));
  ull* dcs = dgs + ng + 1;
  ull* dcand = ws.cand_v.as<ull>(K * 2 * B);
  ull* dgrp = ws.cand_i.as<ull>(K);
  IQCC_CUDA(cudaMemcpyAsync(dgs, gstart.data(), (ng + 1) * sizeof(ull), cudaMemcpyHostToDevice, st));
  IQCC_CUDA(cudaMemcpyAsync(dcs, cstart.data(), (ng + 1) * sizeof(ull), cudaMemcpyHostToDevice, st));
  {
    KernelScope ks("dis_cands");
    k_make_cands<B><<<(unsigned)((ng + 127) / 128), 128, 0, st>>>(s.keys(), dgs, dcs, ng, cap, dcand, dgrp);
  }
  std::vector<ull> cand(K * 2 * B);
  IQCC_CUDA(cudaMemcpyAsync(cand.data(), dcand, K * 2 * B * sizeof(ull), cudaMemcpyDeviceToHost, st));
  IQCC_CUDA(cudaStreamSynchronize(st));
  std::vector<uint64_t> crow(K * 2 * B);
  for (size_t k = 0; k < K; ++k) device_key_to_row(cand.data() + k * 2 * B, B, crow.data() + k * 2 * B);
  std::vector<double> g(K);
  gradients_impl<B>(s, factors, crow.data(), K, poles, g.data());
  // best per group (|g| desc, canonical asc), screen, rank
  struct Pick {
    size_t c;
    double g;
  };
  auto cless = [&](size_t a, size_t b) {
    for (int w = 0; w < 2 * B; ++w) {
      const ull x = cand[a * 2 * B + w], y = cand[b * 2 * B + w];
      if (x != y) return x < y;
    }
    return false;
  };
  std::vector<Pick> picks;
  for (size_t gi = 0; gi < ng; ++gi) {
    size_t best = SIZE_MAX;
    for (size_t c = cstart[gi]; c < cstart[gi + 1]; ++c)
      if (best == SIZE_MAX || std::fabs(g[c]) > std::fabs(g[best]) ||
          (std::fabs(g[c]) == std::fabs(g[best]) && cless(c, best)))
        best = c;
    if (best != SIZE_MAX && std::fabs(g[best]) >= thr) picks.push_back({best, g[best]});
  }
  std::stable_sort(picks.begin(), picks.end(), [&](const Pick& a, const Pick& b) {
    if (std::fabs(a.g) != std::fabs(b.g)) return std::fabs(a.g) > std::fabs(b.g);
    return cless(a.c, b.c);
  });
  (void)top_k;
  rows_out.resize(picks.size() * 2 * B);
  g_out.resize(picks.size());
  for (size_t i = 0; i < picks.size(); ++i) {
    std::copy(crow.begin() + picks[i].c * 2 * B, crow.begin() + (picks[i].c + 1) * 2 * B,
              rows_out.begin() + i * 2 * B);
    g_out[i] = picks[i].g;
  }
  return picks.size();
}

size_t dis_store(DeviceStore& s, const double* factors, bool poles, size_t top_k, double thr,
                 size_t cap, std::vector<uint64_t>& rows_out, std::vector<double>& g_out) {
  switch (s.B) {
    case 1: return dis_impl<1>(s, factors, poles, top_k, thr, cap, rows_out, g_out);
    case 2: return dis_impl<2>(s, factors, poles, top_k, thr, cap, rows_out, g_out);
    default: return dis_impl<4>(s, factors, poles, top_k, thr, cap, rows_out, g_out);
  }
}

// ------------------------------------------------- partition bit choice
// ones[pos][class]: present terms of `class` (key on the chosen bits) with
// bit `pos` set; positions in reference numbering (x: q, z: n + q).
template <int B>
__global__ void __launch_bounds__(256) k_bit_counts(const ull* __restrict__ keys,
                                                    const double* __restrict__ coef, size_t M,
                                                    Filter filt, int nq, const int* __restrict__ chosen,
                                                    int r, unsigned* __restrict__ ones,
                                                    unsigned* __restrict__ cls_cnt) {
  extern __shared__ unsigned sh[];  // [2nq][1<<r] + [1<<r]
  const int ncls = 1 << r, npos = 2 * nq;
  for (int i = threadIdx.x; i < npos * ncls + ncls; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < M; i += (size_t)gridDim.x * blockDim.x) {
    const Key<B> k = load_key<B>(keys, i);
    if (!filter_keep(filt, i, coef[i], i == 0 && key_is_identity<B>(k))) continue;
    int cls = 0;
    for (int b = 0; b < r; ++b) {
      const int p = chosen[b];
      const int q = p < nq ? p : p - nq;
      const int w = (p < nq ? 0 : B) + (q >> 6);
      ull v = 0;
#pragma unroll
      for (int j = 0; j < 2 * B; ++j) v = (j == w) ? k.w[j] : v;
      cls |= (int)((v >> (63 - (q & 63))) & 1ull) << b;
    }
    atomicAdd(sh + npos * ncls + cls, 1u);
#pragma unroll
    for (int w = 0; w < 2 * B; ++w) {
      ull s = k.w[w];
      while (s) {
        const int lz = __clzll((long long)s);
        const int q = 64 * (w % B) + lz;
        const int p = (w < B ? 0 : nq) + q;
        atomicAdd(sh + p * ncls + cls, 1u);
        s &= ~(1ull << (63 - lz));
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < npos * ncls; i += blockDim.x)
    if (sh[i]) atomicAdd(ones + i, sh[i]);
  for (int i = threadIdx.x; i < ncls; i += blockDim.x)
    if (sh[npos * ncls + i]) atomicAdd(cls_cnt + i, sh[npos * ncls + i]);
}

double choose_bits_store(DeviceStore& s, size_t m, size_t* bits_out) {
  const int nq = (int)s.n_qubits, npos = 2 * nq;
  if ((int)m > npos) throw std::invalid_argument("choose_partition_bits: m exceeds representation width");
  Workspace& ws = workspace();
  cudaStream_t st = stream();
  std::vector<int> chosen;
  std::vector<unsigned> final_cnt;
  int* dch = reinterpret_cast<int*>(ws.levels.as<int>(64));
  for (size_t r = 0; r <= m; ++r) {
    const int ncls = 1 << r;
    unsigned* ones = ws.misc2.as<unsigned>((size_t)npos * ncls + ncls);
    unsigned* cls = ones + (size_t)npos * ncls;
    IQCC_CUDA(cudaMemsetAsync(ones, 0, ((size_t)npos * ncls + ncls) * sizeof(unsigned), st));
    if (!chosen.empty())
      IQCC_CUDA(cudaMemcpyAsync(dch, chosen.data(), chosen.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    const size_t smem = ((size_t)npos * ncls + ncls) * sizeof(unsigned);
    if (smem > 200 * 1024) throw std::runtime_error("choose_partition_bits: too many classes for the device counter");
    const unsigned grid = (unsigned)std::min<size_t>(592, std::max<size_t>(1, (s.M + 255) / 256));
    {
      KernelScope ks("partition_bits");
      switch (s.B) {
        case 1:
          IQCC_CUDA(cudaFuncSetAttribute(k_bit_counts<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
          k_bit_counts<1><<<grid, 256, smem, st>>>(s.keys(), s.coef(), s.M, s.filt, nq, dch, (int)r, ones, cls);
          break;
        case 2:
          IQCC_CUDA(cudaFuncSetAttribute(k_bit_counts<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
          k_bit_counts<2><<<grid, 256, smem, st>>>(s.keys(), s.coef(), s.M, s.filt, nq, dch, (int)r, ones, cls);
          break;
        default:
          IQCC_CUDA(cudaFuncSetAttribute(k_bit_counts<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
          k_bit_counts<4><<<grid, 256, smem, st>>>(s.keys(), s.coef(), s.M, s.filt, nq, dch, (int)r, ones, cls);
          break;
      }
    }
    std::vector<unsigned> h((size_t)npos * ncls + ncls);
    IQCC_CUDA(cudaMemcpyAsync(h.data(), ones, h.size() * sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    IQCC_CUDA(cudaStreamSynchronize(st));
    if (r == m) {
      final_cnt.assign(h.begin() + (size_t)npos * ncls, h.end());
      break;
    }
    // greedy: minimize the largest of the 2^(r+1) classes; lowest position wins ties
    size_t best_pos = npos, best_max = SIZE_MAX;
    for (int p = 0; p < npos; ++p) {
      if (std::find(chosen.begin(), chosen.end(), p) != chosen.end()) continue;
      size_t worst = 0;
      for (int c = 0; c < ncls; ++c) {
        const size_t one = h[(size_t)p * ncls + c], all = h[(size_t)npos * ncls + c];
        worst = std::max(worst, std::max(one, all - one));
      }
      if (worst < best_max) {
        best_max = worst;
        best_pos = p;
      }
    }
    chosen.push_back((int)best_pos);
  }
  for (size_t i = 0; i < m; ++i) bits_out[i] = chosen[i];
  if (s.logical == 0 || m == 0) return 1.0;
  const double ideal = (double)s.logical / (double)(1u << m);
  return (double)*std::max_element(final_cnt.begin(), final_cnt.end()) / std::max(1.0, ideal);
}

}  // namespace iqcc_b200
