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

// Factor rows F4[q][code], code = x | z << 1 (0: I -> 1.0, 1: X, 2: Z, 3: Y),
// 64*B rows (padding qubits are identities).  Every lane of a warp walks the
// qubits in the same ascending order, so the table reads of a warp hit one
// 32-byte row (one shared-memory wavefront) and there is no divergence;
// identity positions multiply by 1.0, which is exact, so the product is
// bit-identical to expect_word's product over the support only
// (iqcc/qmf.hpp:67-80).
template <int B, class Fn>
__device__ __forceinline__ void for_each_qubit_code(const Key<B>& k, Fn&& fn) {
#pragma unroll
  for (int w = 0; w < B; ++w) {
#pragma unroll
    for (int h = 1; h >= 0; --h) {  // device bits 63..32 hold qubits 64w + 0..31
      const unsigned xh = (unsigned)(k.w[w] >> (32 * h)), zh = (unsigned)(k.w[B + w] >> (32 * h));
#pragma unroll
      for (int b = 31; b >= 0; --b) {
        const int q = 64 * w + (1 - h) * 32 + (31 - b);
        fn(q, ((xh >> b) & 1u) | (((zh >> b) & 1u) << 1));
      }
    }
  }
}

template <int B>
__device__ __forceinline__ double lockstep_expect(const Key<B>& k, const double* __restrict__ f4) {
  double val = 1.0;
  for_each_qubit_code<B>(k, [&](int q, unsigned code) { val = __dmul_rn(val, f4[4 * q + code]); });
  return val;
}

template <int B>
__global__ void __launch_bounds__(256) k_expect(const ull* __restrict__ keys,
                                                const double* __restrict__ coef, size_t M,
                                                Filter filt, const double* __restrict__ f4_g,
                                                double* __restrict__ partial) {
  __shared__ double f4[4 * 64 * B];
  __shared__ double rs[256], rc[256];
  for (int i = threadIdx.x; i < 4 * 64 * B; i += blockDim.x) f4[i] = f4_g[i];
  __syncthreads();
  TwoSum acc;
  const size_t per = (M + gridDim.x - 1) / gridDim.x;
  const size_t lo = blockIdx.x * per, hi = min(M, lo + per);
  for (size_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const Key<B> k = load_key<B>(keys, i);
    const double c = coef[i];
    if (!filter_keep(filt, i, c, i == 0 && key_is_identity<B>(k))) continue;
    acc.add(__dmul_rn(c, lockstep_expect<B>(k, f4)));
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

// Nibble tables: the qubit slots in groups of four; for group g the 256
// products of its four factors, indexed by the group's z nibble | x nibble
// << 4 (nibbles as they sit in the bit-reversed device words: bit 3 =
// qubit 4g).  A term's value is the product of its 16B group entries in
// ascending group order: 16B dmuls and table reads instead of 64B, at the
// price of the per-term rounding order (the sum is within 1e-15 relative of
// expect_word's; the engine's energies are specified to 1e-10).  With the z
// nibble in the low index bits, terms whose x nibble is 0 (most groups of a
// molecular Hamiltonian) read 16 consecutive entries: distinct banks.
__global__ void k_nibble_table(const double* __restrict__ f4, int ngroups, double* __restrict__ tab) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ngroups * 256) return;
  const int g = i >> 8, idx = i & 255, zn = idx & 15, xn = idx >> 4;
  double v = 1.0;
  for (int j = 3; j >= 0; --j) {  // nibble bit 3 = qubit 4g: ascending qubit order
    const int q = 4 * g + (3 - j);
    const unsigned code = ((xn >> j) & 1u) | (((zn >> j) & 1u) << 1);
    v = __dmul_rn(v, f4[4 * q + code]);
  }
  tab[i] = v;
}

template <int B, int NT>
__global__ void __launch_bounds__(NT) k_expect_nib(const ull* __restrict__ keys,
                                                   const double* __restrict__ coef, size_t M,
                                                   Filter filt, const double* __restrict__ tab_g,
                                                   double* __restrict__ partial) {
  constexpr int NG = 16 * B;  // groups of four qubit slots
  extern __shared__ double tab[];  // [NG][256]
  __shared__ double rs[NT], rc[NT];
  for (int i = threadIdx.x; i < NG * 256; i += blockDim.x) tab[i] = tab_g[i];
  __syncthreads();
  TwoSum acc;
  const size_t per = (M + gridDim.x - 1) / gridDim.x;
  const size_t lo = blockIdx.x * per, hi = min(M, lo + per);
  // the next term's row and coefficient are in flight while this one is
  // multiplied out (the loop is otherwise one dependent load per term)
  Key<B> kn;
  double cn = 0.0;
  if (lo + threadIdx.x < hi) {
    kn = load_key<B>(keys, lo + threadIdx.x);
    cn = coef[lo + threadIdx.x];
  }
  for (size_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const Key<B> k = kn;
    const double c = cn;
    if (i + blockDim.x < hi) {
      kn = load_key<B>(keys, i + blockDim.x);
      cn = coef[i + blockDim.x];
    }
    if (!filter_keep(filt, i, c, i == 0 && key_is_identity<B>(k))) continue;
    double v = 1.0;
#pragma unroll
    for (int w = 0; w < B; ++w) {
#pragma unroll
      for (int h = 1; h >= 0; --h) {
        const unsigned xh = (unsigned)(k.w[w] >> (32 * h)), zh = (unsigned)(k.w[B + w] >> (32 * h));
#pragma unroll
        for (int n = 7; n >= 0; --n) {  // bits 31..28 hold the lowest qubits of the half
          const int g = 16 * w + 8 * (1 - h) + (7 - n);
          const unsigned idx = ((zh >> (4 * n)) & 15u) | (((xh >> (4 * n)) & 15u) << 4);
          v = __dmul_rn(v, tab[g * 256 + idx]);
        }
      }
    }
    acc.add(__dmul_rn(c, v));
  }
  rs[threadIdx.x] = acc.s;
  rc[threadIdx.x] = acc.c;
  __syncthreads();
  for (int o = NT / 2; o > 0; o >>= 1) {  // fixed tree: deterministic
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

/// F4 rows from the host factor table [nq][3] = (X, Z, Y).
static std::vector<double> factor_rows(const double* factors, int nq, uint32_t B) {
  std::vector<double> f4((size_t)4 * 64 * B, 1.0);
  for (int q = 0; q < nq; ++q) {
    f4[4 * q + 1] = factors[3 * q + 0];
    f4[4 * q + 2] = factors[3 * q + 1];
    f4[4 * q + 3] = factors[3 * q + 2];
  }
  return f4;
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
  const std::vector<double> f4 = factor_rows(factors, nq, s.B);
  double* tab = ws.tables.as<double>(f4.size());
  IQCC_CUDA(cudaMemcpyAsync(tab, f4.data(), f4.size() * sizeof(double), cudaMemcpyHostToDevice, st));
  // IQCC_EXPECT_EXACT=1: the lockstep product over every qubit slot (each
  // term's value bit-identical to expect_word); default: nibble tables
  const bool exact = getenv("IQCC_EXPECT_EXACT") && atoi(getenv("IQCC_EXPECT_EXACT")) != 0;
  // nibble tables take 32 KB per device block of the key: 512-thread CTAs,
  // 2 per SM at B <= 2 (32 warps), 1 at B = 4
  const unsigned per_sm = exact ? 8u : (s.B >= 4 ? 1u : (s.B == 2 ? 3u : 6u));
  const unsigned grid = (unsigned)std::min<size_t>(148 * (exact ? 8u : (s.B >= 4 ? 1u : 2u)),
                                                   std::max<size_t>(1, (s.M + 1023) / 1024));
  (void)per_sm;
  double* part = ws.partials.as<double>(2 * grid);
  if (exact) {
    KernelScope ks("expect");
    switch (s.B) {
      case 1: k_expect<1><<<grid, 256, 0, st>>>(s.keys(), s.coef(), s.M, s.filt, tab, part); break;
      case 2: k_expect<2><<<grid, 256, 0, st>>>(s.keys(), s.coef(), s.M, s.filt, tab, part); break;
      default: k_expect<4><<<grid, 256, 0, st>>>(s.keys(), s.coef(), s.M, s.filt, tab, part); break;
    }
  } else {
    const int ng = 16 * (int)s.B;
    double* nib = ws.misc2.as<double>((size_t)ng * 256);
    const size_t smem = (size_t)ng * 256 * sizeof(double);
    KernelScope ks("expect");
    k_nibble_table<<<(ng * 256 + 255) / 256, 256, 0, st>>>(tab, ng, nib);
    switch (s.B) {
      case 1:
        IQCC_CUDA(cudaFuncSetAttribute(k_expect_nib<1, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_expect_nib<1, 512><<<grid, 512, smem, st>>>(s.keys(), s.coef(), s.M, s.filt, nib, part);
        break;
      case 2:
        IQCC_CUDA(cudaFuncSetAttribute(k_expect_nib<2, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_expect_nib<2, 512><<<grid, 512, smem, st>>>(s.keys(), s.coef(), s.M, s.filt, nib, part);
        break;
      default:
        IQCC_CUDA(cudaFuncSetAttribute(k_expect_nib<4, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_expect_nib<4, 512><<<grid, 512, smem, st>>>(s.keys(), s.coef(), s.M, s.filt, nib, part);
        break;
    }
  }
  return host_sum_pairs(fetch(part, 2 * grid));
}

// -------------------------------------------------------- QMF gradient
// d/d angle_k of c * prod_j f_j is c * rest_k * f'_k with rest_k the product
// of the other factors.  For a term without a zero factor rest_k * f'_k =
// P * (f'_k / f_k), so the gradient is a weighted histogram:
//   g[k] = sum_code R[k][code] * H[k][code],  H[k][code] = sum of c*P over
//   the terms with letter `code` at qubit k,   R = f' / f  (host, per Omega).
// A term with exactly one zero factor (at k0) contributes only to k0:
// c * P_nz * f'_k0 (P_nz = product of its nonzero factors); two or more
// zeros contribute nothing (iqcc/qmf.hpp:94-148, prefix/suffix products).
// Phase 1 (thread per term): the product in lockstep (as expect), staged in
// shared memory with the term's key.  Phase 2 (thread per qubit): every
// qubit's thread walks the staged batch and adds each weight to the bin of
// the term's letter at that qubit (two-level sums: per batch, then running).
// Deterministic: fixed batches per block, blocks summed on the host in order.
constexpr int kQB = 256;  // terms per batch = threads per block

template <int B, bool ZEROS>
__global__ void __launch_bounds__(kQB) k_qmf_grad(const ull* __restrict__ keys,
                                                  const double* __restrict__ coef, size_t M,
                                                  Filter filt, const double* __restrict__ f4_g,
                                                  const unsigned char* __restrict__ zm_g, int nq,
                                                  double* __restrict__ partial) {
  __shared__ double f4[4 * 64 * B];
  __shared__ unsigned char zm[64 * B];  // bit `code`: that factor is zero
  __shared__ ull skx[kQB * B], skz[kQB * B];  // staged keys (x / z planes)
  __shared__ double wa[kQB], wb[kQB];
  __shared__ int k0s[kQB];
  __shared__ double rs[kQB], rc[kQB];
  for (int i = threadIdx.x; i < 4 * 64 * B; i += kQB) f4[i] = f4_g[i];
  for (int i = threadIdx.x; i < 64 * B; i += kQB) zm[i] = ZEROS ? zm_g[i] : 0;
  __syncthreads();
  // phase 2: TPQ threads per qubit slot, each summing every TPQ-th staged term
  constexpr int TPQ = 4 / B;
  const int k = threadIdx.x % (64 * B), part = threadIdx.x / (64 * B);
  // 32-bit half of the staged word holding the qubit, and the bit in it
  const int kw = k >> 6, khalf = (k & 63) < 32 ? 1 : 0, kb = 31 - (k & 31);
  double h[3] = {0.0, 0.0, 0.0}, h1[3] = {0.0, 0.0, 0.0};
  TwoSum e;
  for (size_t base = (size_t)blockIdx.x * kQB; base < M; base += (size_t)gridDim.x * kQB) {
    const size_t i = base + threadIdx.x;
    double a = 0.0, b1 = 0.0;
    int k0 = -1;
    Key<B> key;
#pragma unroll
    for (int w = 0; w < 2 * B; ++w) key.w[w] = 0;
    if (i < M) {
      key = load_key<B>(keys, i);
      const double c = coef[i];
      if (filter_keep(filt, i, c, i == 0 && key_is_identity<B>(key))) {
        double p = 1.0;
        int nz = 0;
        for_each_qubit_code<B>(key, [&](int q, unsigned code) {
          if (ZEROS && ((zm[q] >> code) & 1u)) {
            ++nz;
            k0 = q;
          } else {
            p = __dmul_rn(p, f4[4 * q + code]);
          }
        });
        const double w = __dmul_rn(c, p);
        if (nz == 0) {
          a = w;
          e.add(w);
        } else if (nz == 1) {
          b1 = w;
        }
      }
    }
#pragma unroll
    for (int w = 0; w < B; ++w) {
      skx[threadIdx.x * B + w] = key.w[w];
      skz[threadIdx.x * B + w] = key.w[B + w];
    }
    wa[threadIdx.x] = a;
    wb[threadIdx.x] = b1;
    k0s[threadIdx.x] = k0;
    __syncthreads();
    if (k < nq) {
      // four interleaved accumulator sets keep four independent add chains
      double ba[4][3] = {};
      const int n = (int)min((size_t)kQB, M - base);
      const unsigned* sx32 = reinterpret_cast<const unsigned*>(skx) + 2 * kw + khalf;
      const unsigned* sz32 = reinterpret_cast<const unsigned*>(skz) + 2 * kw + khalf;
      for (int t0 = part; t0 < n; t0 += 4 * TPQ) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int t = t0 + u * TPQ;
          if (t < n) {
            const unsigned code = ((sx32[2 * B * t] >> kb) & 1u) | (((sz32[2 * B * t] >> kb) & 1u) << 1);
            const double v = wa[t];
            if (code == 1) ba[u][0] = __dadd_rn(ba[u][0], v);
            if (code == 2) ba[u][1] = __dadd_rn(ba[u][1], v);
            if (code == 3) ba[u][2] = __dadd_rn(ba[u][2], v);
            if (ZEROS && k0s[t] == k) {
              const double w1 = wb[t];
              if (code == 1) h1[0] = __dadd_rn(h1[0], w1);
              if (code == 2) h1[1] = __dadd_rn(h1[1], w1);
              if (code == 3) h1[2] = __dadd_rn(h1[2], w1);
            }
          }
        }
      }
#pragma unroll
      for (int c = 0; c < 3; ++c)
        h[c] = __dadd_rn(h[c], __dadd_rn(__dadd_rn(ba[0][c], ba[1][c]), __dadd_rn(ba[2][c], ba[3][c])));
    }
    __syncthreads();
  }
  double* out = partial + (size_t)blockIdx.x * (6 * (size_t)nq * TPQ + 2);
  if (k < nq) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      out[6 * ((size_t)nq * part + k) + c] = h[c];
      out[6 * ((size_t)nq * part + k) + 3 + c] = h1[c];
    }
  }
  rs[threadIdx.x] = e.s;
  rc[threadIdx.x] = e.c;
  __syncthreads();
  for (int o = kQB / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      TwoSum x{rs[threadIdx.x], rc[threadIdx.x]}, y{rs[threadIdx.x + o], rc[threadIdx.x + o]};
      x.merge(y);
      rs[threadIdx.x] = x.s;
      rc[threadIdx.x] = x.c;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[6 * (size_t)nq * TPQ] = rs[0];
    out[6 * (size_t)nq * TPQ + 1] = rc[0];
  }
}

// ---------------------------------------- QMF gradient, no zero factors
// H[k][code] = sum of w = c*P over the terms whose letter at qubit k is
// `code` (see above).  One warp takes 32 terms at a time (one per lane):
//  * every lane's 32-bit slice of its x and z words is transposed across the
//    warp (5 butterfly shuffles), so lane k holds, for qubit k of the slice,
//    the 32-term masks of X (x & ~z), Z (z & ~x) and Y (x & z) letters;
//  * the 32 weights form 8 groups of 4 whose 16 subset sums sit in shared
//    memory (Four Russians): each group adds S_u[mask nibble] to the lane's
//    three bins with one conflict-free read instead of four adds per term.
// Work per term is O(qubit slots / 32) instead of O(qubits); the order of
// every sum is fixed (deterministic).  P is the nibble-table product.
__device__ __forceinline__ unsigned transpose32(unsigned x) {
  const int lane = threadIdx.x & 31;
  const unsigned hi[5] = {0xFFFF0000u, 0xFF00FF00u, 0xF0F0F0F0u, 0xCCCCCCCCu, 0xAAAAAAAAu};
#pragma unroll
  for (int t = 0; t < 5; ++t) {
    const int sft = 16 >> t;
    const unsigned y = __shfl_xor_sync(0xffffffffu, x, sft);
    x = (lane & sft) ? ((x & hi[t]) | ((y >> sft) & ~hi[t])) : ((x & ~hi[t]) | ((y << sft) & hi[t]));
  }
  return x;
}

template <int B, int NT>
__global__ void __launch_bounds__(NT) k_qmf_grad_fr(const ull* __restrict__ keys, const double* __restrict__ coef,
                                                    size_t M, Filter filt, const double* __restrict__ nib_g,
                                                    double* __restrict__ partial) {
  constexpr int NG = 16 * B, NS = 2 * B;  // nibble groups; 32-qubit slices
  constexpr int NW = NT / 32;              // warps sharing one nibble table
  extern __shared__ double shq[];
  double* tab = shq;                       // [NG][256]
  double* St = shq + NG * 256;             // [NW][8 groups][16]
  double* Wt = St + NW * 128;              // [NW][32]
  double* red = Wt + NW * 32;              // [NW][NS][32][3] block reduction
  for (int i = threadIdx.x; i < NG * 256; i += blockDim.x) tab[i] = nib_g[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* S = St + warp * 128;
  double* Wl = Wt + warp * 32;
  double acc[NS][3];
#pragma unroll
  for (int a = 0; a < NS; ++a) acc[a][0] = acc[a][1] = acc[a][2] = 0.0;
  TwoSum e;
  const size_t nchunk = (M + 31) / 32;
  const size_t cstep = (size_t)gridDim.x * NW;
  Key<B> kn;
  double cn = 0.0;
  {
    const size_t i0 = ((size_t)blockIdx.x * NW + warp) * 32 + lane;
    if (i0 < M) {
      kn = load_key<B>(keys, i0);
      cn = coef[i0];
    }
  }
  for (size_t ch = (size_t)blockIdx.x * NW + warp; ch < nchunk; ch += cstep) {
    const size_t i = ch * 32 + lane;
    Key<B> k;
#pragma unroll
    for (int w = 0; w < 2 * B; ++w) k.w[w] = 0;
    double wt = 0.0;
    const Key<B> kk = kn;
    const double c = cn;
    if ((ch + cstep) * 32 + lane < M) {  // the next chunk's row in flight
      kn = load_key<B>(keys, (ch + cstep) * 32 + lane);
      cn = coef[(ch + cstep) * 32 + lane];
    }
    if (i < M) {
      if (filter_keep(filt, i, c, i == 0 && key_is_identity<B>(kk))) {
        k = kk;
        double v = 1.0;
#pragma unroll
        for (int w = 0; w < B; ++w)
#pragma unroll
          for (int h = 1; h >= 0; --h) {
            const unsigned xh = (unsigned)(k.w[w] >> (32 * h)), zh = (unsigned)(k.w[B + w] >> (32 * h));
#pragma unroll
            for (int n = 7; n >= 0; --n) {
              const int g = 16 * w + 8 * (1 - h) + (7 - n);
              v = __dmul_rn(v, tab[g * 256 + (((zh >> (4 * n)) & 15u) | (((xh >> (4 * n)) & 15u) << 4))]);
            }
          }
        wt = __dmul_rn(c, v);
        e.add(wt);
      }
    }
    Wl[lane] = wt;
    __syncwarp();
    // subset sums of the 8 groups of 4 terms: lane -> (group 2r + lane/16, subset lane%16)
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int u = 2 * r + (lane >> 4), sub = lane & 15;
      double sum = 0.0;
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if ((sub >> b) & 1) sum = __dadd_rn(sum, Wl[4 * u + b]);
      S[u * 16 + sub] = sum;
    }
    __syncwarp();
#pragma unroll
    for (int w = 0; w < B; ++w)
#pragma unroll
      for (int h = 1; h >= 0; --h) {
        const int sl = 2 * w + (1 - h);
        const unsigned xt = transpose32((unsigned)(k.w[w] >> (32 * h)));
        const unsigned zt = transpose32((unsigned)(k.w[B + w] >> (32 * h)));
        const unsigned mx = xt & ~zt, mz = zt & ~xt, my = xt & zt;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          acc[sl][0] = __dadd_rn(acc[sl][0], S[u * 16 + ((mx >> (4 * u)) & 15u)]);
          acc[sl][1] = __dadd_rn(acc[sl][1], S[u * 16 + ((mz >> (4 * u)) & 15u)]);
          acc[sl][2] = __dadd_rn(acc[sl][2], S[u * 16 + ((my >> (4 * u)) & 15u)]);
        }
      }
    __syncwarp();
  }
  // lane k of slice sl holds qubit 32*sl + (31 - k); warps summed in order
#pragma unroll
  for (int a = 0; a < NS; ++a)
#pragma unroll
    for (int c = 0; c < 3; ++c) red[((warp * NS + a) * 32 + lane) * 3 + c] = acc[a][c];
  __shared__ double rs[NT], rc[NT];
  rs[threadIdx.x] = e.s;
  rc[threadIdx.x] = e.c;
  __syncthreads();
  for (int j = threadIdx.x; j < NS * 32 * 3; j += blockDim.x) {
    double v = 0.0;
    for (int wp = 0; wp < NW; ++wp) v = __dadd_rn(v, red[wp * NS * 96 + j]);
    const int a = j / 96, r = j % 96, ln = r / 3, c = r % 3;
    const int q = 32 * a + (31 - ln);
    partial[(size_t)blockIdx.x * (NS * 96 + 2) + 3 * q + c] = v;
  }
  for (int o = NT / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      TwoSum x{rs[threadIdx.x], rc[threadIdx.x]}, y{rs[threadIdx.x + o], rc[threadIdx.x + o]};
      x.merge(y);
      rs[threadIdx.x] = x.s;
      rc[threadIdx.x] = x.c;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    partial[(size_t)blockIdx.x * (NS * 96 + 2) + NS * 96] = rs[0];
    partial[(size_t)blockIdx.x * (NS * 96 + 2) + NS * 96 + 1] = rc[0];
  }
}

double qmf_grad_store(DeviceStore& s, const double* factors, const double* derivs, double* grad) {
  Workspace& ws = workspace();
  cudaStream_t st = stream();
  const int nq = (int)s.n_qubits;
  std::fill(grad, grad + 2 * nq, 0.0);
  if (s.logical == 0) return 0.0;
  std::vector<double> f4 = factor_rows(factors, nq, s.B);
  std::vector<unsigned char> zm((size_t)64 * s.B, 0);
  bool zeros = false;
  for (int q = 0; q < nq; ++q)
    for (int c = 1; c < 4; ++c)
      if (f4[4 * q + c] == 0.0) {
        zm[q] |= (unsigned char)(1u << c);
        zeros = true;
      }
  double* tab = ws.tables.as<double>(f4.size() + zm.size() / 8 + 8);
  unsigned char* zmd = reinterpret_cast<unsigned char*>(tab + f4.size());
  IQCC_CUDA(cudaMemcpyAsync(tab, f4.data(), f4.size() * sizeof(double), cudaMemcpyHostToDevice, st));
  IQCC_CUDA(cudaMemcpyAsync(zmd, zm.data(), zm.size(), cudaMemcpyHostToDevice, st));
  if (!zeros && !(getenv("IQCC_QMF_GRAD_BINS") && atoi(getenv("IQCC_QMF_GRAD_BINS")))) {
    // no zero factor anywhere: every term is a c*P weight (bit-sliced kernel)
    // B <= 2: one 1024-thread CTA per SM shares one nibble table (32 warps);
    // B = 4 (a 128 KB table): 256 threads
    const int ng = 16 * (int)s.B, ns = 2 * (int)s.B;
    const int nt = s.B >= 4 ? 256 : 1024, nw = nt / 32;
    double* nib = ws.misc2.as<double>((size_t)ng * 256);
    const size_t smem = ((size_t)ng * 256 + (size_t)nw * 128 + (size_t)nw * 32 + (size_t)nw * ns * 96) * sizeof(double);
    const unsigned grid = (unsigned)std::min<size_t>(148, std::max<size_t>(1, (s.M + nt - 1) / nt));
    const size_t stride = (size_t)ns * 96 + 2;
    double* part = ws.grad_part.as<double>((size_t)grid * stride);
    {
      KernelScope ks("qmf_grad");
      k_nibble_table<<<(ng * 256 + 255) / 256, 256, 0, st>>>(tab, ng, nib);
#define IQCC_QF(B_, NT_)                                                                                        \
  IQCC_CUDA(cudaFuncSetAttribute(k_qmf_grad_fr<B_, NT_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
  k_qmf_grad_fr<B_, NT_><<<grid, NT_, smem, st>>>(s.keys(), s.coef(), s.M, s.filt, nib, part)
      switch (s.B) {
        case 1: IQCC_QF(1, 1024); break;
        case 2: IQCC_QF(2, 1024); break;
        default: IQCC_QF(4, 256); break;
      }
#undef IQCC_QF
    }
    const std::vector<double> h = fetch(part, (size_t)grid * stride);
    std::vector<double> H(3 * (size_t)64 * s.B, 0.0);
    double es = 0.0, ec = 0.0;
    for (unsigned b = 0; b < grid; ++b) {
      const double* p = h.data() + (size_t)b * stride;
      for (size_t j = 0; j < (size_t)ns * 96; ++j) H[j] += p[j];
      const double x = p[stride - 2];
      const double t = es + x;
      ec += std::fabs(es) >= std::fabs(x) ? (es - t) + x : (x - t) + es;
      es = t;
      ec += p[stride - 1];
    }
    for (int q = 0; q < nq; ++q)
      for (int c = 0; c < 3; ++c) {  // bins (X, Z, Y) = codes 1, 2, 3
        const double f = f4[4 * q + 1 + c];
        const double dth = derivs[6 * q + 2 * c], dph = derivs[6 * q + 2 * c + 1];
        grad[q] += H[3 * q + c] * (dth / f);
        grad[nq + q] += H[3 * q + c] * (dph / f);
      }
    return es + ec;
  }
  const unsigned grid = (unsigned)std::min<size_t>(148 * 6, std::max<size_t>(1, (s.M + kQB - 1) / kQB));
  const size_t tpq = 4 / s.B;  // threads per qubit slot in the kernel's phase 2
  const size_t stride = 6 * (size_t)nq * tpq + 2;
  double* part = ws.grad_part.as<double>((size_t)grid * stride);
  {
    KernelScope ks("qmf_grad");
#define IQCC_QG(B_)                                                                                     \
  if (zeros)                                                                                            \
    k_qmf_grad<B_, true><<<grid, kQB, 0, st>>>(s.keys(), s.coef(), s.M, s.filt, tab, zmd, nq, part);  \
  else                                                                                                  \
    k_qmf_grad<B_, false><<<grid, kQB, 0, st>>>(s.keys(), s.coef(), s.M, s.filt, tab, zmd, nq, part)
    switch (s.B) {
      case 1: IQCC_QG(1); break;
      case 2: IQCC_QG(2); break;
      default: IQCC_QG(4); break;
    }
#undef IQCC_QG
  }
  std::vector<double> h = fetch(part, (size_t)grid * stride);
  std::vector<double> H(6 * (size_t)nq, 0.0);
  double es = 0.0, ec = 0.0;
  for (unsigned b = 0; b < grid; ++b) {
    const double* p = h.data() + (size_t)b * stride;
    for (size_t r = 0; r < tpq; ++r)
      for (size_t j = 0; j < 6 * (size_t)nq; ++j) H[j] += p[6 * nq * r + j];
    const double x = p[stride - 2];
    const double t = es + x;
    ec += std::fabs(es) >= std::fabs(x) ? (es - t) + x : (x - t) + es;
    es = t;
    ec += p[stride - 1];
  }
  // derivs [q][6] = (dth, dph) for X, Z, Y; bins [q][code-1] with code 1 X, 2 Z, 3 Y
  for (int q = 0; q < nq; ++q) {
    for (int c = 0; c < 3; ++c) {
      const double f = f4[4 * q + 1 + c];
      const double dth = derivs[6 * q + 2 * c], dph = derivs[6 * q + 2 * c + 1];
      const double hn = H[6 * q + c], h1 = H[6 * q + 3 + c];
      if (f != 0.0) {
        grad[q] += hn * (dth / f);
        grad[nq + q] += hn * (dph / f);
      }
      grad[q] += h1 * dth;
      grad[nq + q] += h1 * dph;
    }
  }
  return es + ec;
}

// --------------------------------------------------------------- DIS
// g(P) = sum_k Im(c_k i^t) <omega|T_k P|omega>, skipping Im == 0; for real
// c_k, Im(c i^t) = c (t=1), -c (t=3), 0 otherwise (even t: commuting).
// One candidate per thread; the term range [lo, hi) is streamed through
// shared memory tiles shared by the whole block.
// All lanes of a warp read the same staged term; each lane's product T^P is
// taken over U = supp(T) | (union of the warp's candidate supports) in
// ascending qubit order, identity positions multiplying by 1.0 (exact), so
// the loop is warp-uniform, the factor reads of a warp hit one row, and the
// value is bit-identical to expect_word over supp(T^P).  Candidates of one
// flip group share their support (dis_candidates), so U is supp(T) plus a
// few qubits.
template <int B>
__global__ void __launch_bounds__(128) k_dis_full(const ull* __restrict__ keys,
                                                  const double* __restrict__ coef, size_t M,
                                                  Filter filt, const double* __restrict__ f4_g,
                                                  const ull* __restrict__ cands, size_t K,
                                                  double* __restrict__ g_out) {
  constexpr int TT = 128;
  __shared__ double f4[4 * 64 * B];
  __shared__ ull tk[TT * 2 * B];
  __shared__ double tc[TT];
  for (int i = threadIdx.x; i < 4 * 64 * B; i += blockDim.x) f4[i] = f4_g[i];
  const size_t cid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  Key<B> P;
#pragma unroll
  for (int w = 0; w < 2 * B; ++w) P.w[w] = 0;
  if (cid < K) P = load_key<B>(cands, cid);
  ull up[B];
#pragma unroll
  for (int w = 0; w < B; ++w) {
    const ull s = P.w[w] | P.w[B + w];
    const unsigned lo = __reduce_or_sync(0xffffffffu, (unsigned)s);
    const unsigned hi = __reduce_or_sync(0xffffffffu, (unsigned)(s >> 32));
    up[w] = ((ull)hi << 32) | lo;
  }
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
    const int n = (int)min((size_t)TT, M - base);
    // two terms per iteration: their products walk the union of both
    // supports (and U) in ascending order, a term multiplying by the exact
    // 1.0 of code 0 where it has no letter, so each chain is the
    // single-term chain (bit-identical) and the two run side by side; the
    // sum still adds term j before term j + 1
    for (int j = 0; j < n; j += 2) {
      Key<B> k[2];
      double c[2];
      bool anti[2], any[2];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int jj = min(j + t, n - 1);
#pragma unroll
        for (int w = 0; w < 2 * B; ++w) k[t].w[w] = tk[(size_t)jj * 2 * B + w];
        c[t] = j + t < n ? tc[jj] : 0.0;
        anti[t] = cid < K && c[t] != 0.0 && anticommutes<B>(k[t], P);
        any[t] = __any_sync(0xffffffffu, anti[t]);  // warp-uniform
      }
      if (!any[0] && !any[1]) continue;
      const Key<B> kp0 = key_xor<B>(k[0], P), kp1 = key_xor<B>(k[1], P);
      double v0 = 1.0, v1 = 1.0;
#pragma unroll
      for (int w = 0; w < B; ++w) {
        ull s = (any[0] ? k[0].w[w] | k[0].w[B + w] : 0ull) | (any[1] ? k[1].w[w] | k[1].w[B + w] : 0ull) | up[w];
        while (s) {
          const int lz = __clzll((long long)s);
          const int bit = 63 - lz;
          const unsigned c0 =
              (unsigned)((kp0.w[w] >> bit) & 1ull) | ((unsigned)((kp0.w[B + w] >> bit) & 1ull) << 1);
          const unsigned c1 =
              (unsigned)((kp1.w[w] >> bit) & 1ull) | ((unsigned)((kp1.w[B + w] >> bit) & 1ull) << 1);
          v0 = __dmul_rn(v0, f4[4 * (64 * w + lz) + c0]);
          v1 = __dmul_rn(v1, f4[4 * (64 * w + lz) + c1]);
          s &= ~(1ull << bit);
        }
      }
      if (anti[0]) {
        const double im = product_phase<B>(k[0], P) == 1 ? c[0] : -c[0];
        g = __dadd_rn(g, __dmul_rn(im, v0));
      }
      if (anti[1]) {
        const double im = product_phase<B>(k[1], P) == 1 ? c[1] : -c[1];
        g = __dadd_rn(g, __dmul_rn(im, v1));
      }
    }
  }
  if (cid < K) g_out[cid] = g;
}

// The generic-Omega gradient with nibble tables (about
// n/4 table reads and multiplies per pair): <omega|T^P|omega> is the
// product of the tables of T^P's 4-qubit groups (k_nibble_table), in two
// interleaved partial products for instruction-level parallelism.  The
// rounding order differs from expect_word's ascending-qubit product, so a
// gradient is within ~1e-15 relative of the reference's (the engine's
// energies and gradients are specified to 1e-10); IQCC_DIS_EXACT=1 (and
// dis_candidates, whose ranking must match the reference's bit for bit)
// takes k_dis_full.
template <int B>
__global__ void __launch_bounds__(256) k_dis_nib(const ull* __restrict__ keys, const double* __restrict__ coef,
                                                 size_t M, Filter filt, const double* __restrict__ tab_g, int ng,
                                                 const ull* __restrict__ cands, size_t K,
                                                 double* __restrict__ g_part) {
  constexpr int TT = 256;
  extern __shared__ double tab[];  // [ng][256]
  __shared__ ull tk[TT * 2 * B];
  __shared__ double tc[TT];
  for (int i = threadIdx.x; i < ng * 256; i += blockDim.x) tab[i] = tab_g[i];
  const size_t cid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  // term slice blockIdx.y of gridDim.y (partial sums, added in slice order)
  const size_t per = ((M + gridDim.y - 1) / gridDim.y + TT - 1) / TT * TT;
  const size_t lo = blockIdx.y * per, hi = min(M, lo + per);
  Key<B> P;
#pragma unroll
  for (int w = 0; w < 2 * B; ++w) P.w[w] = 0;
  if (cid < K) P = load_key<B>(cands, cid);
  double g = 0.0;
  for (size_t base = lo; base < hi; base += TT) {
    __syncthreads();
    const size_t i = base + threadIdx.x;
    if (i < hi) {
      const Key<B> k = load_key<B>(keys, i);
      double c = coef[i];
      if (!filter_keep(filt, i, c, i == 0 && key_is_identity<B>(k))) c = 0.0;  // Im(0) == 0: skipped
#pragma unroll
      for (int w = 0; w < 2 * B; ++w) tk[(size_t)threadIdx.x * 2 * B + w] = k.w[w];
      tc[threadIdx.x] = c;
    }
    __syncthreads();
    const int n = (int)min((size_t)TT, hi - base);
    // two terms per iteration: two independent sets of multiply chains
    // (the loop is bound by table-read and multiply latency, with the
    // table capping residency at 3 blocks per SM)
    for (int j = 0; j < n; j += 2) {
      Key<B> k[2];
      double c[2];
      bool anti[2];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int jj = min(j + t, n - 1);
#pragma unroll
        for (int w = 0; w < 2 * B; ++w) k[t].w[w] = tk[(size_t)jj * 2 * B + w];
        c[t] = j + t < n ? tc[jj] : 0.0;
        anti[t] = cid < K && c[t] != 0.0 && anticommutes<B>(k[t], P);
      }
      if (!__any_sync(0xffffffffu, anti[0] || anti[1])) continue;  // warp-uniform
      double v[2][4];
#pragma unroll
      for (int t = 0; t < 2; ++t) v[t][0] = v[t][1] = v[t][2] = v[t][3] = 1.0;
#pragma unroll
      for (int w = 0; w < B; ++w)
#pragma unroll
        for (int h = 1; h >= 0; --h) {
          unsigned xh[2], zh[2];
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            xh[t] = (unsigned)((k[t].w[w] ^ P.w[w]) >> (32 * h));
            zh[t] = (unsigned)((k[t].w[B + w] ^ P.w[B + w]) >> (32 * h));
          }
#pragma unroll
          for (int nn = 7; nn >= 0; --nn) {
            const int q = 16 * w + 8 * (1 - h) + (7 - nn);
            if (q < ng) {
#pragma unroll
              for (int t = 0; t < 2; ++t)
                v[t][q & 3] = __dmul_rn(
                    v[t][q & 3], tab[q * 256 + (((zh[t] >> (4 * nn)) & 15u) | (((xh[t] >> (4 * nn)) & 15u) << 4))]);
            }
          }
        }
#pragma unroll
      for (int t = 0; t < 2; ++t)
        if (anti[t]) {
          const double im = product_phase<B>(k[t], P) == 1 ? c[t] : -c[t];
          g = __dadd_rn(g, __dmul_rn(im, __dmul_rn(__dmul_rn(v[t][0], v[t][1]), __dmul_rn(v[t][2], v[t][3]))));
        }
    }
  }
  if (cid < K) g_part[blockIdx.y * K + cid] = g;
}

// The generic-Omega gradient by factor ratios (default when no factor of
// Omega is zero).  T^P differs from T only in the nibble groups P touches
// (a DIS candidate touches at most 4), so
//   <omega|T^P|omega> = E_T * prod_{g in G(P)} f_g((T^P)_g) / f_g(T_g),
// with E_T = prod_g f_g(T_g) and the reciprocals 1/f_g(T_g) computed once
// per staged term and shared by the block's candidates: about 2|G(P)|
// table reads and multiplies per anticommuting pair instead of n/4.  A term
// whose E_T could lose precision (|E_T| < 1e-280) or a candidate touching
// more than 4 groups takes the full nibble product.  Rounding differs from
// expect_word's ascending product by a few ulps per term (the gradient is
// specified to 1e-10; tests pin 1e-13).
// 128 staged terms per tile; 1024 candidates (threads) per block share the
// staged E_T / reciprocals and the tables (512 at 200-256 qubits, whose
// wider rows need more than 64 registers).  Measured on C4 (100 qubits):
// 256 threads x 64 / 128 / 256 terms 8.0 / 10.2 / 19.1 s, 512 x 64 6.3 s,
// 1024 x 32 / 64 / 128 6.1 / 5.8 / 5.6 s (profiles/r2s2_summary.md).
constexpr int kRatioTT = 128;
__host__ __device__ constexpr int ratio_nt(int B) { return B >= 4 ? 512 : 1024; }
template <int B>
__global__ void __launch_bounds__(ratio_nt(B)) k_dis_ratio(const ull* __restrict__ keys, const double* __restrict__ coef,
                                                   size_t M, Filter filt, const double* __restrict__ tab_g, int ng,
                                                   const ull* __restrict__ cands, size_t K,
                                                   double* __restrict__ g_part) {
  constexpr int TT = kRatioTT;
  extern __shared__ double smd[];
  double* tab = smd;                     // [ng][256]
  double* rinv = tab + (size_t)ng * 256;  // [TT][ng]
  double* te = rinv + (size_t)TT * ng;    // [TT]
  double* tc = te + TT;                   // [TT]
  ull* tk = reinterpret_cast<ull*>(tc + TT);  // [TT][2B]
  int* tslow = reinterpret_cast<int*>(tk + (size_t)TT * 2 * B);  // [TT]
  unsigned char* tcode = reinterpret_cast<unsigned char*>(tslow + TT);  // [TT][ng] group codes of T
  for (int i = threadIdx.x; i < ng * 256; i += blockDim.x) tab[i] = tab_g[i];
  const size_t cid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const size_t per = ((M + gridDim.y - 1) / gridDim.y + TT - 1) / TT * TT;
  const size_t lo = blockIdx.y * per, hi = min(M, lo + per);
  Key<B> P;
#pragma unroll
  for (int w = 0; w < 2 * B; ++w) P.w[w] = 0;
  if (cid < K) P = load_key<B>(cands, cid);
  // the candidate's touched groups: (group, word, shift, code) packed
  unsigned e[4] = {0u, 0u, 0u, 0u};
  int mg = 0;
#pragma unroll
  for (int w = 0; w < B; ++w)
#pragma unroll
    for (int h = 1; h >= 0; --h)
#pragma unroll
      for (int nn = 7; nn >= 0; --nn) {
        const int q = 16 * w + 8 * (1 - h) + (7 - nn);
        const int sh = 32 * h + 4 * nn;
        const unsigned code = (unsigned)(((P.w[B + w] >> sh) & 15u) | (((P.w[w] >> sh) & 15u) << 4));
        if (q < ng && code) {
          const unsigned ent = (unsigned)q | ((unsigned)w << 6) | ((unsigned)sh << 8) | (code << 16);
          if (mg == 0) e[0] = ent;
          else if (mg == 1) e[1] = ent;
          else if (mg == 2) e[2] = ent;
          else if (mg == 3) e[3] = ent;
          ++mg;
        }
      }
  const bool general = mg > 4;
  double g = 0.0;
  for (size_t base = lo; base < hi; base += TT) {
    __syncthreads();
    for (int i = threadIdx.x; i < TT; i += blockDim.x) {
      const size_t ti = base + i;
      Key<B> k;
#pragma unroll
      for (int w = 0; w < 2 * B; ++w) k.w[w] = 0;
      double c = 0.0;
      if (ti < hi) {
        k = load_key<B>(keys, ti);
        c = coef[ti];
        if (!filter_keep(filt, ti, c, ti == 0 && key_is_identity<B>(k))) c = 0.0;
      }
      double E = 1.0;
#pragma unroll
      for (int w = 0; w < B; ++w)
#pragma unroll
        for (int h = 1; h >= 0; --h)
#pragma unroll
          for (int nn = 7; nn >= 0; --nn) {
            const int q = 16 * w + 8 * (1 - h) + (7 - nn);
            if (q < ng) {
              const int sh = 32 * h + 4 * nn;
              const unsigned co = (unsigned)(((k.w[B + w] >> sh) & 15u) | (((k.w[w] >> sh) & 15u) << 4));
              const double f = tab[q * 256 + (int)co];
              E = __dmul_rn(E, f);
              rinv[(size_t)i * ng + q] = __drcp_rn(f);
              tcode[(size_t)i * ng + q] = (unsigned char)co;
            }
          }
#pragma unroll
      for (int w = 0; w < 2 * B; ++w) tk[(size_t)i * 2 * B + w] = k.w[w];
      tc[i] = c;
      te[i] = E;
      tslow[i] = !(fabs(E) >= 1e-280);
    }
    __syncthreads();
    const int n = (int)min((size_t)TT, hi - base);
    for (int j = 0; j < n; ++j) {
      const ull* kj = tk + (size_t)j * 2 * B;
      const double c = tc[j];
      Key<B> k;
#pragma unroll
      for (int w = 0; w < 2 * B; ++w) k.w[w] = kj[w];
      const bool anti = cid < K && c != 0.0 && anticommutes<B>(k, P);
      if (!anti) continue;
      double val;
      if (general || tslow[j]) {  // full nibble product of T^P
        val = 1.0;
#pragma unroll
        for (int w = 0; w < B; ++w)
#pragma unroll
          for (int h = 1; h >= 0; --h)
#pragma unroll
            for (int nn = 7; nn >= 0; --nn) {
              const int q = 16 * w + 8 * (1 - h) + (7 - nn);
              if (q < ng) {
                const int sh = 32 * h + 4 * nn;
                const ull xw = k.w[w] ^ P.w[w], zw = k.w[B + w] ^ P.w[B + w];
                val = __dmul_rn(val, tab[q * 256 + (int)(((zw >> sh) & 15u) | (((xw >> sh) & 15u) << 4))]);
              }
            }
      } else {
        val = te[j];
        const double* rj = rinv + (size_t)j * ng;
        const unsigned char* cj = tcode + (size_t)j * ng;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          if (m < mg) {
            const unsigned ent = e[m];
            const int q = (int)(ent & 63u);
            const unsigned co = cj[q];
            val = __dmul_rn(__dmul_rn(val, tab[q * 256 + (int)(co ^ (ent >> 16))]), rj[q]);
          }
        }
      }
      const double im = product_phase<B>(k, P) == 1 ? c : -c;
      g = __dadd_rn(g, __dmul_rn(im, val));
    }
  }
  if (cid < K) g_part[blockIdx.y * K + cid] = g;
}

/// g[k] = the slices' partial sums in slice order.
__global__ void k_dis_fold(const double* __restrict__ g_part, size_t K, int S, double* __restrict__ g) {
  const size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (k >= K) return;
  double v = g_part[k];
  for (int s = 1; s < S; ++s) v = __dadd_rn(v, g_part[s * K + k]);
  g[k] = v;
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
                           size_t K, bool flip_group_only, double* g, bool exact = false) {
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
    const std::vector<double> f4 = factor_rows(factors, nq, B);
    // nibble path: term slices so that the candidate blocks fill the SMs
    // (the table limits a SM to a few resident blocks); partials after f4
    const unsigned cb = (unsigned)((K + 255) / 256);
    const int S = (int)std::max<size_t>(1, std::min<size_t>({8, (148 * 4 + cb - 1) / cb, (s.M + 4095) / 4096}));
    double* f4d = ws.grad_part.as<double>(f4.size() + (size_t)8 * K);  // slices <= 8 on every path
    double* gpart = f4d + f4.size();
    IQCC_CUDA(cudaMemcpyAsync(f4d, f4.data(), f4.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    const char* ex = getenv("IQCC_DIS_EXACT");
    const char* nib_env = getenv("IQCC_DIS_NIB");
    const int ngr = std::max(1, (nq + 3) / 4);
    const size_t smem_ratio = ((size_t)ngr * 256 + (size_t)kRatioTT * ngr + 2 * (size_t)kRatioTT) * sizeof(double) +
                              (size_t)kRatioTT * 2 * B * sizeof(ull) + (size_t)kRatioTT * sizeof(int) +
                              (size_t)kRatioTT * ngr;
    bool zero_factor = false;  // a zero factor makes the ratios undefined
    for (size_t i = 0; i < f4.size(); ++i) zero_factor = zero_factor || f4[i] == 0.0;
    const bool ratio = !(nib_env && atoi(nib_env)) && !zero_factor && smem_ratio <= (size_t)220 * 1024;
    if (exact || (ex && atoi(ex))) {
      KernelScope ks("dis_gradient");
      k_dis_full<B><<<(unsigned)((K + 127) / 128), 128, 0, st>>>(s.keys(), s.coef(), s.M, s.filt, f4d, dc,
                                                                  K, dg);
    } else {
      // nibble tables of the groups holding qubits (the rest are all 1.0)
      const int ng = std::max(1, (nq + 3) / 4);
      double* nibt = ws.misc2.as<double>((size_t)ng * 256);
      k_nibble_table<<<(unsigned)((ng * 256 + 255) / 256), 256, 0, st>>>(f4d, ng, nibt);
      const size_t smem = (size_t)ng * 256 * sizeof(double);
      if (ratio) {
        if (func_attr_once((const void*)k_dis_ratio<B>, ctx_device(ctx_current())))
          IQCC_CUDA(cudaFuncSetAttribute(k_dis_ratio<B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         220 * 1024));
        KernelScope ks("dis_gradient");
        constexpr int kRatioNT = ratio_nt(B);
        const unsigned cbr = (unsigned)((K + kRatioNT - 1) / kRatioNT);
        const int Sr = (int)std::max<size_t>(1, std::min<size_t>({8, (148 * 4 + cbr - 1) / cbr, (s.M + 4095) / 4096}));
        k_dis_ratio<B><<<dim3(cbr, (unsigned)Sr), kRatioNT, smem_ratio, st>>>(s.keys(), s.coef(), s.M, s.filt, nibt,
                                                                              ng, dc, K, gpart);
        k_dis_fold<<<(unsigned)((K + 255) / 256), 256, 0, st>>>(gpart, K, Sr, dg);
        count_launch("dis_gradient");
        count_launch("dis_gradient");
      } else {
      if (func_attr_once((const void*)k_dis_nib<B>, ctx_device(ctx_current())))
        IQCC_CUDA(cudaFuncSetAttribute(k_dis_nib<B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(16 * B * 256 * sizeof(double))));
      KernelScope ks("dis_gradient");
      k_dis_nib<B><<<dim3(cb, (unsigned)S), 256, smem, st>>>(s.keys(), s.coef(), s.M, s.filt, nibt, ng, dc, K,
                                                             gpart);
      k_dis_fold<<<(unsigned)((K + 255) / 256), 256, 0, st>>>(gpart, K, S, dg);
      count_launch("dis_gradient");
      count_launch("dis_gradient");
      }
    }
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
  gradients_impl<B>(s, factors, crow.data(), K, poles, g.data(), true);  // the ranking: exact values
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


// ------------------------------------------------ polynomial kernels
// build_poly_kernels (iqcc/optimizer.hpp:340-368) over the device store:
//   h_kernel[a][b] = sum_i c_i i^(t1+t2) <omega| W_a P_i W_b |omega>
//   n_kernel[a][b] = i^tw <omega| W_a W_b |omega>
// for the t subset words W of a build_poly expansion, a <= b (b > a is the
// conjugate).  One (a, b) pair per thread; the block streams the store
// through shared-memory tiles and every lane of a warp reads the same staged
// term.  Per term the product W_a P W_b and its phase come from the same
// popcount rule as multiply_into (pauli.hpp:202-215); its expectation runs
// over U = supp(P) | (union of the warp's supp(W_a) | supp(W_b)) in ascending
// qubit order with identity positions multiplying by 1.0 (exact), so each
// per-term value is bit-identical to sandwich's (optimizer.hpp:288-333),
// including its complex arithmetic: (c + 0i)(pr + pi i) = (c pr - 0 pi,
// c pi + 0 pr), then times e, skipped when e == 0.  A pair's terms are summed
// in canonical order inside one chunk of the store; chunks (only when the
// pair count alone cannot fill the GPU) are summed on the host in order, so
// the result is bit-identical to the reference whenever one chunk covers the
// store.  At the poles only the run of terms whose x plane is x_a ^ x_b
// contributes (sandwich's binary search): one thread per pair walks that
// run, bit-identical always.
struct PolyPair {
  unsigned a, b;
};

template <int B>
__device__ __forceinline__ void sandwich_term(const Key<B>& wa, const Key<B>& wb, const Key<B>& k,
                                              Key<B>& w, int& t) {
  const Key<B> w1 = key_xor<B>(wa, k);
  t = (product_phase<B>(wa, k) + product_phase<B>(w1, wb)) & 3;
  w = key_xor<B>(w1, wb);
}

__device__ __forceinline__ void sandwich_add(double c, int t, double e, double& re, double& im) {
  const double pr = t == 0 ? 1.0 : (t == 2 ? -1.0 : 0.0);
  const double pi = t == 1 ? 1.0 : (t == 3 ? -1.0 : 0.0);
  const double vr = __dsub_rn(__dmul_rn(c, pr), __dmul_rn(0.0, pi));
  const double vi = __dadd_rn(__dmul_rn(c, pi), __dmul_rn(0.0, pr));
  re = __dadd_rn(re, __dmul_rn(vr, e));
  im = __dadd_rn(im, __dmul_rn(vi, e));
}

template <int B>
__global__ void __launch_bounds__(128) k_poly_h(const ull* __restrict__ keys,
                                                const double* __restrict__ coef, size_t M,
                                                Filter filt, const double* __restrict__ f4_g,
                                                const ull* __restrict__ words,
                                                const PolyPair* __restrict__ pairs, size_t np,
                                                size_t chunk, double* __restrict__ out) {
  constexpr int TT = 128;
  __shared__ double f4[4 * 64 * B];
  __shared__ ull tk[TT * 2 * B];
  __shared__ double tc[TT];
  for (int i = threadIdx.x; i < 4 * 64 * B; i += blockDim.x) f4[i] = f4_g[i];
  const size_t pid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  Key<B> wa, wb;
#pragma unroll
  for (int w = 0; w < 2 * B; ++w) wa.w[w] = wb.w[w] = 0;
  if (pid < np) {
    wa = load_key<B>(words, pairs[pid].a);
    wb = load_key<B>(words, pairs[pid].b);
  }
  ull up[B];
#pragma unroll
  for (int w = 0; w < B; ++w) {
    const ull s = wa.w[w] | wa.w[B + w] | wb.w[w] | wb.w[B + w];
    const unsigned lo = __reduce_or_sync(0xffffffffu, (unsigned)s);
    const unsigned hi = __reduce_or_sync(0xffffffffu, (unsigned)(s >> 32));
    up[w] = ((ull)hi << 32) | lo;
  }
  const size_t lo = blockIdx.y * chunk, hi = min(M, lo + chunk);
  double re = 0.0, im = 0.0;
  for (size_t base = lo; base < hi; base += TT) {
    __syncthreads();
    const size_t i = base + threadIdx.x;
    if (i < hi) {
      const Key<B> k = load_key<B>(keys, i);
      const double c = coef[i];
      const bool keep = filter_keep(filt, i, c, i == 0 && key_is_identity<B>(k));
#pragma unroll
      for (int w = 0; w < 2 * B; ++w) tk[(size_t)threadIdx.x * 2 * B + w] = k.w[w];
      tc[threadIdx.x] = keep ? c : dead_value();
    }
    __syncthreads();
    const int n = (int)min((size_t)TT, hi - base);
    // two staged terms per iteration: independent dmul chains (ILP); the
    // positions walked are the union of both supports and U, a term's
    // identity positions multiply by 1.0 (exact), and the two values are
    // added in canonical order
    for (int j = 0; j < n; j += 2) {
      const double c0 = tc[j];
      const double c1 = j + 1 < n ? tc[j + 1] : dead_value();
      const bool d0 = is_dead(c0), d1 = is_dead(c1);  // block-uniform
      if (d0 && d1) continue;
      Key<B> k0, k1;
#pragma unroll
      for (int w = 0; w < 2 * B; ++w) {
        k0.w[w] = d0 ? 0ull : tk[(size_t)j * 2 * B + w];
        k1.w[w] = d1 ? 0ull : tk[(size_t)(j + 1) * 2 * B + w];
      }
      Key<B> p0, p1;
      int t0, t1;
      sandwich_term<B>(wa, wb, k0, p0, t0);
      sandwich_term<B>(wa, wb, k1, p1, t1);
      double e0 = 1.0, e1 = 1.0;
#pragma unroll
      for (int w = 0; w < B; ++w) {
        ull s = k0.w[w] | k0.w[B + w] | k1.w[w] | k1.w[B + w] | up[w];
        while (s) {  // warp-uniform
          const int lz = __clzll((long long)s);
          const int bit = 63 - lz;
          const double* row = f4 + 4 * (64 * w + lz);
          const unsigned q0 = (unsigned)((p0.w[w] >> bit) & 1ull) | ((unsigned)((p0.w[B + w] >> bit) & 1ull) << 1);
          const unsigned q1 = (unsigned)((p1.w[w] >> bit) & 1ull) | ((unsigned)((p1.w[B + w] >> bit) & 1ull) << 1);
          e0 = __dmul_rn(e0, row[q0]);
          e1 = __dmul_rn(e1, row[q1]);
          s &= ~(1ull << bit);
        }
      }
      if (!d0 && e0 != 0.0) sandwich_add(c0, t0, e0, re, im);
      if (!d1 && e1 != 0.0) sandwich_add(c1, t1, e1, re, im);
    }
  }
  if (pid < np) {
    out[2 * (blockIdx.y * np + pid)] = re;
    out[2 * (blockIdx.y * np + pid) + 1] = im;
  }
}

// Poles: the x run [lower_bound(x_a ^ x_b), upper_bound) of the store.
template <int B>
__global__ void k_poly_h_poles(const ull* __restrict__ keys, const double* __restrict__ coef,
                               size_t M, Filter filt, const double* __restrict__ tab, int nq,
                               const ull* __restrict__ words, const PolyPair* __restrict__ pairs,
                               size_t np, double* __restrict__ out) {
  const size_t pid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (pid >= np) return;
  const Key<B> wa = load_key<B>(words, pairs[pid].a), wb = load_key<B>(words, pairs[pid].b);
  Key<B> tgt;
#pragma unroll
  for (int w = 0; w < B; ++w) {
    tgt.w[w] = wa.w[w] ^ wb.w[w];
    tgt.w[B + w] = 0;
  }
  size_t lo = 0, hi = M;
  while (lo < hi) {
    const size_t mid = (lo + hi) >> 1;
    if (cmp_x<B>(load_key<B>(keys, mid), tgt) < 0) lo = mid + 1; else hi = mid;
  }
  double re = 0.0, im = 0.0;
  for (size_t i = lo; i < M; ++i) {
    const Key<B> k = load_key<B>(keys, i);
    if (cmp_x<B>(k, tgt) != 0) break;
    const double c = coef[i];
    if (!filter_keep(filt, i, c, i == 0 && key_is_identity<B>(k))) continue;
    Key<B> prod;
    int t;
    sandwich_term<B>(wa, wb, k, prod, t);
    const double e = word_expect<B>(prod, tab);
    if (e != 0.0) sandwich_add(c, t, e, re, im);
  }
  out[2 * pid] = re;
  out[2 * pid + 1] = im;
}

// n_kernel: i^tw <W_a W_b> (complex times real: (pr e, pi e)).
template <int B>
__global__ void k_poly_n(const double* __restrict__ tab, const ull* __restrict__ words,
                         const PolyPair* __restrict__ pairs, size_t np, double* __restrict__ out) {
  const size_t pid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (pid >= np) return;
  const Key<B> wa = load_key<B>(words, pairs[pid].a), wb = load_key<B>(words, pairs[pid].b);
  const int t = product_phase<B>(wa, wb);
  const double e = word_expect<B>(key_xor<B>(wa, wb), tab);
  const double pr = t == 0 ? 1.0 : (t == 2 ? -1.0 : 0.0);
  const double pi = t == 1 ? 1.0 : (t == 3 ? -1.0 : 0.0);
  out[2 * pid] = __dmul_rn(pr, e);
  out[2 * pid + 1] = __dmul_rn(pi, e);
}

template <int B>
static void poly_impl(DeviceStore& s, const double* factors, bool poles, const uint64_t* words_rows,
                      size_t t, double* hk, double* nk, bool worker_local) {
  if (poles) store_materialize(s);  // the x-run search wants live keys only
  Workspace& ws = workspace();
  cudaStream_t st = stream();
  const int nq = (int)s.n_qubits;
  std::vector<ull> wk(t * 2 * B);
  for (size_t k = 0; k < t; ++k) row_to_device_key(words_rows + k * 2 * B, B, wk.data() + k * 2 * B);
  std::vector<PolyPair> pr;
  pr.reserve(t * (t + 1) / 2);
  for (unsigned a = 0; a < t; ++a)
    for (unsigned b = a; b < t; ++b) pr.push_back({a, b});
  const size_t np = pr.size();
  const unsigned pblocks = (unsigned)((np + 127) / 128);
  // chunks of >= 4096 terms, only as many as needed to fill 8 blocks (32
  // warps) per SM: the per-lane product is a dependent dmul chain, so the
  // kernel needs warps to hide its latency
  // IQCC_POLY_EXACT=1: one chunk, each pair summed in canonical order over
  // the whole store (bit-identical to the reference at any size, slower)
  const bool exact = getenv("IQCC_POLY_EXACT") && atoi(getenv("IQCC_POLY_EXACT")) != 0;
  size_t chunks = 1;
  if (!poles && !exact && s.M > 4096)
    chunks = std::min<size_t>((s.M + 4095) / 4096, std::max<size_t>(1, (148 * 8 + pblocks - 1) / pblocks));
  chunks = std::min<size_t>(chunks, 65535);
  const size_t chunk = chunks == 1 ? std::max<size_t>(s.M, 1) : (s.M + chunks - 1) / chunks;
  ull* dw = ws.misc3.as<ull>(std::max<size_t>(t, 1) * 2 * B);
  PolyPair* dp = ws.misc2.as<PolyPair>(std::max<size_t>(np, 1));
  double* tab = ws.tables.as<double>(3 * (size_t)std::max(nq, 1));
  double* part = ws.partials.as<double>(2 * np * chunks + 2 * np);
  double* dn = part + 2 * np * chunks;
  IQCC_CUDA(cudaMemcpyAsync(dw, wk.data(), wk.size() * sizeof(ull), cudaMemcpyHostToDevice, st));
  IQCC_CUDA(cudaMemcpyAsync(dp, pr.data(), np * sizeof(PolyPair), cudaMemcpyHostToDevice, st));
  IQCC_CUDA(cudaMemcpyAsync(tab, factors, 3 * nq * sizeof(double), cudaMemcpyHostToDevice, st));
  {
    KernelScope ks("poly_kernels");
    if (poles) {
      k_poly_h_poles<B><<<pblocks, 128, 0, st>>>(s.keys(), s.coef(), s.M, s.filt, tab, nq, dw, dp, np, part);
    } else {
      const std::vector<double> f4 = factor_rows(factors, nq, B);
      double* f4d = ws.grad_part.as<double>(f4.size());
      IQCC_CUDA(cudaMemcpyAsync(f4d, f4.data(), f4.size() * sizeof(double), cudaMemcpyHostToDevice, st));
      k_poly_h<B><<<dim3(pblocks, (unsigned)chunks), 128, 0, st>>>(s.keys(), s.coef(), s.M, s.filt, f4d, dw,
                                                                   dp, np, chunk, part);
    }
    k_poly_n<B><<<pblocks, 128, 0, st>>>(tab, dw, dp, np, dn);
    count_launch("poly_kernels");
  }
  const std::vector<double> h = fetch(part, 2 * np * chunks + 2 * np);
  const double* hn = h.data() + 2 * np * chunks;
  for (size_t p = 0; p < np; ++p) {
    double re = h[2 * p], im = h[2 * p + 1];  // chunk 0 as is (no +0 added)
    for (size_t c = 1; c < chunks; ++c) {
      re += h[2 * (c * np + p)];
      im += h[2 * (c * np + p) + 1];
    }
    const size_t a = pr[p].a, b = pr[p].b;
    if (worker_local) {  // partitioned form (optimizer.hpp:386-394): zeroed local += hv, += conj(hv) off the diagonal
      hk[2 * (a * t + b)] = 0.0 + re;
      hk[2 * (a * t + b) + 1] = 0.0 + im;
      if (b != a) {
        hk[2 * (b * t + a)] = 0.0 + re;
        hk[2 * (b * t + a) + 1] = 0.0 + -im;
      }
    } else {
      hk[2 * (a * t + b)] = re;
      hk[2 * (a * t + b) + 1] = im;
      hk[2 * (b * t + a)] = re;  // std::conj
      hk[2 * (b * t + a) + 1] = -im;
    }
    nk[2 * (a * t + b)] = hn[2 * p];
    nk[2 * (a * t + b) + 1] = hn[2 * p + 1];
    nk[2 * (b * t + a)] = hn[2 * p];
    nk[2 * (b * t + a) + 1] = -hn[2 * p + 1];
  }
}

void poly_kernels_store(DeviceStore& s, const double* factors, bool poles, const uint64_t* words,
                        size_t t, double* hk, double* nk, bool worker_local) {
  if (t == 0) return;
  switch (s.B) {
    case 1: poly_impl<1>(s, factors, poles, words, t, hk, nk, worker_local); break;
    case 2: poly_impl<2>(s, factors, poles, words, t, hk, nk, worker_local); break;
    default: poly_impl<4>(s, factors, poles, words, t, hk, nk, worker_local); break;
  }
}

}  // namespace iqcc_b200
