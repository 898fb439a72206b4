// io.cu — streaming Pauli text I/O and the FCIDUMP -> Jordan-Wigner ingest
// (iqcc/io.hpp:31-101, 154-276) feeding device term stores.
//
// Text is host work by nature (a file is read and written sequentially), so
// the host does exactly the reference's character-level steps —
// std::from_chars for coefficients, "%.17g" for writing them, the FCIDUMP
// record grammar — and the device does everything per term:
//   parse : letters -> key rows (one thread per term), then from_terms on
//           the device: a stable LSD radix sort of the key rows, duplicates
//           combined in file order, keep_term(1e-12), compaction;
//   write : key rows -> letter strings, chunk by chunk, while the host
//           formats and writes the previous chunk;
//   JW    : the one- and two-electron expansion (4 / 16 ladder products per
//           integral and spin pair, jordan_wigner :229-276) one thread per
//           (integral, spin pair), then the same device from_terms.
// from_terms combines duplicates in emission (file) order; the reference's
// std::sort leaves the order of equal words unspecified, so a word with
// three or more contributions can differ from it in the last bits of its
// sum (two addends commute exactly).  Real sums only: an imaginary part
// surviving the combination is rejected (the device stores real sums).
#include <algorithm>
#include <cctype>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "engine.cuh"

namespace iqcc_b200 {

namespace {

[[noreturn]] void parse_fail(const std::string& path, size_t line, const std::string& msg) {
  throw std::runtime_error(path + ":" + std::to_string(line) + ": " + msg);
}

uint32_t dev_blocks(size_t n) {
  const uint32_t b = n == 0 ? 1 : (uint32_t)((n + 63) / 64);
  return b == 3 ? 4 : b;
}

// ------------------------------------------------------ device from_terms
// Raw terms: key rows [N][2B] (device layout), complex coefficients [N][2].
// Stable LSD radix sort on 8-bit digits of every key word (least
// significant word first) through a permutation, then one thread per run of
// equal keys sums its coefficients in sorted (= emission) order.
constexpr int kSortPerBlock = 4096;

__global__ void k_ft_hist(const ull* __restrict__ keys, const unsigned* __restrict__ perm, size_t N, int W,
                          int word, int shift, unsigned* __restrict__ hist) {
  __shared__ unsigned h[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const size_t b0 = blockIdx.x * (size_t)kSortPerBlock;
  for (size_t i = b0 + threadIdx.x; i < min(N, b0 + kSortPerBlock); i += blockDim.x)
    atomicAdd(h + ((keys[(size_t)perm[i] * W + word] >> shift) & 255u), 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[(size_t)i * gridDim.x + blockIdx.x] = h[i];
}

// exclusive scan of the digit-major histogram (one block)
__global__ void __launch_bounds__(1024) k_ft_scan(unsigned* __restrict__ hist, size_t n) {
  __shared__ unsigned sm[1024 / 32 + 2];
  const size_t per = (n + 1023) / 1024;
  const size_t lo = threadIdx.x * per, hi = min(n, lo + per);
  unsigned c = 0;
  for (size_t k = lo; k < hi; ++k) c += hist[k];
  unsigned run = block_exclusive<1024>(c, 0u, OpAdd(), sm, (unsigned*)nullptr);
  for (size_t k = lo; k < hi; ++k) {
    const unsigned v = hist[k];
    hist[k] = run;
    run += v;
  }
}

// stable scatter: one warp per block walks its slice in order
__global__ void k_ft_scatter(const ull* __restrict__ keys, const unsigned* __restrict__ perm, size_t N, int W,
                             int word, int shift, const unsigned* __restrict__ hist,
                             unsigned* __restrict__ out) {
  __shared__ unsigned base[256];
  const int lane = threadIdx.x;
  for (int i = lane; i < 256; i += 32) base[i] = hist[(size_t)i * gridDim.x + blockIdx.x];
  __syncwarp();
  const size_t b0 = blockIdx.x * (size_t)kSortPerBlock, b1 = min(N, b0 + kSortPerBlock);
  for (size_t i0 = b0; i0 < b1; i0 += 32) {
    const size_t i = i0 + lane;
    const bool v = i < b1;
    const unsigned p = v ? perm[i] : 0u;
    const unsigned d = v ? (unsigned)((keys[(size_t)p * W + word] >> shift) & 255u) : 256u;
    // rank among lanes with the same digit (stable within the warp)
    const unsigned same = __match_any_sync(0xffffffffu, d);
    const unsigned before = __popc(same & ((1u << lane) - 1u));
    if (v) out[base[d] + before] = p;
    __syncwarp();
    if (v && before == 0) base[d] += __popc(same);
    __syncwarp();
  }
}

template <int B>
__global__ void k_ft_heads(const ull* __restrict__ keys, const unsigned* __restrict__ perm, size_t N,
                           unsigned char* __restrict__ head) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  head[i] = i == 0 || key_cmp<B>(load_key<B>(keys, perm[i - 1]), load_key<B>(keys, perm[i])) != 0;
}

// per head: the run's complex sum in sorted order, keep_term(thr) (identity
// always kept, |c| = hypot), imaginary residue flagged
template <int B>
__global__ void k_ft_combine(const ull* __restrict__ keys, const double* __restrict__ cf,
                             const unsigned* __restrict__ perm, const unsigned char* __restrict__ head, size_t N,
                             double thr, unsigned char* __restrict__ keep, double* __restrict__ sum_re,
                             ull* __restrict__ err) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  keep[i] = 0;
  if (!head[i]) return;
  double re = cf[2 * (size_t)perm[i]], im = cf[2 * (size_t)perm[i] + 1];
  for (size_t j = i + 1; j < N && !head[j]; ++j) {
    re = __dadd_rn(re, cf[2 * (size_t)perm[j]]);
    im = __dadd_rn(im, cf[2 * (size_t)perm[j] + 1]);
  }
  const Key<B> k = load_key<B>(keys, perm[i]);
  const bool id = key_is_identity<B>(k);
  bool kp = id || ((re != 0.0 || im != 0.0) && hypot(re, im) >= thr);
  if (kp && im != 0.0) atomicAdd(err, 1ull);
  keep[i] = kp;
  sum_re[i] = re;
}

template <int B>
__global__ void k_ft_emit(const ull* __restrict__ keys, const unsigned* __restrict__ perm,
                          const unsigned char* __restrict__ keep, const double* __restrict__ sum_re,
                          const unsigned* __restrict__ pos, size_t N, ull* __restrict__ okeys,
                          double* __restrict__ ocoef) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= N || !keep[i]) return;
  store_key<B>(okeys, pos[i], load_key<B>(keys, perm[i]));
  ocoef[pos[i]] = sum_re[i];
}

__global__ void k_iota(unsigned* __restrict__ p, size_t N) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i < N) p[i] = (unsigned)i;
}

// exclusive prefix of keep flags (block sums then a second pass)
__global__ void k_flag_sums(const unsigned char* __restrict__ f, size_t N, unsigned* __restrict__ bsum) {
  __shared__ unsigned sm[256 / 32 + 2];
  const size_t b0 = blockIdx.x * (size_t)2048;
  unsigned c = 0;
  for (int k = 0; k < 8; ++k) {
    const size_t i = b0 + (size_t)threadIdx.x * 8 + k;
    if (i < N) c += f[i];
  }
  unsigned tot;
  block_exclusive<256>(c, 0u, OpAdd(), sm, &tot);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

// exclusive scan of the block sums in place (one block) + the total
__global__ void __launch_bounds__(1024) k_flag_scan(unsigned* __restrict__ bsum, size_t nb,
                                                    unsigned* __restrict__ total) {
  __shared__ unsigned sm[1024 / 32 + 2];
  const size_t per = (nb + 1023) / 1024;
  const size_t lo = threadIdx.x * per, hi = min(nb, lo + per);
  unsigned c = 0;
  for (size_t k = lo; k < hi; ++k) c += bsum[k];
  unsigned tot;
  unsigned run = block_exclusive<1024>(c, 0u, OpAdd(), sm, &tot);
  for (size_t k = lo; k < hi; ++k) {
    const unsigned v = bsum[k];
    bsum[k] = run;
    run += v;
  }
  if (threadIdx.x == 0) *total = tot;
}

__global__ void k_flag_pos(const unsigned char* __restrict__ f, size_t N, const unsigned* __restrict__ bpfx,
                           unsigned* __restrict__ pos) {
  __shared__ unsigned sm[256 / 32 + 2];
  const size_t b0 = blockIdx.x * (size_t)2048;
  unsigned c[8], t = 0;
  for (int k = 0; k < 8; ++k) {
    const size_t i = b0 + (size_t)threadIdx.x * 8 + k;
    c[k] = i < N ? f[i] : 0u;
    t += c[k];
  }
  unsigned run = block_exclusive<256>(t, 0u, OpAdd(), sm, (unsigned*)nullptr) + bpfx[blockIdx.x];
  for (int k = 0; k < 8; ++k) {
    const size_t i = b0 + (size_t)threadIdx.x * 8 + k;
    if (i < N) pos[i] = run;
    run += c[k];
  }
}

/// from_terms (iqcc/pauli.hpp:302-326) of N raw device terms into s.
template <int B>
void from_terms_device(DeviceStore& s, size_t n_qubits, const ull* keys, const double* cf, size_t N,
                       double thr) {
  Workspace& ws = workspace();
  cudaStream_t st = stream();
  constexpr int W = 2 * B;
  s.n_qubits = (uint32_t)n_qubits;
  s.B = B;
  s.filt = Filter{};
  s.meta_valid = false;
  if (N == 0) {
    s.ensure(1);
    s.M = s.logical = 0;
    s.has_identity = false;
    return;
  }
  if (N > 0xFFFFFFF0ull) throw std::invalid_argument("from_terms: more than 2^32 raw terms");
  unsigned* perm = ws.inv_perm.as<unsigned>(N + 8);
  unsigned* perm2 = ws.rdelta.as<unsigned>(N + 8);
  const unsigned g256 = (unsigned)((N + 255) / 256);
  const unsigned nb = (unsigned)((N + kSortPerBlock - 1) / kSortPerBlock);
  unsigned* hist = ws.misc2.as<unsigned>((size_t)256 * nb + 8);
  {
    KernelScope ks("from_terms");
    k_iota<<<g256, 256, 0, st>>>(perm, N);
    for (int word = W - 1; word >= 0; --word)
      for (int shift = 0; shift < 64; shift += 8) {
        k_ft_hist<<<nb, 256, 0, st>>>(keys, perm, N, W, word, shift, hist);
        k_ft_scan<<<1, 1024, 0, st>>>(hist, (size_t)256 * nb);
        k_ft_scatter<<<nb, 32, 0, st>>>(keys, perm, N, W, word, shift, hist, perm2);
        std::swap(perm, perm2);
        count_launch("from_terms");
        count_launch("from_terms");
      }
  }
  unsigned char* head = ws.mbits.as<unsigned char>(2 * N + 16);
  unsigned char* keep = head + N + 8;
  double* sum_re = ws.stage_coef.as<double>(N);
  ull* err = ws.counters.as<ull>(16);
  IQCC_CUDA(cudaMemsetAsync(err, 0, sizeof(ull), st));
  const unsigned nfb = (unsigned)((N + 2047) / 2048);
  unsigned* bsum = ws.misc.as<unsigned>((size_t)nfb + 8);
  unsigned* pos = ws.tile_pfx.as<unsigned>(N + 8);
  unsigned* btot = bsum + nfb + 2;
  {
    KernelScope ks("from_terms");
    k_ft_heads<B><<<g256, 256, 0, st>>>(keys, perm, N, head);
    k_ft_combine<B><<<g256, 256, 0, st>>>(keys, cf, perm, head, N, thr, keep, sum_re, err);
    k_flag_sums<<<nfb, 256, 0, st>>>(keep, N, bsum);
    k_flag_scan<<<1, 1024, 0, st>>>(bsum, nfb, btot);
    k_flag_pos<<<nfb, 256, 0, st>>>(keep, N, bsum, pos);
  }
  ull h[2];
  IQCC_CUDA(cudaMemcpyAsync(h, err, sizeof(ull), cudaMemcpyDeviceToHost, st));
  unsigned total = 0;
  IQCC_CUDA(cudaMemcpyAsync(&total, btot, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
  host_sync(st);
  if (h[0]) throw std::runtime_error("from_terms: " + std::to_string(h[0]) +
                                     " combined coefficients keep an imaginary part; the device stores real sums");
  s.ensure(total);
  {
    KernelScope ks("from_terms");
    k_ft_emit<B><<<g256, 256, 0, st>>>(keys, perm, keep, sum_re, pos, N, s.keys(), s.coef());
  }
  s.M = s.logical = total;
  ull first[2 * kMaxB] = {};
  if (total) {
    IQCC_CUDA(cudaMemcpyAsync(first, s.keys(), W * sizeof(ull), cudaMemcpyDeviceToHost, st));
    host_sync(st);
  }
  bool id = total > 0;
  for (int w = 0; w < W; ++w) id = id && first[w] == 0;
  s.has_identity = id;
}

void from_terms_any(DeviceStore& s, size_t n_qubits, const ull* keys, const double* cf, size_t N, double thr) {
  switch (dev_blocks(n_qubits)) {
    case 1: from_terms_device<1>(s, n_qubits, keys, cf, N, thr); break;
    case 2: from_terms_device<2>(s, n_qubits, keys, cf, N, thr); break;
    default: from_terms_device<4>(s, n_qubits, keys, cf, N, thr); break;
  }
}

// -------------------------------------------------------- letters <-> rows
// letters [N][n] ('I','X','Y','Z'; validated on the host) -> device key rows
__global__ void k_letters_to_keys(const char* __restrict__ letters, size_t N, int n, int B,
                                  ull* __restrict__ keys) {
  const size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (t >= N) return;
  const char* s = letters + t * (size_t)n;
  for (int blk = 0; blk < B; ++blk) {
    ull x = 0, z = 0;
    for (int j = blk * 64; j < min(n, blk * 64 + 64); ++j) {
      const char c = s[j];
      const ull bit = 1ull << (63 - (j & 63));  // bit-reversed device word
      if (c == 'X' || c == 'Y') x |= bit;
      if (c == 'Z' || c == 'Y') z |= bit;
    }
    keys[t * 2 * B + blk] = x;
    keys[t * 2 * B + B + blk] = z;
  }
}

// device key rows [r0, r1) of a store -> letters [r1 - r0][n]
__global__ void k_keys_to_letters(const ull* __restrict__ keys, size_t r0, size_t r1, int n, int B,
                                  char* __restrict__ out) {
  const size_t t = r0 + blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (t >= r1) return;
  char* o = out + (t - r0) * (size_t)n;
  for (int j = 0; j < n; ++j) {
    const ull x = keys[t * 2 * B + j / 64], z = keys[t * 2 * B + B + j / 64];
    const int b = 63 - (j & 63);
    o[j] = "IXZY"[((x >> b) & 1ull) | (((z >> b) & 1ull) << 1)];
  }
}

// ---------------------------------------------------------- Jordan-Wigner
// Ladder operator on spin orbital p (jw_ladder, io.hpp:211-226): the terms
// 0.5 X_p Z_{<p} and (-+0.5 i) Y_p Z_{<p} (creation: -0.5i).
struct CTerm {
  ull w[8];  // device key (x blocks then z blocks)
  double re, im;
};

__device__ __forceinline__ void jw_term(int p, bool creation, int which, int B, CTerm& t) {
  for (int k = 0; k < 2 * B; ++k) t.w[k] = 0;
  for (int j = 0; j < p; ++j) t.w[B + j / 64] |= 1ull << (63 - (j & 63));  // Z string
  t.w[p / 64] |= 1ull << (63 - (p & 63));                                  // X
  if (which == 0) {
    t.re = 0.5;
    t.im = 0.0;
  } else {
    t.w[B + p / 64] |= 1ull << (63 - (p & 63));  // Y = X with a z bit
    t.re = 0.0;
    t.im = creation ? -0.5 : 0.5;
  }
}

// std::complex<double> product (a + bi)(c + di) = (ac - bd) + (ad + bc)i
__device__ __forceinline__ void cmul(double a, double b, double c, double d, double& re, double& im) {
  re = __dsub_rn(__dmul_rn(a, c), __dmul_rn(b, d));
  im = __dadd_rn(__dmul_rn(a, d), __dmul_rn(b, c));
}

// word product + phase (multiply_into, pauli.hpp:202-215) as a complex factor
__device__ __forceinline__ void wmul(const CTerm& a, const ull* bw, int B, ull* out, double& pr, double& pi) {
  int t = 0;
  for (int k = 0; k < B; ++k) {
    const ull px = a.w[k], pz = a.w[B + k], qx = bw[k], qz = bw[B + k];
    const ull rx = px ^ qx, rz = pz ^ qz;
    t += __popcll(px & pz) + __popcll(qx & qz) - __popcll(rx & rz) + 2 * __popcll(pz & qx);
    out[k] = rx;
    out[B + k] = rz;
  }
  t = ((t % 4) + 4) % 4;
  const double tab_re[4] = {1, 0, -1, 0}, tab_im[4] = {0, 1, 0, -1};
  pr = tab_re[t];
  pi = tab_im[t];
}

struct JWArgs {
  int n_so, B;
  const int* one;     // [n1][3] = (p, q, spin)
  const double* h1;   // [n1] integral values
  size_t n1;
  const int* two;     // [n2][6] = (p, q, r, s, sa, sb)
  const double* g2;   // [n2]
  size_t n2;
  ull* keys;          // out [4 n1 + 16 n2][2B]
  double* cf;         // out [..][2]
};

// one-body: emit2(cre[2p+sp], ann[2q+sp], h) (io.hpp:247-253)
__global__ void k_jw_one(JWArgs a) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= a.n1) return;
  const int p = a.one[3 * i], q = a.one[3 * i + 1], sp = a.one[3 * i + 2];
  const double scale = a.h1[i];
  size_t o = i * 4;
  for (int x = 0; x < 2; ++x) {
    CTerm ta;
    jw_term(2 * p + sp, true, x, a.B, ta);
    for (int y = 0; y < 2; ++y) {
      CTerm tb;
      jw_term(2 * q + sp, false, y, a.B, tb);
      ull w[8];
      double pr, pi;
      wmul(ta, tb.w, a.B, w, pr, pi);
      // scale * ta.coeff * tb.coeff * prod.phase(), left to right
      double r1, i1, r2, i2, r3, i3;
      cmul(scale, 0.0, ta.re, ta.im, r1, i1);
      cmul(r1, i1, tb.re, tb.im, r2, i2);
      cmul(r2, i2, pr, pi, r3, i3);
      for (int k = 0; k < 2 * a.B; ++k) a.keys[o * 2 * a.B + k] = w[k];
      a.cf[2 * o] = r3;
      a.cf[2 * o + 1] = i3;
      ++o;
    }
  }
}

// two-body: emit4(cre[2p+sa], cre[2r+sb], ann[2s+sb], ann[2q+sa], 0.5 g) (io.hpp:255-273)
__global__ void k_jw_two(JWArgs a) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= a.n2) return;
  const int* t6 = a.two + 6 * i;
  const int p = t6[0], q = t6[1], r = t6[2], s = t6[3], sa = t6[4], sb = t6[5];
  const double scale = __dmul_rn(0.5, a.g2[i]);
  const int B = a.B;
  size_t o = i * 16 + a.n1 * 4;
  for (int x = 0; x < 2; ++x) {
    CTerm ta;
    jw_term(2 * p + sa, true, x, B, ta);
    for (int y = 0; y < 2; ++y) {
      CTerm tb;
      jw_term(2 * r + sb, true, y, B, tb);
      CTerm ab;
      double pr, pi;
      wmul(ta, tb.w, B, ab.w, pr, pi);
      double c1r, c1i, cabr, cabi;
      cmul(ta.re, ta.im, tb.re, tb.im, c1r, c1i);  // ta.coeff * tb.coeff
      cmul(c1r, c1i, pr, pi, cabr, cabi);          // * ab.phase()
      for (int z = 0; z < 2; ++z) {
        CTerm tc;
        jw_term(2 * s + sb, false, z, B, tc);
        CTerm abc;
        wmul(ab, tc.w, B, abc.w, pr, pi);
        double c2r, c2i, cabcr, cabci;
        cmul(cabr, cabi, tc.re, tc.im, c2r, c2i);  // cab * tc.coeff
        cmul(c2r, c2i, pr, pi, cabcr, cabci);      // * abc.phase()
        for (int u = 0; u < 2; ++u) {
          CTerm td;
          jw_term(2 * q + sa, false, u, B, td);
          ull w[8];
          wmul(abc, td.w, B, w, pr, pi);
          // scale * cabc * td.coeff * abcd.phase(), left to right
          double r1, i1, r2, i2, r3, i3;
          cmul(scale, 0.0, cabcr, cabci, r1, i1);
          cmul(r1, i1, td.re, td.im, r2, i2);
          cmul(r2, i2, pr, pi, r3, i3);
          for (int k = 0; k < 2 * B; ++k) a.keys[o * 2 * B + k] = w[k];
          a.cf[2 * o] = r3;
          a.cf[2 * o + 1] = i3;
          ++o;
        }
      }
    }
  }
}

/// FCIDUMP reader (read_fcidump, io.hpp:154-205): header through &END or a
/// '/', NORB / NELEC / MS2 fields, then `value i j k l` records (1-based;
/// 0 0 0 0 = core energy; k = l = 0 one-electron; else two-electron with
/// its eight symmetric images).
struct Integrals {
  long norb = 0, nelec = 0, ms2 = 0;
  double core = 0.0;
  std::vector<double> h, g;
  double& hx(long p, long q) { return h[p * norb + q]; }
  double& gx(long p, long q, long r, long s) { return g[((p * norb + q) * norb + r) * norb + s]; }
};

Integrals read_fcidump_host(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open " + path);
  std::string header, line;
  size_t lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    header += line + " ";
    if (line.find("&END") != std::string::npos || line.find('/') != std::string::npos) break;
    if (lineno > 100) parse_fail(path, lineno, "unterminated FCIDUMP header");
  }
  auto field = [&](const char* key, long& out) {
    const std::string k = std::string(key) + "=";
    const size_t pos = header.find(k);
    if (pos == std::string::npos) return false;
    out = std::strtol(header.c_str() + pos + k.size(), nullptr, 10);
    return true;
  };
  Integrals I;
  if (!field("NORB", I.norb) || I.norb <= 0) parse_fail(path, lineno, "missing NORB");
  if (!field("NELEC", I.nelec) || I.nelec < 0) parse_fail(path, lineno, "missing NELEC");
  field("MS2", I.ms2);
  const long n = I.norb;
  I.h.assign((size_t)n * n, 0.0);
  I.g.assign((size_t)n * n * n * n, 0.0);
  while (std::getline(in, line)) {
    ++lineno;
    if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
    std::istringstream ls(line);
    double v;
    long i, j, k, l;
    if (!(ls >> v >> i >> j >> k >> l)) parse_fail(path, lineno, "bad integral record");
    if (i == 0 && j == 0 && k == 0 && l == 0) {
      I.core = v;
    } else if (k == 0 && l == 0) {
      if (i < 1 || i > n || j < 1 || j > n) parse_fail(path, lineno, "orbital index out of range");
      I.hx(i - 1, j - 1) = v;
      I.hx(j - 1, i - 1) = v;
    } else {
      if (i < 1 || i > n || j < 1 || j > n || k < 1 || k > n || l < 1 || l > n)
        parse_fail(path, lineno, "orbital index out of range");
      const long a[2][2] = {{i - 1, j - 1}, {j - 1, i - 1}}, b[2][2] = {{k - 1, l - 1}, {l - 1, k - 1}};
      for (auto& x : a)
        for (auto& y : b) {
          I.gx(x[0], x[1], y[0], y[1]) = v;
          I.gx(y[0], y[1], x[0], x[1]) = v;
        }
    }
  }
  // IntegralSet::validate_symmetry (io.hpp:123-143)
  const double tol = 1e-10;
  for (long p = 0; p < n; ++p)
    for (long q = 0; q < n; ++q)
      if (std::abs(I.hx(p, q) - I.hx(q, p)) > tol) throw std::runtime_error("integral symmetry violation in h");
  for (long p = 0; p < n; ++p)
    for (long q = 0; q < n; ++q)
      for (long r = 0; r < n; ++r)
        for (long s = 0; s < n; ++s) {
          const double v = I.gx(p, q, r, s);
          if (std::abs(v - I.gx(q, p, r, s)) > tol || std::abs(v - I.gx(p, q, s, r)) > tol ||
              std::abs(v - I.gx(r, s, p, q)) > tol)
            throw std::runtime_error("integral symmetry violation in g");
        }
  return I;
}

}  // namespace

// ------------------------------------------------------------------ entry
void store_read_pauli_file(DeviceStore& s, const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open " + path);
  std::vector<char> letters;
  std::vector<double> cf;  // re, im pairs
  size_t n_qubits = 0;
  bool have_width = false;
  std::string line;
  size_t lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    const size_t first = line.find_first_not_of(" \t\r");
    if (first == std::string::npos) continue;
    if (line[first] == '#') {  // "# qubits: N" pins the width
      std::istringstream hdr(line.substr(first + 1));
      std::string key;
      size_t n;
      if (hdr >> key >> n && key == "qubits:") {
        n_qubits = n;
        have_width = true;
      }
      continue;
    }
    std::istringstream ls(line);
    std::string cs, word, rest;
    if (!(ls >> cs >> word)) parse_fail(path, lineno, "expected `<coefficient> <letters>`");
    if (ls >> rest) parse_fail(path, lineno, "trailing content '" + rest + "'");
    double c;
    const auto r = std::from_chars(cs.data(), cs.data() + cs.size(), c);
    if (r.ec != std::errc{} || r.ptr != cs.data() + cs.size()) parse_fail(path, lineno, "bad coefficient '" + cs + "'");
    if (!std::isfinite(c)) parse_fail(path, lineno, "non-finite coefficient");
    if (!have_width) {
      n_qubits = word.size();
      have_width = true;
    } else if (word.size() != n_qubits) {
      parse_fail(path, lineno, "inconsistent string length (expected " + std::to_string(n_qubits) + ")");
    }
    for (char ch : word)
      if (ch != 'I' && ch != 'X' && ch != 'Y' && ch != 'Z')
        parse_fail(path, lineno, std::string("invalid Pauli letter '") + ch + "'");
    letters.insert(letters.end(), word.begin(), word.end());
    cf.push_back(c);
    cf.push_back(0.0);
  }
  if (!have_width) throw std::runtime_error(path + ": no terms and no `# qubits:` header");
  if (n_qubits > 256) throw std::invalid_argument("more than 256 qubits are not supported");
  const size_t N = cf.size() / 2;
  const uint32_t B = dev_blocks(n_qubits);
  Workspace& ws = workspace();
  cudaStream_t st = stream();
  ull* keys = ws.xbuf_keys.as<ull>(std::max<size_t>(N, 1) * 2 * B);
  double* dcf = ws.xbuf_coef.as<double>(std::max<size_t>(N, 1) * 2);
  if (N) {
    char* dl = ws.stage_rows.as<char>(letters.size() + 8);
    IQCC_CUDA(cudaMemcpyAsync(dl, letters.data(), letters.size(), cudaMemcpyHostToDevice, st));
    IQCC_CUDA(cudaMemcpyAsync(dcf, cf.data(), cf.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    KernelScope ks("io_parse");
    k_letters_to_keys<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(dl, N, (int)n_qubits, (int)B, keys);
  }
  from_terms_any(s, n_qubits, keys, dcf, N, 1e-12);
}

void store_write_pauli_file(DeviceStore& s, const std::string& path) {
  // canonical live terms (device compaction), then chunks of letter strings
  // rendered by the device while the host writes the previous chunk
  store_materialize(s);
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot open " + path + " for writing");
  out << "# qubits: " << s.n_qubits << "\n";
  const size_t N = s.logical, n = s.n_qubits;
  cudaStream_t st = stream();
  Workspace& ws = workspace();
  const size_t chunk = std::max<size_t>(1, std::min<size_t>(N, (size_t)(64u << 20) / std::max<size_t>(n, 1)));
  std::vector<double> coef(N);
  if (N) IQCC_CUDA(cudaMemcpyAsync(coef.data(), s.coef(), N * sizeof(double), cudaMemcpyDeviceToHost, st));
  char* dl = ws.stage_rows.as<char>(2 * chunk * std::max<size_t>(n, 1) + 8);
  char* hl = static_cast<char*>(host_pinned(2 * chunk * std::max<size_t>(n, 1) + 8));
  auto render = [&](size_t c0, int slot) {
    const size_t c1 = std::min(N, c0 + chunk);
    char* d = dl + (size_t)slot * chunk * n;
    KernelScope ks("io_write");
    k_keys_to_letters<<<(unsigned)((c1 - c0 + 255) / 256), 256, 0, st>>>(s.keys(), c0, c1, (int)n, (int)s.B, d);
    IQCC_CUDA(cudaMemcpyAsync(hl + (size_t)slot * chunk * n, d, (c1 - c0) * n, cudaMemcpyDeviceToHost, st));
  };
  cudaEvent_t ready[2];
  IQCC_CUDA(cudaEventCreateWithFlags(&ready[0], cudaEventDisableTiming));
  IQCC_CUDA(cudaEventCreateWithFlags(&ready[1], cudaEventDisableTiming));
  if (N) {
    render(0, 0);
    IQCC_CUDA(cudaEventRecord(ready[0], st));
  }
  std::string buf;
  char num[64];
  int slot = 0;
  for (size_t c0 = 0; c0 < N; c0 += chunk, slot ^= 1) {
    const size_t c1 = std::min(N, c0 + chunk);
    if (c1 < N) {  // next chunk on the device while this one is written
      render(c1, slot ^ 1);
      IQCC_CUDA(cudaEventRecord(ready[slot ^ 1], st));
    }
    IQCC_CUDA(cudaEventSynchronize(ready[slot]));
    buf.clear();
    const char* lt = hl + (size_t)slot * chunk * n;
    for (size_t i = c0; i < c1; ++i) {
      std::snprintf(num, sizeof num, "%.17g", coef[i]);  // write_pauli_file's format
      buf += num;
      buf += ' ';
      buf.append(lt + (i - c0) * n, n);
      buf += '\n';
    }
    out.write(buf.data(), (std::streamsize)buf.size());
  }
  cudaEventDestroy(ready[0]);
  cudaEventDestroy(ready[1]);
  if (!out) throw std::runtime_error("write failed: " + path);
}

size_t store_jordan_wigner_fcidump(DeviceStore& s, const std::string& path) {
  Integrals I = read_fcidump_host(path);
  const long n = I.norb;
  const int n_so = (int)(2 * n);
  if (n_so > 256) throw std::invalid_argument("more than 256 qubits are not supported");
  const uint32_t B = dev_blocks((size_t)n_so);
  // nonzero integrals in the reference's loop order (io.hpp:247-273)
  std::vector<int> one, two;
  std::vector<double> h1, g2;
  for (long p = 0; p < n; ++p)
    for (long q = 0; q < n; ++q) {
      const double v = I.hx(p, q);
      if (std::abs(v) < 1e-14) continue;
      for (int sp = 0; sp < 2; ++sp) {
        one.insert(one.end(), {(int)p, (int)q, sp});
        h1.push_back(v);
      }
    }
  for (long p = 0; p < n; ++p)
    for (long q = 0; q < n; ++q)
      for (long r = 0; r < n; ++r)
        for (long t = 0; t < n; ++t) {
          const double v = I.gx(p, q, r, t);
          if (std::abs(v) < 1e-14) continue;
          for (int sa = 0; sa < 2; ++sa)
            for (int sb = 0; sb < 2; ++sb) {
              two.insert(two.end(), {(int)p, (int)q, (int)r, (int)t, sa, sb});
              g2.push_back(v);
            }
        }
  const size_t n1 = h1.size(), n2 = g2.size();
  const size_t N = 1 + 4 * n1 + 16 * n2;  // the core-energy identity term first
  Workspace& ws = workspace();
  cudaStream_t st = stream();
  ull* keys = ws.xbuf_keys.as<ull>(N * 2 * B + 8);
  double* cf = ws.xbuf_coef.as<double>(2 * N + 8);
  int* dint = ws.levels.as<int>(one.size() + two.size() + 8);
  double* dval = ws.partials.as<double>(n1 + n2 + 8);
  IQCC_CUDA(cudaMemcpyAsync(dint, one.data(), one.size() * sizeof(int), cudaMemcpyHostToDevice, st));
  IQCC_CUDA(cudaMemcpyAsync(dint + one.size(), two.data(), two.size() * sizeof(int), cudaMemcpyHostToDevice, st));
  IQCC_CUDA(cudaMemcpyAsync(dval, h1.data(), n1 * sizeof(double), cudaMemcpyHostToDevice, st));
  IQCC_CUDA(cudaMemcpyAsync(dval + n1, g2.data(), n2 * sizeof(double), cudaMemcpyHostToDevice, st));
  // term 0: core_energy * identity
  std::vector<ull> zero(2 * B, 0);
  IQCC_CUDA(cudaMemcpyAsync(keys, zero.data(), 2 * B * sizeof(ull), cudaMemcpyHostToDevice, st));
  const double core[2] = {I.core, 0.0};
  IQCC_CUDA(cudaMemcpyAsync(cf, core, sizeof(core), cudaMemcpyHostToDevice, st));
  JWArgs a{n_so, (int)B, dint, dval, n1, dint + one.size(), dval + n1, n2, keys + 2 * B, cf + 2};
  {
    KernelScope ks("jordan_wigner");
    if (n1) k_jw_one<<<(unsigned)((n1 + 127) / 128), 128, 0, st>>>(a);
    if (n2) k_jw_two<<<(unsigned)((n2 + 127) / 128), 128, 0, st>>>(a);
  }
  IQCC_CUDA(cudaStreamSynchronize(st));
  from_terms_any(s, (size_t)n_so, keys, cf, N, 1e-12);
  return (size_t)I.nelec;
}

}  // namespace iqcc_b200
