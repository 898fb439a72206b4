// engine.cuh — shared device helpers and host context of the B200 iQCC engine.
//
// Device term store (one per sum / shard): key rows [M][2B] uint64 holding the
// BIT-REVERSED words of the reference row (x blocks then z blocks,
// iqcc/pauli.hpp:373-377), and coef [M] fp64 (real part).
// Bit reversal maps the reference's canonical order (iqcc/pauli.hpp:146-161:
// lowest differing bit most significant, x plane first) onto plain
// lexicographic unsigned order of the rows, so comparisons are word compares
// and the first differing canonical position is 64*w + clz(a^b).
// popcount-based algebra (commutation, product phase) is invariant under the
// reversal.  Rows are 16/32/64 B for B = 1/2/4, loaded as 128-bit vectors;
// a random access to a 124-qubit row touches exactly one 32 B sector.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <functional>
#include <vector>

#include "../../include/iqcc_b200.h"

namespace iqcc_b200 {

typedef unsigned long long ull;

constexpr int kMaxB = 4;        // up to 256 qubits
constexpr int kLevelsPerChunk = 8;
constexpr int kThrPerChunk = 2 * kLevelsPerChunk;

template <int B>
struct Key {
  ull w[2 * B];
};

template <int B>
__device__ __forceinline__ Key<B> load_key(const ull* __restrict__ keys, size_t i) {
  Key<B> k;
  const ulonglong2* p = reinterpret_cast<const ulonglong2*>(keys + i * (2 * B));
#pragma unroll
  for (int j = 0; j < B; ++j) {
    ulonglong2 v = __ldg(p + j);
    k.w[2 * j] = v.x;
    k.w[2 * j + 1] = v.y;
  }
  return k;
}

template <int B>
__device__ __forceinline__ void store_key(ull* __restrict__ keys, size_t i, const Key<B>& k) {
  ulonglong2* p = reinterpret_cast<ulonglong2*>(keys + i * (2 * B));
#pragma unroll
  for (int j = 0; j < B; ++j) p[j] = make_ulonglong2(k.w[2 * j], k.w[2 * j + 1]);
}

template <int B>
__device__ __forceinline__ int key_cmp(const Key<B>& a, const Key<B>& b) {
#pragma unroll
  for (int w = 0; w < 2 * B; ++w)
    if (a.w[w] != b.w[w]) return a.w[w] < b.w[w] ? -1 : 1;
  return 0;
}

template <int B>
__device__ __forceinline__ bool key_is_identity(const Key<B>& a) {
  ull o = 0;
#pragma unroll
  for (int w = 0; w < 2 * B; ++w) o |= a.w[w];
  return o == 0;
}

/// First differing canonical position (0 = x bit of qubit 0), or 0x7fff when equal.
template <int B>
__device__ __forceinline__ int key_lcp(const Key<B>& a, const Key<B>& b) {
  int r = 0x7fff;
#pragma unroll
  for (int w = 2 * B - 1; w >= 0; --w) {
    ull d = a.w[w] ^ b.w[w];
    if (d) r = 64 * w + __clzll((long long)d);
  }
  return r;
}

/// Symplectic product parity (commutes, iqcc/pauli.hpp:188-193): 1 = anticommute.
template <int B>
__device__ __forceinline__ int anticommutes(const Key<B>& k, const Key<B>& p) {
  int s = 0;
#pragma unroll
  for (int b = 0; b < B; ++b) s += __popcll((k.w[b] & p.w[B + b]) ^ (k.w[B + b] & p.w[b]));
  return s & 1;
}

/// Phase exponent t of k*p = i^t (k^p) (multiply_into, iqcc/pauli.hpp:202-215), mod 4.
template <int B>
__device__ __forceinline__ int product_phase(const Key<B>& k, const Key<B>& p) {
  int t = 0;
#pragma unroll
  for (int b = 0; b < B; ++b) {
    ull kx = k.w[b], kz = k.w[B + b], px = p.w[b], pz = p.w[B + b];
    t += __popcll(kx & kz) + __popcll(px & pz) - __popcll((kx ^ px) & (kz ^ pz)) +
         2 * __popcll(kz & px);
  }
  return t & 3;
}

template <int B>
__device__ __forceinline__ Key<B> key_xor(const Key<B>& a, const Key<B>& b) {
  Key<B> r;
#pragma unroll
  for (int w = 0; w < 2 * B; ++w) r.w[w] = a.w[w] ^ b.w[w];
  return r;
}

/// Bit at canonical position pos (0 .. 128B-1).
template <int B>
__device__ __forceinline__ unsigned key_bit(const Key<B>& k, int pos) {
  int w = pos >> 6;
  ull v = 0;
#pragma unroll
  for (int j = 0; j < 2 * B; ++j) v = (j == w) ? k.w[j] : v;
  return (unsigned)(v >> (63 - (pos & 63))) & 1u;
}

/// Lazy compress filter attached to a store (compress, iqcc/pauli.hpp:425-474):
/// keep(i) = identity || !active || (|c| >= eps && (!has_v || |c| > v ||
/// (|c| == v && i <= cut))).  |c| of a real coefficient is std::abs(complex)
/// exactly (hypot(re, 0) == |re|).
struct Filter {
  int active = 0;
  int has_v = 0;
  double eps = 0.0;
  double v = 0.0;
  long long cut = 0;  // last kept index among |c| == v (-1: none)
};

/// Dead slot: a term removed by a dressing step (cancelled partner or below
/// the drop threshold) whose slot was kept so that every output tile's
/// offset is known before the merge runs.  Encoded as a NaN payload that a
/// live coefficient never carries (uploads reject NaN); the next step skips
/// dead slots and does not re-emit them.
constexpr ull kDeadBits = 0x7FF4DEAD0000DEADull;
__device__ __forceinline__ bool is_dead(double c) {
  return (ull)__double_as_longlong(c) == kDeadBits;
}
__device__ __forceinline__ double dead_value() { return __longlong_as_double((long long)kDeadBits); }

__device__ __forceinline__ bool filter_keep(const Filter& f, size_t i, double c, bool identity) {
  if (is_dead(c)) return false;
  if (identity || !f.active) return true;
  double a = fabs(c);
  if (!(a >= f.eps)) return false;
  if (!f.has_v) return true;
  return a > f.v || (a == f.v && (long long)i <= f.cut);
}

/// Coarse |c| histogram bin for compress(): the IEEE exponent of |c|
/// offset so 2^-192 .. 2^63 map to bins 1..254; smaller/larger values
/// collect in bins 0/255 (the select then refines over all 63 bits).
constexpr int kHistBins = 256;
__device__ __forceinline__ unsigned hist_bin(double a) {
  const int e = (int)((ull)__double_as_longlong(a) >> 52) - (1023 - 192);
  return (unsigned)min(max(e, 0), kHistBins - 1);
}

/// Fine |c| histogram of the merge for the compress select: the 4 exponent
/// bins from the speculated cut floor's bin up, 16 sub-bins each (the top 4
/// mantissa bits), appended to the 256-bin histogram.  The select then
/// starts with exponent + 4 mantissa bits fixed (16x fewer candidates).
constexpr int kSubBinsPer = 16, kSubWindow = 4, kSubBins = kSubBinsPer * kSubWindow;
constexpr int kSubBits = 4;  // log2(kSubBinsPer)
__host__ __device__ inline int hist_bin_of(double a) {
  unsigned long long b;
  memcpy(&b, &a, 8);
  const int e = (int)(b >> 52) - (1023 - 192);
  return e < 0 ? 0 : (e > kHistBins - 1 ? kHistBins - 1 : e);
}
/// window start (exponent bin) of the last merge's fine histogram; < 0: none
int merge_sub_window();

/// keep_term (iqcc/pauli.hpp:180-184) for a real coefficient.
__device__ __forceinline__ bool keep_term(double c, bool identity, double thr) {
  if (identity) return true;
  if (c == 0.0) return false;
  return fabs(c) >= thr;
}

// ---------------------------------------------------------------- scans
template <class T, class Op>
__device__ __forceinline__ T warp_inclusive(T v, Op op) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v = op(n, v);
  }
  return v;
}

template <class T, class Op>
__device__ __forceinline__ T warp_inclusive_rev(T v, Op op) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_down_sync(0xffffffffu, v, o);
    if (lane + o < 32) v = op(v, n);
  }
  return v;
}

/// Block-wide exclusive scan (NT threads, NT % 32 == 0); `scratch` holds NT/32+1 T.
template <int NT, class T, class Op>
__device__ __forceinline__ T block_exclusive(T v, T identity, Op op, T* scratch, T* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T inc = warp_inclusive(v, op);
  if (lane == 31) scratch[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T s = lane < NT / 32 ? scratch[lane] : identity;
    T si = warp_inclusive(s, op);
    if (lane < NT / 32) scratch[lane] = si;
  }
  __syncthreads();
  T base = warp > 0 ? scratch[warp - 1] : identity;
  T excl_in_warp = __shfl_up_sync(0xffffffffu, inc, 1);
  if (lane == 0) excl_in_warp = identity;
  T out = op(base, excl_in_warp);
  if (total) *total = scratch[NT / 32 - 1];
  __syncthreads();
  return out;
}

/// Block-wide exclusive scan from the right (thread NT-1 first).
template <int NT, class T, class Op>
__device__ __forceinline__ T block_exclusive_rev(T v, T identity, Op op, T* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T inc = warp_inclusive_rev(v, op);
  if (lane == 0) scratch[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T s = lane < NT / 32 ? scratch[lane] : identity;
    // reverse inclusive over warps: combine with higher warp ids
    T si = s;
    for (int o = 1; o < 32; o <<= 1) {
      T n = __shfl_down_sync(0xffffffffu, si, o);
      if (lane + o < NT / 32) si = op(si, n);
    }
    if (lane < NT / 32) scratch[lane] = si;
  }
  __syncthreads();
  T base = warp + 1 < NT / 32 ? scratch[warp + 1] : identity;
  T excl_in_warp = __shfl_down_sync(0xffffffffu, inc, 1);
  if (lane == 31) excl_in_warp = identity;
  T out = op(excl_in_warp, base);
  __syncthreads();
  return out;
}

struct OpAdd {
  template <class T>
  __device__ __forceinline__ T operator()(T a, T b) const { return a + b; }
};
struct OpMax {
  __device__ __forceinline__ int operator()(int a, int b) const { return a > b ? a : b; }
  __device__ __forceinline__ long long operator()(long long a, long long b) const { return a > b ? a : b; }
};
struct OpMin {
  __device__ __forceinline__ int operator()(int a, int b) const { return a < b ? a : b; }
  __device__ __forceinline__ long long operator()(long long a, long long b) const { return a < b ? a : b; }
};

/// Decoupled look-back (single-pass prefix over tiles processed in
/// dynamic-id order).  status[t]: bits 63:62 = 0 invalid / 1 aggregate /
/// 2 inclusive prefix, bits 61:0 = value.  Called by ALL 32 lanes of ONE
/// warp per tile: each probe reads 32 predecessors in parallel and stops at
/// the nearest one carrying an inclusive prefix.  Returns the exclusive
/// prefix to every lane.
__device__ __forceinline__ ull ld_acquire(const ull* p) {
  ull v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(ull* p, ull v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ ull lookback_warp(ull* status, ull tile, ull agg) {
  const ull AGG = 1ull << 62, PFX = 2ull << 62, VAL = (1ull << 62) - 1;
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) st_release(status, PFX | agg);
    return 0;
  }
  if (lane == 0) st_release(status + tile, AGG | agg);
  ull excl = 0;
  long long end = (long long)tile - 1;
  for (;;) {
    const long long idx = end - lane;
    ull v = idx >= 0 ? ld_acquire(status + idx) : PFX;
    while (__any_sync(0xffffffffu, (v & ~VAL) == 0)) {
      if ((v & ~VAL) == 0) v = ld_acquire(status + idx);
    }
    const unsigned pm = __ballot_sync(0xffffffffu, (v & ~VAL) == PFX);
    ull part = v & VAL;
    if (pm) {
      const int first = __ffs(pm) - 1;
      if (lane > first) part = 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    excl += part;
    if (pm) break;
    end -= 32;
  }
  if (lane == 0) st_release(status + tile, PFX | (excl + agg));
  return excl;
}

// ---------------------------------------------------------------- debug
// Bounds checks on scattered writes: a violation records (site, index,
// bound) in dbg[0..2] and the write is skipped (see iqcc_gpu debug_check).
__device__ __forceinline__ bool dbg_ok(ull* dbg, unsigned site, ull idx, ull bound) {
  if (idx < bound) return true;
  if (atomicCAS(dbg, 0ull, (ull)site) == 0ull) {
    dbg[1] = idx;
    dbg[2] = bound;
  }
  return false;
}

// ---------------------------------------------------------------- host side
struct Ctx;
Ctx& ctx();
cudaStream_t stream();
/// Engine contexts (one per host thread, see capi.cu): create one on a
/// device, bind it to the calling thread (returns the previous binding),
/// free it (its stream, scratch and cached blocks).
Ctx* ctx_new(int device);
Ctx* ctx_bind(Ctx* c);
Ctx* ctx_current();
int ctx_device(const Ctx* c);
void ctx_free(Ctx* c);
/// True the first time (kernel, device) is seen: cudaFuncSetAttribute is a
/// per-device setting.
bool func_attr_once(const void* fn, int device);
void count_launch(const char* family);
void add_alg_bytes(const char* family, double bytes);
void check_cuda(cudaError_t e, const char* what);
#define IQCC_CUDA(x) ::iqcc_b200::check_cuda((x), #x)

/// Kernel-family timing scope (CUDA events on the engine stream) when
/// profiling is enabled; always counts the launch.
/// cudaStreamSynchronize that books the host's blocked time under the
/// profile family "host_wait" (launch-bound vs GPU-bound diagnosis).
void host_sync(cudaStream_t st);
/// Page-locked host scratch (>= 8 KiB) for small device->host reads, so the
/// copies stay asynchronous; valid until the next call.
void* host_pinned(size_t bytes);
/// Small device->host read (<= 64 KiB) that does not go through a copy
/// engine: a one-block kernel stores the bytes into the context's mapped
/// page-locked buffer, and the next host_sync() copies them to dst.  Copy
/// engines run their queues in order, so a 4-byte cudaMemcpy D2H of one
/// context waits behind another context's multi-GB download; SM stores
/// over PCIe do not.  Larger reads fall back to cudaMemcpyAsync.  dst must
/// stay valid until that host_sync().
void d2h_small(void* dst, const void* src, size_t bytes, cudaStream_t st);
/// A second, large page-locked buffer of the context (grows, reused): the
/// staging of the host-side coefficient reformatting in upload/download.
void* host_staging(size_t bytes);

/// Host wall time of a region, booked under a profile family (profiling on).
struct HostScope {
  const char* family;
  double t0;
  explicit HostScope(const char* f);
  ~HostScope();
};

struct KernelScope {
  const char* family;
  cudaEvent_t a = nullptr, b = nullptr;
  explicit KernelScope(const char* f);
  ~KernelScope();
};

/// Grow-only device scratch buffer.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  bool big = false;  // cudaMalloc (large) vs stream-ordered pool (small)
  void* get(size_t n);
  template <class T>
  T* as(size_t count) { return static_cast<T*>(get(count * sizeof(T))); }
  void release();
};

struct Workspace {
  DevBuf lcp, mbits, fmask, tile_cnt, tile_pfx, fwd_agg, bwd_agg, fwd_carry, bwd_carry;
  DevBuf inv_perm, rdelta, part_a, part_b, tile_status, counters, hist, cand_v, cand_i, cand_v2, cand_i2, qflag, qbits;
  DevBuf levels, stage_rows, stage_coef, partials, grad_part, tables, misc, misc2, misc3;
  DevBuf xbuf_keys, xbuf_coef, rbuf_keys, rbuf_coef;
  DevBuf out_keys, out_coef;  // double buffer swapped with the store after a step
  DevBuf dbg;                 // 4 x u64 bounds-check record
  void release_all();
};
Workspace& workspace();
ull* debug_buffer();          // device dbg record (zeroed at init)
void debug_check(const char* where);  // throws if a bounds check fired

struct DeviceStore {
  uint32_t n_qubits = 0, B = 1;
  size_t M = 0;        // physical terms
  DevBuf kbuf, cbuf;   // key rows [cap][2B], coef [cap]
  Filter filt;         // lazy compress filter (see filter_keep)
  size_t logical = 0;  // terms that pass filt
  bool has_identity = false;
  // Next-step metadata written by the previous merge of a dress_sequence:
  // LCP of every slot with its predecessor and the anticommute bits against
  // the next entangler meta_P (device key words); replaces that step's
  // classify pass.  Any other change of the slots clears meta_valid.
  bool meta_valid = false;
  ull meta_P[8] = {};
  double spec_cut = 0.0;  // last compress cut: dress_sequence's slot speculation guess
  DevBuf meta_lcp, meta_amask;
  ull* keys() const { return static_cast<ull*>(kbuf.p); }
  double* coef() const { return static_cast<double*>(cbuf.p); }
  void ensure(size_t n);  // capacity >= n terms, contents NOT kept
  void free_all() {
    kbuf.release();
    cbuf.release();
    meta_lcp.release();
    meta_amask.release();
    meta_valid = false;
  }
};

struct CompressResult {
  size_t dropped_terms = 0;
  double dropped_weight = 0.0;
};

// implemented in the .cu files
void store_upload(DeviceStore& s, size_t n_qubits, const uint64_t* rows, const double* coeff,
                  size_t M, bool host_src);
size_t store_download(DeviceStore& s, uint64_t* rows, double* coeff, size_t cap, bool host_dst);
void store_generate_mol(DeviceStore& s, size_t n_qubits, size_t n_terms, uint64_t seed);
void store_materialize(DeviceStore& s);
void store_clone(const DeviceStore& src, DeviceStore& dst);
/// Pauli text I/O and the FCIDUMP -> JW ingest (io.cu, iqcc/io.hpp).
void store_read_pauli_file(DeviceStore& s, const std::string& path);
void store_write_pauli_file(DeviceStore& s, const std::string& path);
size_t store_jordan_wigner_fcidump(DeviceStore& s, const std::string& path);

struct DressOutcome {
  size_t n_anticommuting = 0;
  size_t count_eps = 0;  // emitted terms passing (identity || |c| >= eps)
  size_t n_ge_theta = 0;  // emitted non-identity terms with |c| >= theta (theta > 0 only)
  size_t n_pairs = 0;     // survivor/product partner pairs (same word)
  // partitioned steps (merge_reducer set): {count_eps, n_ge_theta, identity}
  // summed over the ranks, fetched with the merge counters (one round trip)
  bool has_glob = false;
  unsigned long long glob[3] = {0, 0, 0};
};
struct Reducer;
/// While set, every merge also allreduces its (count_eps, n_ge_theta,
/// identity) on the device before the counter read-back.
void set_merge_reducer(Reducer* red);
/// One dressing step in place; if want_hist, also accumulates the |c|
/// histogram of emitted terms for a following compress(eps).
/// next_row (optional, device-width row): the entangler of the following
/// step; the merge then also writes that step's classify metadata.
/// theta > 0: a compress whose cut is >= theta follows (theta <= eps: known;
/// a power of two above eps: speculated, the caller verifies n_ge_theta);
/// terms below theta/2 get no output slot (SlotRule in dress.cu).
/// anti_only: keep only the anticommuting part (commuting terms and the
/// identity are dropped): with (cos, sin) = (-sin tau, cos tau) this is
/// dress_derivative (iqcc/optimizer.hpp:31-48).
DressOutcome dress_step(DeviceStore& s, const uint64_t* gen_row, double cos_tau, double sin_tau,
                        double drop_thr, bool want_hist, double eps,
                        const uint64_t* next_row = nullptr, double theta = 0.0,
                        bool anti_only = false);
/// Undo the last dress_step (the merge's input buffers are still the
/// workspace's output pair): restores the store as it was before the step.
void dress_undo(DeviceStore& s, size_t M, size_t logical, const Filter& filt);
/// Phases of a step for the partitioned path: plan (classify, present
/// prefix, product order; returns the product count A), materialize the
/// sorted products (keys ^ P, values) into a buffer, and merge the store's
/// survivors with products given as a buffer (q_keys != nullptr) or the
/// planned local products.
size_t plan_products(DeviceStore& s, const uint64_t* gen_row, bool products);
/// plan_products without reading the count back: returns its device
/// address (nullptr: empty store); the caller then sets it with
/// plan_set_products before materialize/merge.
/// (survivor slots by SlotRule theta; products always planned in full)
const long long* plan_products_async(DeviceStore& s, const uint64_t* gen_row, double cs = 1.0,
                                     double sn = 0.0, double theta = 0.0);
/// Survivor classification and slot bits only (redo of a failed speculation
/// in the partitioned step: the received products are kept).
void plan_survivors(DeviceStore& s, const uint64_t* gen_row, double cs, double sn, double theta);
/// Slot bits of n received products (values rv): |v| >= thq; thq = 0: all.
void recv_slot_bits(const double* rv, size_t n, double thq);
void plan_set_products(size_t A);
/// The planned product order (sorted rank -> store index) of the last plan.
const unsigned* plan_inv_perm();
/// All planned products written straight into a peer's receive buffer
/// (okeys/ovals: CUDA IPC mapping over NVLink), staged per 256-product tile.
/// [r0, r1) only, on stream `on` (nullptr: the engine stream, profiled as
/// "exchange"), with at most max_grid CTAs (0: 8 per SM).
void push_products(DeviceStore& s, const uint64_t* gen_row, double sn, ull* okeys, double* ovals,
                   size_t r0 = 0, size_t r1 = SIZE_MAX, cudaStream_t on = nullptr, unsigned max_grid = 0);
/// Products [r0, r1) of the planned order (clamped to the product count).
/// thq / obits (optional): also pack the receiver's product slot bits
/// (|v| >= thq) into obits (one bit per product, r0 % 32 == 0).
void materialize_products(DeviceStore& s, const uint64_t* gen_row, double sn, ull* okeys,
                          double* ovals, size_t r0 = 0, size_t r1 = SIZE_MAX,
                          const char* family = "materialize", double thq = 0.0,
                          unsigned* obits = nullptr);
/// recv_slot_bits from bits the sender packed (possibly in peer memory).
void recv_slot_bits_packed(const unsigned* bits, size_t n, double thq);
/// Received products merged chunk by chunk as they land (multi.cu's chunked
/// exchange): chunk c merges survivors [a[c], a[c+1]) with products
/// [r[c], r[c+1]); a[C] = store size, r[C] = product count, every r[c]
/// (c < C) a multiple of 32 * 1024 (whole slot-bit scan blocks).  arrive(c,
/// &qtotal, &Wq) enqueues what must precede chunk c (the wait for its data,
/// its product slot bits) and may narrow the slot-bit view to the words
/// ready so far.
struct ChunkPlan {
  int C = 1;
  std::vector<size_t> a, r;
  std::function<void(int, const unsigned**, size_t*)> arrive;
};
/// Slot bits of n received products computed chunk by chunk:
/// recv_slot_bits_begin sizes the arrays; recv_slot_bits_chunk adds
/// products [r0, r1) (r0 a multiple of 32 * 1024, chunks in order) and
/// returns the prefix total and word count through r1.
void recv_slot_bits_begin(size_t n, double thq, int chunks);
void recv_slot_bits_chunk(const double* rv, size_t r0, size_t r1, size_t n, int c,
                          const unsigned** qtotal, size_t* Wq);
DressOutcome merge_products(DeviceStore& s, const uint64_t* gen_row, double cs, double sn,
                            double drop, bool want_hist, double eps, size_t nQ, const ull* q_keys,
                            const double* q_vals, const uint64_t* next_row = nullptr,
                            double theta = 0.0, const ChunkPlan* cp = nullptr);
/// Selects the compress filter on a store without a filter.  If hist_ready,
/// the histogram/count_eps of the last dress_step are used.
/// Cross-rank hooks for compress_partitioned (iqcc/partition.hpp:325-396);
/// nullptr = single device.
struct Reducer {
  virtual ~Reducer() = default;
  virtual void sum(ull* vals, size_t n) = 0;         // in place, host buffers
  virtual void sum_device(ull* dvals, size_t n) = 0;  // in place on the stream
  /// all ranks' tied keys (device rows, 2B words each), concatenated in rank
  /// order; *mine_offset receives where this rank's keys start.
  virtual std::vector<ull> gather_keys(const std::vector<ull>& mine, size_t words_per_key,
                                       size_t* mine_offset) = 0;
  /// Device allgather of n u64 per rank into recv[world][n] on the stream
  /// (false: not offered; the caller falls back).  world/rank: this group.
  virtual bool allgather_device(const ull* /*send*/, ull* /*recv*/, size_t /*n*/) { return false; }
  virtual bool can_allgather() const { return false; }
  virtual int group_size() const { return 1; }
  virtual int group_rank() const { return 0; }
};
/// glob_known (partitioned, optional): {global count_eps, global identity
/// count} already reduced by the caller, saving the first reduction.
/// cand_floor: a verified lower bound of the cut value (a slot speculation
/// that passed: at least `budget` terms are >= theta), so the select only
/// gathers candidates >= it.
CompressResult compress_store(DeviceStore& s, double eps, size_t max_terms, bool hist_ready,
                              size_t count_eps, bool want_stats, Reducer* red = nullptr,
                              const ull* glob_known = nullptr, double cand_floor = 0.0);
void growth_split(DeviceStore& s, const uint64_t* gen_row, size_t* nc, size_t* na);
/// SortlessStats buckets (iqcc/dressing.hpp:159-189): distinct support
/// patterns of the present terms, and how many of them anticommute.
void sortless_stats(DeviceStore& s, const uint64_t* gen_row, size_t* n_buckets, size_t* n_anti_buckets);

double expect_store(DeviceStore& s, const double* factors);
double qmf_grad_store(DeviceStore& s, const double* factors, const double* derivs, double* grad);
void gradients_store(DeviceStore& s, const double* factors, const uint64_t* cands, size_t K,
                     bool flip_group_only, double* g);
size_t dis_store(DeviceStore& s, const double* factors, bool poles, size_t top_k, double thr,
                 size_t cap_per_group, std::vector<uint64_t>& rows_out, std::vector<double>& g_out);
double choose_bits_store(DeviceStore& s, size_t m, size_t* bits_out);
/// build_poly_kernels (iqcc/optimizer.hpp:340-368): words [t][2B] (device B,
/// reference row layout), hk / nk [t][t][2] on the host.  worker_local:
/// the per-worker h_kernel of the partitioned form (diagonal not conjugated).
void poly_kernels_store(DeviceStore& s, const double* factors, bool poles, const uint64_t* words,
                        size_t t, double* hk, double* nk, bool worker_local = false);
void parallel_poly_kernels_store(DeviceStore& s, const double* factors, bool poles, const uint64_t* words,
                                 size_t t, double* hk, double* nk);
void restrict_store(DeviceStore& s, size_t m, const size_t* bits, const size_t* owner, int rank);

/// merge_sums (iqcc/pauli.hpp:383-415) of two stores into `out`.
void merge_sums_store(DeviceStore& a, DeviceStore& b, double drop, DeviceStore& out);

/// Partitioned sums on the device driven from one host thread (psum.cu).
struct PSum;
PSum* psum_distribute(size_t n_qubits, const uint64_t* rows, const double* coeff, size_t M,
                                      size_t m, const size_t* bits, const size_t* owner, size_t n_workers,
                                      const int* devices);
PSum* psum_from_shards(size_t n_qubits, size_t m, const size_t* bits, const size_t* owner,
                                       size_t n_workers, const int* devices, const uint64_t* const* rows,
                                       const double* const* coeffs, const size_t* sizes);
void psum_destroy(PSum* ps);
size_t psum_parts(const PSum& P);
void psum_sizes(PSum& P, size_t* sizes);
void psum_owner(const PSum& P, size_t* owner);
size_t psum_download_shard(PSum& P, size_t p, uint64_t* rows, double* coeff, size_t cap);
size_t psum_gather(PSum& P, uint64_t* rows, double* coeff, size_t cap);
void psum_dress(PSum& P, const uint64_t* gen, double cs, double sn, double eps, size_t max_terms,
                iqcc_message_record* log, size_t log_cap, size_t* n_log, iqcc_compress_stats* cstats,
                size_t* mask_out);
double psum_expect(PSum& P, const double* factors);
double psum_qmf_energy_gradient(PSum& P, const double* factors, const double* derivs, double* grad);
void psum_gradients(PSum& P, const double* factors, const uint64_t* cands, size_t K, bool flip_only, double* g);
void psum_rebalance(PSum& P, double threshold, size_t* owner_out);

/// Partition bits as (device word, bit) pairs (iqcc/partition.hpp:40-42).
struct PartSpecHost {
  int m = 0;
  int word[16] = {};
  int bit[16] = {};
};
PartSpecHost make_part_spec(const DeviceStore& s, size_t m, const size_t* bits);

/// Reversed row conversion helpers (host).
void row_to_device_key(const uint64_t* row, uint32_t B, ull* key);
void device_key_to_row(const ull* key, uint32_t B, uint64_t* row);

}  // namespace iqcc_b200
