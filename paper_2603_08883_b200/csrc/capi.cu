// capi.cu — engine context (device, stream, scratch, profiling) and the
// extern "C" entry points declared in include/iqcc_b200.h.
//
// Every entry point catches C++ exceptions and maps them onto status codes:
// std::invalid_argument -> IQCC_EINVAL (the reference throws
// std::invalid_argument for precondition violations),
// std::runtime_error -> IQCC_ERUNTIME, CUDA failures -> IQCC_ECUDA.
#include <chrono>
#include <tuple>
#include <vector>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <random>
#include <algorithm>
#include <memory>
#include <optional>
#include <atomic>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/iqcc_b200.h"
#include "engine.cuh"
#include "multi.cuh"

namespace iqcc_b200 {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct ProfileEntry {
  double ms = 0.0;
  double alg_bytes = 0.0;  // algorithmic bytes attributed to the family
  uint64_t launches = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
};

// Freed large blocks are cached for reuse (see DevBuf::get); one cache per
// context, since a context's stream orders every use of its blocks.
struct BigCache {
  std::vector<std::pair<void*, size_t>> blocks;
  size_t bytes = 0;
};

// One engine context per host thread (a device, a stream, the hot path's
// scratch and a block cache).  The C-ABI binds the calling thread
// (iqcc_gpu_init); the partitioned-sum driver (psum.cu) runs one worker
// thread per shard, each with its own context on the shard's device, so
// shards on one device never share scratch and shards on different devices
// run concurrently from one API call.
struct Ctx {
  int device = -1;
  cudaStream_t own = nullptr;
  cudaStream_t cur = nullptr;
  Workspace ws;
  bool profiling = false;
  std::map<std::string, ProfileEntry> prof;
  std::vector<cudaEvent_t> event_pool;
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
  void* staging = nullptr;  // large page-locked buffer for host<->device reformatting
  size_t staging_bytes = 0;
  BigCache big;
  // d2h_small: mapped page-locked landing buffer and the reads pending on it
  unsigned char* peek_host = nullptr;
  unsigned char* peek_dev = nullptr;
  size_t peek_used = 0;
  std::vector<std::tuple<void*, size_t, size_t>> peek_pending;  // (dst, offset, bytes)
};

static thread_local Ctx* g_ctx = nullptr;
static Ctx* g_comm_ctx = nullptr;  // the context that initialised the NCCL communicator
static thread_local std::string g_err;
static std::atomic<uint64_t> g_launches{0};  // every engine kernel launch, all contexts

Ctx& ctx() {
  if (!g_ctx) throw std::runtime_error("iqcc_gpu_init has not been called");
  return *g_ctx;
}
cudaStream_t stream() { return ctx().cur; }
Workspace& workspace() { return ctx().ws; }

ull* debug_buffer() {
  Workspace& ws = ctx().ws;
  if (!ws.dbg.p) {
    ws.dbg.get(4 * sizeof(ull));
    IQCC_CUDA(cudaMemsetAsync(ws.dbg.p, 0, 4 * sizeof(ull), stream()));
  }
  return static_cast<ull*>(ws.dbg.p);
}

void debug_check(const char* where) {
  ull h[3];
  IQCC_CUDA(cudaMemcpyAsync(h, debug_buffer(), sizeof(h), cudaMemcpyDeviceToHost, stream()));
  IQCC_CUDA(cudaStreamSynchronize(stream()));
  if (h[0])
    throw std::runtime_error(std::string("bounds check failed after ") + where + ": site " +
                             std::to_string(h[0]) + " index " + std::to_string(h[1]) + " bound " +
                             std::to_string(h[2]));
}

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw CudaError(std::string("CUDA error ") + cudaGetErrorString(e) + " at " + what);
}

void count_launch(const char* family) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  (void)family;
}

// algorithmic bytes are booked whether or not event profiling is on (a host
// add per step), so a timed pass reports its own roofline numerator
void add_alg_bytes(const char* family, double bytes) { ctx().prof[family].alg_bytes += bytes; }

static cudaEvent_t take_event() {
  Ctx& c = ctx();
  if (!c.event_pool.empty()) {
    cudaEvent_t e = c.event_pool.back();
    c.event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  IQCC_CUDA(cudaEventCreate(&e));
  return e;
}

// NVTX ranges (IQCC_NVTX=1): one range per kernel family launch and per
// host scope, named by family, for nsys / ncu --nvtx timelines.
static bool nvtx_on() {
  static const bool on = getenv("IQCC_NVTX") && atoi(getenv("IQCC_NVTX")) != 0;
  return on;
}

KernelScope::KernelScope(const char* f) : family(f) {
  Ctx& c = ctx();
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (nvtx_on()) nvtxRangePushA(f);
  if (c.profiling) {
    a = take_event();
    b = take_event();
    IQCC_CUDA(cudaEventRecord(a, c.cur));
  }
}

KernelScope::~KernelScope() {
  Ctx& c = ctx();
  if (nvtx_on()) nvtxRangePop();
  cudaError_t le = cudaPeekAtLastError();
  if (a) {
    cudaEventRecord(b, c.cur);
    auto& e = c.prof[family];
    e.launches += 1;
    e.pending.push_back({a, b});
  }
  if (le != cudaSuccess) {
    // surfaced by the next IQCC_CUDA check; keep the error sticky for the caller
    g_err = std::string("kernel launch failed (") + family + "): " + cudaGetErrorString(le);
  }
  static const bool dbg = getenv("IQCC_DEBUG") != nullptr;
  if (dbg) {
    cudaError_t e = cudaStreamSynchronize(c.cur);
    if (e != cudaSuccess) fprintf(stderr, "[iqcc debug] kernel family '%s' failed: %s\n", family, cudaGetErrorString(e));
  }
}

void* host_pinned(size_t bytes) {
  Ctx& c = ctx();
  if (bytes > c.pinned_bytes) {
    if (c.pinned) IQCC_CUDA(cudaFreeHost(c.pinned));
    c.pinned = nullptr;
    c.pinned_bytes = std::max<size_t>(bytes, 8192);
    IQCC_CUDA(cudaMallocHost(&c.pinned, c.pinned_bytes));
  }
  return c.pinned;
}

void* host_staging(size_t bytes) {
  Ctx& c = ctx();
  if (bytes > c.staging_bytes) {
    if (c.staging) IQCC_CUDA(cudaFreeHost(c.staging));
    c.staging = nullptr;
    c.staging_bytes = std::max<size_t>(bytes + bytes / 4, 1 << 20);
    IQCC_CUDA(cudaMallocHost(&c.staging, c.staging_bytes));
  }
  return c.staging;
}

constexpr size_t kPeekCap = (size_t)64 << 10;

__global__ void k_peek(const unsigned char* __restrict__ src, unsigned char* __restrict__ dst, size_t n) {
  for (size_t i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

void d2h_small(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return;
  Ctx& c = ctx();
  const size_t off = (c.peek_used + 15) & ~(size_t)15;
  if (bytes > kPeekCap || off + bytes > kPeekCap) {
    IQCC_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
    return;
  }
  if (!c.peek_host) {
    IQCC_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&c.peek_host), kPeekCap, cudaHostAllocMapped));
    IQCC_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c.peek_dev), c.peek_host, 0));
  }
  count_launch("peek");
  k_peek<<<1, 256, 0, st>>>(static_cast<const unsigned char*>(src), c.peek_dev + off, bytes);
  IQCC_CUDA(cudaGetLastError());
  c.peek_pending.emplace_back(dst, off, bytes);
  c.peek_used = off + bytes;
}

static void peek_flush(Ctx& c) {
  for (auto& [dst, off, n] : c.peek_pending) std::memcpy(dst, c.peek_host + off, n);
  c.peek_pending.clear();
  c.peek_used = 0;
}

// Busy-wait: a blocking/yielding synchronize can leave the GPU idle for a
// scheduler quantum after every step boundary.
static void spin_sync(cudaStream_t st) {
  for (;;) {
    const cudaError_t e = cudaStreamQuery(st);
    if (e == cudaSuccess) return;
    if (e != cudaErrorNotReady) IQCC_CUDA(e);
  }
}

void host_sync(cudaStream_t st) {
  Ctx& c = ctx();
  if (!c.profiling) {
    spin_sync(st);
    peek_flush(c);
    return;
  }
  const auto t0 = std::chrono::steady_clock::now();
  spin_sync(st);
  peek_flush(c);
  const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  auto& e = c.prof["host_wait"];
  e.ms += ms;
  e.launches += 1;
}

static void host_ms(const char* fam, std::chrono::steady_clock::time_point t0) {
  Ctx& c = ctx();
  if (!c.profiling) return;
  auto& e = c.prof[fam];
  e.ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  e.launches += 1;
}

static double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
HostScope::HostScope(const char* f) : family(f), t0(now_ms()) {
  if (nvtx_on()) nvtxRangePushA(f);
}
HostScope::~HostScope() {
  if (nvtx_on()) nvtxRangePop();
  Ctx& c = ctx();
  if (!c.profiling) return;
  auto& e = c.prof[family];
  e.ms += now_ms() - t0;
  e.launches += 1;
}

static void profile_flush() {
  Ctx& c = ctx();
  for (auto& [name, e] : c.prof) {
    for (auto& pr : e.pending) {
      IQCC_CUDA(cudaEventSynchronize(pr.second));
      float ms = 0.f;
      IQCC_CUDA(cudaEventElapsedTime(&ms, pr.first, pr.second));
      e.ms += ms;
      c.event_pool.push_back(pr.first);
      c.event_pool.push_back(pr.second);
    }
    e.pending.clear();
  }
}

// Large buffers (stores, merge outputs, scratch of the hot path) come from
// cudaMalloc: on B200 mapping fresh memory through the stream-ordered pool
// costs ~15-50 ms per call (measured: 16 GB cudaMallocAsync 51 ms vs
// cudaMalloc 1.8 ms), which dominated uncapped growth (C5).  cudaFree
// synchronizes the device, so a large buffer is never freed under a running
// kernel.  Small buffers stay stream-ordered.
constexpr size_t kBigAlloc = (size_t)32 << 20;

// Freed large blocks are cached for reuse (a context runs on one stream, so
// a block handed out again is only touched by later work in stream order).
// A cached block serves a request between a quarter of its size and its
// size (best fit) when it wastes at most kBigSlack bytes, and between half
// and all of its size otherwise: chains of stores growing ~1.5x per step
// find their blocks again on the next chain, while a huge block is not
// pinned under a small live buffer.
constexpr size_t kBigSlack = (size_t)256 << 20;

static void big_release_all(BigCache& bc) {
  if (bc.blocks.empty()) return;
  cudaDeviceSynchronize();
  for (auto& b : bc.blocks) cudaFree(b.first);
  bc.blocks.clear();
  bc.bytes = 0;
}

static void* big_take(size_t want, size_t* got) {
  BigCache& bc = ctx().big;
  size_t best = SIZE_MAX;
  for (size_t i = 0; i < bc.blocks.size(); ++i) {
    const size_t b = bc.blocks[i].second;
    const bool fits = b >= want && (b - want <= kBigSlack ? b / 4 <= want : b / 2 <= want);
    if (fits && (best == SIZE_MAX || b < bc.blocks[best].second)) best = i;
  }
  if (best == SIZE_MAX) return nullptr;
  void* p = bc.blocks[best].first;
  *got = bc.blocks[best].second;
  bc.bytes -= *got;
  bc.blocks.erase(bc.blocks.begin() + best);
  return p;
}

static void devbuf_free(void* p, bool big, size_t bytes) {
  if (!p) return;
  if (big) {
    BigCache& bc = ctx().big;
    bc.blocks.emplace_back(p, bytes);
    bc.bytes += bytes;
    // bound the cache at 64 blocks: the oldest freed block leaves first
    while (bc.blocks.size() > 64) {
      IQCC_CUDA(cudaFree(bc.blocks.front().first));
      bc.bytes -= bc.blocks.front().second;
      bc.blocks.erase(bc.blocks.begin());
    }
  } else {
    IQCC_CUDA(cudaFreeAsync(p, stream()));
  }
}

void* DevBuf::get(size_t n) {
  if (n <= bytes && p) return p;
  HostScope hs("host_alloc");
  cudaStream_t st = stream();
  static const bool verbose = getenv("IQCC_VERBOSE") != nullptr;
  if (verbose) {
    const Workspace& w = ctx().ws;
    fprintf(stderr, "[alloc] buf@ws+%td n=%zu had=%zu\n",
            (const char*)this - (const char*)&w, n, bytes);
  }
  devbuf_free(p, big, bytes);
  p = nullptr;
  bytes = 0;
  size_t want = std::max<size_t>(n + n / 2, 256);  // generous slack: stores grow ~1.5x per step
  big = want >= kBigAlloc;
  if (big) {
    size_t got = 0;
    if ((p = big_take(n, &got)) != nullptr) {
      bytes = got;
      return p;
    }
  }
  cudaError_t e = big ? cudaMalloc(&p, want) : cudaMallocAsync(&p, want, st);
  if (e != cudaSuccess) {
    // retry without slack once the caches have released their blocks
    cudaGetLastError();
    if (verbose) fprintf(stderr, "[alloc] %zu bytes failed: release the caches and retry\n", want);
    IQCC_CUDA(cudaStreamSynchronize(st));
    big_release_all(ctx().big);
    cudaMemPool_t pool;
    IQCC_CUDA(cudaDeviceGetDefaultMemPool(&pool, ctx().device));
    cudaMemPoolTrimTo(pool, 0);
    want = std::max<size_t>(n, 256);
    big = want >= kBigAlloc;
    e = big ? cudaMalloc(&p, want) : cudaMallocAsync(&p, want, st);
    if (e != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      bytes = 0;
      throw std::bad_alloc();
    }
  }
  bytes = want;
  return p;
}

void DevBuf::release() {
  if (p && g_ctx) {
    if (big)
      devbuf_free(p, true, bytes);
    else
      cudaFreeAsync(p, g_ctx->cur);
  }
  p = nullptr;
  bytes = 0;
  big = false;
}

Ctx* ctx_new(int device) {
  IQCC_CUDA(cudaSetDevice(device));
  auto* c = new Ctx();
  c->device = device;
  IQCC_CUDA(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking));
  c->cur = c->own;
  cudaMemPool_t pool;
  IQCC_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t thr = UINT64_MAX;
  IQCC_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  return c;
}

Ctx* ctx_bind(Ctx* c) {
  Ctx* prev = g_ctx;
  g_ctx = c;
  if (c) IQCC_CUDA(cudaSetDevice(c->device));
  return prev;
}

Ctx* ctx_current() { return g_ctx; }

int ctx_device(const Ctx* c) { return c ? c->device : -1; }

void ctx_free(Ctx* c) {
  if (!c) return;
  Ctx* prev = ctx_bind(c);
  cudaStreamSynchronize(c->cur);
  c->ws.release_all();
  cudaStreamSynchronize(c->cur);
  big_release_all(c->big);
  for (cudaEvent_t e : c->event_pool) cudaEventDestroy(e);
  if (c->pinned) cudaFreeHost(c->pinned);
  if (c->staging) cudaFreeHost(c->staging);
  if (c->peek_host) cudaFreeHost(c->peek_host);
  cudaStreamDestroy(c->own);
  delete c;
  ctx_bind(prev == c ? nullptr : prev);
}

bool func_attr_once(const void* fn, int device) {
  // cudaFuncSetAttribute applies per device: remember (kernel, device)
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> done;
  std::lock_guard<std::mutex> lk(mu);
  for (auto& d : done)
    if (d.first == fn && d.second == device) return false;
  done.emplace_back(fn, device);
  return true;
}

void Workspace::release_all() {
  DevBuf* all[] = {&lcp, &mbits, &fmask, &tile_cnt, &tile_pfx, &fwd_agg, &bwd_agg, &fwd_carry,
                   &bwd_carry, &inv_perm, &rdelta, &part_a, &part_b, &tile_status, &counters,
                   &hist, &cand_v, &cand_i, &levels, &stage_rows, &stage_coef, &partials,
                   &grad_part, &tables, &misc, &misc2, &misc3, &xbuf_keys, &xbuf_coef,
                   &rbuf_keys, &rbuf_coef, &out_keys, &out_coef, &dbg};
  for (DevBuf* b : all) b->release();
}

}  // namespace iqcc_b200

using namespace iqcc_b200;

struct iqcc_gpu_sum {
  DeviceStore s;
};

namespace {

int fail(int code, const std::string& msg) {
  g_err = msg;
  if (g_ctx) {  // reads queued by the failed call must not land later
    g_ctx->peek_pending.clear();
    g_ctx->peek_used = 0;
  }
  return code;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return IQCC_OK;
  } catch (const std::invalid_argument& e) {
    return fail(IQCC_EINVAL, e.what());
  } catch (const CudaError& e) {
    return fail(IQCC_ECUDA, e.what());
  } catch (const std::bad_alloc&) {
    return fail(IQCC_ENOMEM, "device out of memory");
  } catch (const std::exception& e) {
    return fail(IQCC_ERUNTIME, e.what());
  }
}

uint32_t ref_blocks(const DeviceStore& s) { return s.n_qubits == 0 ? 1 : (s.n_qubits + 63) / 64; }

/// Reference-layout row (B_ref blocks per plane) -> device-width row.
std::vector<uint64_t> widen_row(const uint64_t* row, uint32_t Bref, uint32_t B) {
  std::vector<uint64_t> r(2 * B, 0);
  for (uint32_t w = 0; w < Bref; ++w) {
    r[w] = row[w];
    r[B + w] = row[Bref + w];
  }
  return r;
}

bool row_is_identity(const uint64_t* row, uint32_t Bref) {
  for (uint32_t w = 0; w < 2 * Bref; ++w)
    if (row[w]) return false;
  return true;
}

void need(const iqcc_gpu_sum* h) {
  if (!h) throw std::invalid_argument("null sum handle");
}

}  // namespace

#pragma GCC visibility push(default)
extern "C" {

const char* iqcc_gpu_last_error(void) { return g_err.c_str(); }

int iqcc_gpu_init(int device) {
  return guarded([&] {
    if (g_ctx && g_ctx->device == device) return;
    if (g_ctx) throw std::invalid_argument("engine already initialised on another device");
    g_ctx = ctx_new(device);
  });
}

int iqcc_gpu_set_stream(void* s) {
  return guarded([&] {
    Ctx& c = ctx();
    IQCC_CUDA(cudaStreamSynchronize(c.cur));
    c.cur = s ? static_cast<cudaStream_t>(s) : c.own;
  });
}

int iqcc_gpu_finalize(void) {
  return guarded([&] {
    if (!g_ctx) return;
    cudaStreamSynchronize(g_ctx->cur);
    // the process-wide communicator goes with the context that created it
    // (a worker thread's context finalizing leaves it alone)
    if (g_comm_ctx == g_ctx) {
      multi_shutdown();
      g_comm_ctx = nullptr;
    }
    ctx_free(g_ctx);
    g_ctx = nullptr;
  });
}

uint64_t iqcc_gpu_launch_count(void) { return g_launches.load(); }

int iqcc_gpu_profile_enable(int on) {
  return guarded([&] { ctx().profiling = on != 0; });
}

int iqcc_gpu_profile_get(const char* name, double* total_ms, uint64_t* launches) {
  return guarded([&] {
    profile_flush();
    auto& p = ctx().prof;
    auto it = p.find(name);
    *total_ms = it == p.end() ? 0.0 : it->second.ms;
    *launches = it == p.end() ? 0 : it->second.launches;
  });
}

int iqcc_gpu_profile_bytes(const char* name, double* bytes) {
  return guarded([&] {
    auto& p = ctx().prof;
    auto it = p.find(name);
    *bytes = it == p.end() ? 0.0 : it->second.alg_bytes;
  });
}

int iqcc_gpu_profile_reset(void) {
  return guarded([&] {
    profile_flush();
    ctx().prof.clear();
  });
}

int iqcc_gpu_sum_create(size_t n_qubits, const uint64_t* rows, const double* coeff, size_t M,
                        iqcc_gpu_sum** out) {
  return guarded([&] {
    ctx();
    auto h = std::make_unique<iqcc_gpu_sum>();
    store_upload(h->s, n_qubits, rows, coeff, M, true);
    *out = h.release();
  });
}

int iqcc_gpu_sum_create_device(size_t n_qubits, const uint64_t* rows, const double* coeff, size_t M,
                               iqcc_gpu_sum** out) {
  return guarded([&] {
    ctx();
    auto h = std::make_unique<iqcc_gpu_sum>();
    store_upload(h->s, n_qubits, rows, coeff, M, false);
    *out = h.release();
  });
}

int iqcc_gpu_sum_generate_mol(size_t n_qubits, size_t n_terms, uint64_t seed, iqcc_gpu_sum** out) {
  return guarded([&] {
    ctx();
    auto h = std::make_unique<iqcc_gpu_sum>();
    store_generate_mol(h->s, n_qubits, n_terms, seed);
    *out = h.release();
  });
}

int iqcc_gpu_read_pauli_file(const char* path, iqcc_gpu_sum** out) {
  return guarded([&] {
    ctx();
    if (!path || !out) throw std::invalid_argument("read_pauli_file: null argument");
    auto h = std::make_unique<iqcc_gpu_sum>();
    store_read_pauli_file(h->s, path);
    *out = h.release();
  });
}

int iqcc_gpu_write_pauli_file(iqcc_gpu_sum* h, const char* path) {
  return guarded([&] {
    need(h);
    if (!path) throw std::invalid_argument("write_pauli_file: null path");
    store_write_pauli_file(h->s, path);
  });
}

int iqcc_gpu_jordan_wigner_fcidump(const char* path, size_t* n_electrons, iqcc_gpu_sum** out) {
  return guarded([&] {
    ctx();
    if (!path || !out) throw std::invalid_argument("jordan_wigner_fcidump: null argument");
    auto h = std::make_unique<iqcc_gpu_sum>();
    const size_t ne = store_jordan_wigner_fcidump(h->s, path);
    if (n_electrons) *n_electrons = ne;
    *out = h.release();
  });
}

int iqcc_gpu_sum_clone(const iqcc_gpu_sum* h, iqcc_gpu_sum** out) {
  return guarded([&] {
    need(h);
    auto c = std::make_unique<iqcc_gpu_sum>();
    store_clone(h->s, c->s);
    *out = c.release();
  });
}

int iqcc_gpu_sum_destroy(iqcc_gpu_sum* h) {
  return guarded([&] {
    if (!h) return;
    if (g_ctx) h->s.free_all();
    delete h;
  });
}

int iqcc_gpu_sum_qubits(const iqcc_gpu_sum* h, size_t* n) {
  return guarded([&] {
    need(h);
    *n = h->s.n_qubits;
  });
}

int iqcc_gpu_sum_size(iqcc_gpu_sum* h, size_t* M) {
  return guarded([&] {
    need(h);
    *M = h->s.logical;
  });
}

int iqcc_gpu_sum_download(iqcc_gpu_sum* h, uint64_t* rows, double* coeff, size_t cap, size_t* M) {
  return guarded([&] {
    need(h);
    *M = store_download(h->s, rows, coeff, cap, true);
  });
}

int iqcc_gpu_sum_download_device(iqcc_gpu_sum* h, uint64_t* rows, double* coeff, size_t cap,
                                 size_t* M) {
  return guarded([&] {
    need(h);
    *M = store_download(h->s, rows, coeff, cap, false);
  });
}

/* Debug/inspection: the physical device store (bit-reversed key rows, raw
 * coefficients including dead-slot NaNs), no filtering. */
int iqcc_gpu_sum_raw(iqcc_gpu_sum* h, uint64_t* keys, double* coef, size_t cap, size_t* M) {
  return guarded([&] {
    need(h);
    *M = h->s.M;
    const size_t n = std::min(cap, h->s.M);
    if (n) {
      IQCC_CUDA(cudaMemcpyAsync(keys, h->s.keys(), n * 2 * h->s.B * sizeof(ull), cudaMemcpyDeviceToHost, stream()));
      IQCC_CUDA(cudaMemcpyAsync(coef, h->s.coef(), n * sizeof(double), cudaMemcpyDeviceToHost, stream()));
    }
    IQCC_CUDA(cudaStreamSynchronize(stream()));
  });
}

int iqcc_gpu_dress(iqcc_gpu_sum* h, const uint64_t* gen, double cos_tau, double sin_tau,
                   double drop_thr, iqcc_dress_stats* stats) {
  return guarded([&] {
    need(h);
    const uint32_t Bref = ref_blocks(h->s);
    if (row_is_identity(gen, Bref)) throw std::invalid_argument("dress_single: identity generator");
    auto row = widen_row(gen, Bref, h->s.B);
    const size_t n_in = h->s.logical;
    DressOutcome o = dress_step(h->s, row.data(), cos_tau, sin_tau, drop_thr, false, 0.0);
    if (stats) {
      stats->n_in = n_in;
      stats->n_anticommuting = o.n_anticommuting;
      stats->n_out = h->s.logical;
    }
  });
}

int iqcc_gpu_compress(iqcc_gpu_sum* h, double eps, size_t max_terms, iqcc_compress_stats* stats) {
  return guarded([&] {
    need(h);
    CompressResult r = compress_store(h->s, eps, max_terms, false, 0, stats != nullptr);
    if (stats) {
      stats->dropped_terms += r.dropped_terms;
      stats->dropped_weight += r.dropped_weight;
    }
  });
}

int iqcc_gpu_dress_sequence(iqcc_gpu_sum* h, size_t K, const uint64_t* gens, const double* cos_tau,
                            const double* sin_tau, double eps, size_t max_terms, double drop_thr,
                            iqcc_compress_stats* stats, size_t* terms_in_total) {
  return guarded([&] {
    need(h);
    if (max_terms < 1) throw std::invalid_argument("dress_sequence: max_terms < 1");
    if (!(drop_thr >= 0.0)) throw std::invalid_argument("dress_sequence: drop_threshold < 0");
    const uint32_t Bref = ref_blocks(h->s);
    for (size_t k = 0; k < K; ++k)
      if (row_is_identity(gens + k * 2 * Bref, Bref))
        throw std::invalid_argument("dress_single: identity generator");
    if (terms_in_total) *terms_in_total = 0;
    const bool fuse = getenv("IQCC_NO_META") == nullptr;  // A/B switch for the fused classify
    // Output slots only for terms the following compress can keep (SlotRule,
    // dress.cu): theta = eps is exact; theta = a power of two at least one
    // binade under the previous cut is speculated and verified after the
    // merge (more than max_terms terms at or above it), else the step is
    // undone and redone with theta = eps.  Off when drop statistics are
    // requested (they count every dropped term).
    const bool slots = stats == nullptr && getenv("IQCC_NO_SPEC") == nullptr;
    auto spec_theta = [&](const Filter& f) {
      if (!slots || !f.active || !f.has_v || !(f.v > 0.0) || !std::isfinite(f.v)) return 0.0;
      return f.v;  // scaled by the next step's |cos| below
    };
    const char* sc_env = getenv("IQCC_SPEC_SCALE");  // test hook: force bad guesses
    const double spec_scale = sc_env ? std::atof(sc_env) : 1.0;
    double spec = slots ? h->s.spec_cut : 0.0;
    for (size_t k = 0; k < K; ++k) {
      auto row = widen_row(gens + k * 2 * Bref, Bref, h->s.B);
      std::vector<uint64_t> next;
      if (fuse && k + 1 < K) next = widen_row(gens + (k + 1) * 2 * Bref, Bref, h->s.B);
      if (terms_in_total) *terms_in_total += h->s.logical;
      const bool maybe = eps > 0.0 || max_terms != SIZE_MAX;
      const auto t0 = std::chrono::steady_clock::now();
      std::optional<KernelScope> outer(std::in_place, "span_dress");
      const double exact = slots && eps > 0.0 ? eps : 0.0;
      // the previous cut, shrunk by what an anticommuting survivor loses (|cos|)
      const double guess = spec * std::min(1.0, std::fabs(cos_tau[k])) * 0.999 * spec_scale;
      const double theta = maybe && guess > eps && max_terms != SIZE_MAX ? guess : exact;
      const size_t M0 = h->s.M, L0 = h->s.logical;
      const Filter F0 = h->s.filt;
      DressOutcome o = dress_step(h->s, row.data(), cos_tau[k], sin_tau[k], drop_thr, maybe, eps,
                                  next.empty() ? nullptr : next.data(), theta);
      if (getenv("IQCC_VERBOSE"))
        fprintf(stderr, "[dress] k=%zu theta=%.3e exact=%.3e n_ge=%zu slots=%zu products=%zu pairs=%zu\n", k,
                theta, exact, o.n_ge_theta, h->s.M, o.n_anticommuting, o.n_pairs);
      // the slotted sum compresses like the full one iff the top `budget`
      // terms are all >= theta and either the compress cuts or nothing below
      // theta holds a slot
      const size_t idc = h->s.has_identity ? 1 : 0;
      const size_t budget = max_terms - idc;
      const bool spec_ok = o.n_ge_theta >= budget &&
                           (o.count_eps > max_terms || o.count_eps == o.n_ge_theta + idc);
      double floor_cut = theta > exact && spec_ok ? theta : 0.0;  // verified: cut >= theta
      if (theta > exact && !spec_ok) {  // speculation failed: redo exactly
        dress_undo(h->s, M0, L0, F0);
        host_ms("spec_redo", std::chrono::steady_clock::now());
        o = dress_step(h->s, row.data(), cos_tau[k], sin_tau[k], drop_thr, maybe, eps,
                       next.empty() ? nullptr : next.data(), exact);
        spec = 0.0;  // relearn from the next cut
        h->s.spec_cut = 0.0;
      }
      outer.reset();
      host_ms("host_dress", t0);
      if (eps > 0.0 || h->s.logical > max_terms) {
        const auto t1 = std::chrono::steady_clock::now();
        CompressResult r;
        {
          KernelScope outer2("span_compress");
          r = compress_store(h->s, eps, max_terms, maybe, o.count_eps, stats != nullptr, nullptr, nullptr,
                             floor_cut);
        }
        // a compress that cut sets the next guess; one that did not (every
        // slotted term kept) hands on the verified floor theta
        const double sv = spec_theta(h->s.filt);
        if (sv > 0.0) {
          spec = h->s.spec_cut = sv;
        } else if (floor_cut > 0.0) {
          // no cut: every live term holds a slot, so |c| >= theta is the
          // store's verified floor (it decays by |cos| per uncut step; the
          // last cut would overestimate it and fail the next guess)
          spec = h->s.spec_cut = floor_cut;
        }
        host_ms("host_compress", t1);
        if (stats) {
          stats->dropped_terms += r.dropped_terms;
          stats->dropped_weight += r.dropped_weight;
        }
      }
    }
  });
}

int iqcc_gpu_sortless_stats(iqcc_gpu_sum* h, const uint64_t* gen, double sin_tau, size_t* n_buckets,
                            size_t* new_term_streams) {
  return guarded([&] {
    need(h);
    auto row = widen_row(gen, ref_blocks(h->s), h->s.B);
    size_t nb = 0, na = 0;
    sortless_stats(h->s, row.data(), &nb, &na);
    if (n_buckets) *n_buckets = nb;
    if (new_term_streams) *new_term_streams = sin_tau != 0.0 ? na : 0;
  });
}

int iqcc_gpu_growth_split(iqcc_gpu_sum* h, const uint64_t* gen, size_t* nc, size_t* na) {
  return guarded([&] {
    need(h);
    auto row = widen_row(gen, ref_blocks(h->s), h->s.B);
    growth_split(h->s, row.data(), nc, na);
  });
}

// qcc_energy / qcc_gradient (iqcc/optimizer.hpp:19-77): device-resident
// dressing chains on working copies of the store; merges drop exact zeros
// only (MergeOptions{0.0, ...}) and nothing is compressed.
namespace {
struct ScratchStore {
  DeviceStore s;
  ~ScratchStore() { s.free_all(); }
};
void check_gens(const uint64_t* gens, size_t K, uint32_t Bref) {
  for (size_t k = 0; k < K; ++k)
    if (row_is_identity(gens + k * 2 * Bref, Bref))
      throw std::invalid_argument("dress_single: identity generator");
}
}  // namespace

int iqcc_gpu_qcc_energy(iqcc_gpu_sum* h, size_t K, const uint64_t* gens, const double* cos_tau,
                        const double* sin_tau, const double* factors, double* energy) {
  return guarded([&] {
    need(h);
    const uint32_t Bref = ref_blocks(h->s);
    check_gens(gens, K, Bref);
    ScratchStore d;
    store_clone(h->s, d.s);
    for (size_t k = 0; k < K; ++k) {
      const auto row = widen_row(gens + k * 2 * Bref, Bref, d.s.B);
      dress_step(d.s, row.data(), cos_tau[k], sin_tau[k], 0.0, false, 0.0);
    }
    *energy = expect_store(d.s, factors);
  });
}

int iqcc_gpu_qcc_gradient(iqcc_gpu_sum* h, size_t K, const uint64_t* gens, const double* cos_tau,
                          const double* sin_tau, const double* factors, double* grad) {
  return guarded([&] {
    need(h);
    const uint32_t Bref = ref_blocks(h->s);
    check_gens(gens, K, Bref);
    ScratchStore a;  // forward chain A_k = h dressed through entanglers [0, k)
    store_clone(h->s, a.s);
    for (size_t k = 0; k < K; ++k) {
      const auto rk = widen_row(gens + k * 2 * Bref, Bref, a.s.B);
      {
        ScratchStore d;  // derivative of step k, dressed through the rest
        store_clone(a.s, d.s);
        dress_step(d.s, rk.data(), -sin_tau[k], cos_tau[k], 0.0, false, 0.0, nullptr, 0.0, true);
        for (size_t j = k + 1; j < K; ++j) {
          const auto rj = widen_row(gens + j * 2 * Bref, Bref, d.s.B);
          dress_step(d.s, rj.data(), cos_tau[j], sin_tau[j], 0.0, false, 0.0);
        }
        grad[k] = expect_store(d.s, factors);
      }
      if (k + 1 < K) dress_step(a.s, rk.data(), cos_tau[k], sin_tau[k], 0.0, false, 0.0);
    }
  });
}

int iqcc_gpu_expect(iqcc_gpu_sum* h, const double* factors, double* energy) {
  return guarded([&] {
    need(h);
    *energy = expect_store(h->s, factors);
  });
}

int iqcc_gpu_qmf_energy_gradient(iqcc_gpu_sum* h, const double* factors, const double* derivs,
                                 double* energy, double* grad) {
  return guarded([&] {
    need(h);
    *energy = qmf_grad_store(h->s, factors, derivs, grad);
  });
}

int iqcc_gpu_gradients(iqcc_gpu_sum* h, const double* factors, const uint64_t* cands, size_t K,
                       int flip_group_only, double* g) {
  return guarded([&] {
    need(h);
    const uint32_t Bref = ref_blocks(h->s);
    std::vector<uint64_t> wide(K * 2 * h->s.B);
    for (size_t k = 0; k < K; ++k) {
      auto r = widen_row(cands + k * 2 * Bref, Bref, h->s.B);
      std::copy(r.begin(), r.end(), wide.begin() + k * 2 * h->s.B);
    }
    gradients_store(h->s, factors, wide.data(), K, flip_group_only != 0, g);
  });
}

int iqcc_gpu_poly_kernels(iqcc_gpu_sum* h, const double* factors, int at_poles, const uint64_t* words,
                          size_t t, double* h_kernel, double* n_kernel) {
  return guarded([&] {
    need(h);
    if (t > 0 && (!words || !h_kernel || !n_kernel))
      throw std::invalid_argument("build_poly_kernels: null buffer");
    const uint32_t Bref = ref_blocks(h->s);
    std::vector<uint64_t> wide(t * 2 * h->s.B);
    for (size_t k = 0; k < t; ++k) {
      auto r = widen_row(words + k * 2 * Bref, Bref, h->s.B);
      std::copy(r.begin(), r.end(), wide.begin() + k * 2 * h->s.B);
    }
    poly_kernels_store(h->s, factors, at_poles != 0, wide.data(), t, h_kernel, n_kernel);
  });
}

int iqcc_gpu_dis_candidates(iqcc_gpu_sum* h, const double* factors, int at_poles, size_t top_k,
                            double screen_thr, size_t per_group_cap, int has_seed, uint64_t seed,
                            uint64_t* rows_out, double* g_out, size_t cap, size_t* n_picks) {
  return guarded([&] {
    need(h);
    if (top_k < 1) throw std::invalid_argument("dis_candidates: top_k < 1");
    std::vector<uint64_t> rows;
    std::vector<double> g;
    size_t n = dis_store(h->s, factors, at_poles != 0, top_k, screen_thr, per_group_cap, rows, g);
    std::vector<size_t> order(n);
    for (size_t i = 0; i < n; ++i) order[i] = i;
    if (has_seed) {  // iqcc/dis.hpp:172-188: reshuffle runs of equal magnitude
      std::mt19937_64 rng(seed);
      size_t i = 0;
      while (i < n) {
        size_t j = i + 1;
        const double mag = std::abs(g[order[i]]);
        while (j < n && std::abs(std::abs(g[order[j]]) - mag) <= 1e-12 * std::max(1.0, mag)) ++j;
        std::shuffle(order.begin() + i, order.begin() + j, rng);
        i = j;
      }
    }
    const uint32_t Bref = ref_blocks(h->s), B = h->s.B;
    const size_t w = std::min(cap, std::min(n, top_k));
    for (size_t i = 0; i < w; ++i) {
      const size_t o = order[i];
      for (uint32_t b = 0; b < Bref; ++b) {
        rows_out[i * 2 * Bref + b] = rows[o * 2 * B + b];
        rows_out[i * 2 * Bref + Bref + b] = rows[o * 2 * B + B + b];
      }
      g_out[i] = g[o];
    }
    *n_picks = n;
  });
}

int iqcc_gpu_choose_partition_bits(iqcc_gpu_sum* h, size_t m, size_t* bits_out, double* imbalance) {
  return guarded([&] {
    need(h);
    *imbalance = choose_bits_store(h->s, m, bits_out);
  });
}

int iqcc_gpu_sum_restrict(iqcc_gpu_sum* h, size_t m, const size_t* bits, const size_t* owner,
                          int rank) {
  return guarded([&] {
    need(h);
    restrict_store(h->s, m, bits, owner, rank);
  });
}

int iqcc_gpu_nccl_unique_id(void* out128) {
  return guarded([&] { multi_unique_id(out128); });
}

int iqcc_gpu_comm_init(const void* uid, int rank, int world) {
  return guarded([&] {
    ctx();
    multi_init(uid, rank, world);
    g_comm_ctx = g_ctx;
  });
}

int iqcc_gpu_comm_destroy(void) {
  return guarded([&] {
    multi_shutdown();
    g_comm_ctx = nullptr;
  });
}

int iqcc_gpu_parallel_dress(iqcc_gpu_sum* h, size_t m, const size_t* bits, const size_t* owner,
                            const uint64_t* gen, double cos_tau, double sin_tau, double eps,
                            size_t max_terms, iqcc_exchange_stats* xs, iqcc_compress_stats* cs) {
  return guarded([&] {
    need(h);
    const uint32_t Bref = ref_blocks(h->s);
    if (row_is_identity(gen, Bref)) throw std::invalid_argument("parallel_dress: identity generator");
    if (max_terms < 1) throw std::invalid_argument("compress_partitioned: max_terms < 1");
    auto row = widen_row(gen, Bref, h->s.B);
    multi_prepare(h->s);
    parallel_dress_step(h->s, m, bits, owner, row.data(), cos_tau, sin_tau, eps, max_terms, xs, cs);
  });
}

int iqcc_gpu_parallel_reserve(iqcc_gpu_sum* h, size_t terms) {
  return guarded([&] {
    need(h);
    parallel_reserve(h->s, terms);
  });
}

int iqcc_gpu_parallel_compress(iqcc_gpu_sum* h, double eps, size_t max_terms, iqcc_compress_stats* cs) {
  return guarded([&] {
    need(h);
    if (!(eps >= 0.0)) throw std::invalid_argument("compress_partitioned: epsilon < 0");
    if (max_terms < 1) throw std::invalid_argument("compress_partitioned: max_terms < 1");
    parallel_compress_store(h->s, eps, max_terms, cs);
  });
}

int iqcc_gpu_parallel_dress_sequence(iqcc_gpu_sum* h, size_t m, const size_t* bits,
                                     const size_t* owner, size_t K, const uint64_t* gens,
                                     const double* cos_tau, const double* sin_tau, double eps,
                                     size_t max_terms, iqcc_exchange_stats* xs,
                                     iqcc_compress_stats* cs, size_t* terms_in_total) {
  return guarded([&] {
    need(h);
    const uint32_t Bref = ref_blocks(h->s);
    if (max_terms < 1) throw std::invalid_argument("compress_partitioned: max_terms < 1");
    for (size_t k = 0; k < K; ++k)
      if (row_is_identity(gens + k * 2 * Bref, Bref))
        throw std::invalid_argument("parallel_dress: identity generator");
    size_t local_in = 0;
    multi_prepare(h->s);
    // output-slot speculation as in iqcc_gpu_dress_sequence; the cut is
    // global (compress_partitioned), so every rank guesses the same theta
    // and the verification runs on allreduced counts
    const bool slots = cs == nullptr && getenv("IQCC_NO_SPEC") == nullptr;
    const char* sc_env = getenv("IQCC_SPEC_SCALE");  // test hook: force bad guesses
    const double spec_scale = sc_env ? std::atof(sc_env) : 1.0;
    double spec = slots ? h->s.spec_cut : 0.0;
    const bool maybe = eps > 0.0 || max_terms != SIZE_MAX;
    for (size_t k = 0; k < K; ++k) {
      auto row = widen_row(gens + k * 2 * Bref, Bref, h->s.B);
      std::vector<uint64_t> next;
      if (k + 1 < K) next = widen_row(gens + (k + 1) * 2 * Bref, Bref, h->s.B);
      local_in += h->s.logical;
      const double exact = slots && eps > 0.0 ? eps : 0.0;
      const double guess = spec * std::min(1.0, std::fabs(cos_tau[k])) * 0.999 * spec_scale;
      const double theta = maybe && guess > eps && max_terms != SIZE_MAX ? guess : exact;
      bool failed = false;
      parallel_dress_step(h->s, m, bits, owner, row.data(), cos_tau[k], sin_tau[k], eps, max_terms,
                          xs ? xs + k : nullptr, cs, next.empty() ? nullptr : next.data(), theta,
                          exact, &failed);
      if (failed) spec = h->s.spec_cut = 0.0;
      const Filter& f = h->s.filt;
      if (slots && f.active && f.has_v && f.v > 0.0 && std::isfinite(f.v))
        spec = h->s.spec_cut = f.v;
      else if (slots && !failed && theta > exact)  // no cut: theta is the verified floor
        spec = h->s.spec_cut = theta;
    }
    if (terms_in_total) *terms_in_total = parallel_sum(local_in);
  });
}

int iqcc_gpu_parallel_expect(iqcc_gpu_sum* h, const double* factors, double* energy) {
  return guarded([&] {
    need(h);
    *energy = parallel_expect_store(h->s, factors);
  });
}

int iqcc_gpu_parallel_poly_kernels(iqcc_gpu_sum* h, const double* factors, int at_poles, const uint64_t* words,
                                   size_t t, double* h_kernel, double* n_kernel) {
  return guarded([&] {
    need(h);
    if (t > 0 && (!words || !h_kernel || !n_kernel))
      throw std::invalid_argument("build_poly_kernels: null buffer");
    const uint32_t Bref = ref_blocks(h->s);
    std::vector<uint64_t> wide(t * 2 * h->s.B);
    for (size_t k = 0; k < t; ++k) {
      auto r = widen_row(words + k * 2 * Bref, Bref, h->s.B);
      std::copy(r.begin(), r.end(), wide.begin() + k * 2 * h->s.B);
    }
    parallel_poly_kernels_store(h->s, factors, at_poles != 0, wide.data(), t, h_kernel, n_kernel);
  });
}

int iqcc_gpu_parallel_qmf_energy_gradient(iqcc_gpu_sum* h, const double* factors, const double* derivs,
                                          double* energy, double* grad) {
  return guarded([&] {
    need(h);
    *energy = parallel_qmf_grad_store(h->s, factors, derivs, grad);
  });
}

int iqcc_gpu_parallel_gradients(iqcc_gpu_sum* h, const double* factors, const uint64_t* cands, size_t K,
                                int flip_group_only, double* g) {
  return guarded([&] {
    need(h);
    const uint32_t Bref = ref_blocks(h->s);
    std::vector<uint64_t> wide(std::max<size_t>(K, 1) * 2 * h->s.B);
    for (size_t k = 0; k < K; ++k) {
      auto r = widen_row(cands + k * 2 * Bref, Bref, h->s.B);
      std::copy(r.begin(), r.end(), wide.begin() + k * 2 * h->s.B);
    }
    parallel_gradients_store(h->s, factors, wide.data(), K, flip_group_only != 0, g);
  });
}

int iqcc_gpu_merge_sums(iqcc_gpu_sum* a, iqcc_gpu_sum* b, double drop_thr, iqcc_gpu_sum** out) {
  return guarded([&] {
    need(a);
    need(b);
    if (!(drop_thr >= 0.0)) throw std::invalid_argument("merge_sums: drop_threshold < 0");
    auto h = std::make_unique<iqcc_gpu_sum>();
    merge_sums_store(a->s, b->s, drop_thr, h->s);
    *out = h.release();
  });
}

// ---- partitioned sums (psum.cu)
int iqcc_gpu_psum_distribute(size_t n_qubits, const uint64_t* rows, const double* coeff, size_t M, size_t m,
                             const size_t* bits, const size_t* owner, size_t n_workers, const int* devices,
                             iqcc_gpu_psum** out) {
  return guarded([&] {
    if (!out || !bits || !owner) throw std::invalid_argument("psum_distribute: null argument");
    *out = reinterpret_cast<iqcc_gpu_psum*>(
        psum_distribute(n_qubits, rows, coeff, M, m, bits, owner, n_workers, devices));
  });
}

int iqcc_gpu_psum_create_shards(size_t n_qubits, size_t m, const size_t* bits, const size_t* owner,
                                size_t n_workers, const int* devices, const uint64_t* const* rows,
                                const double* const* coeffs, const size_t* sizes, iqcc_gpu_psum** out) {
  return guarded([&] {
    if (!out || !owner || !sizes || (m && !bits)) throw std::invalid_argument("psum_create_shards: null argument");
    *out = reinterpret_cast<iqcc_gpu_psum*>(
        psum_from_shards(n_qubits, m, bits, owner, n_workers, devices, rows, coeffs, sizes));
  });
}

static PSum& psum_of(iqcc_gpu_psum* ph) {
  if (!ph) throw std::invalid_argument("null partitioned-sum handle");
  return *reinterpret_cast<PSum*>(ph);
}

int iqcc_gpu_psum_destroy(iqcc_gpu_psum* ph) {
  return guarded([&] {
    if (ph) psum_destroy(reinterpret_cast<PSum*>(ph));
  });
}

int iqcc_gpu_psum_info(iqcc_gpu_psum* ph, size_t* n_partitions, size_t* total_terms) {
  return guarded([&] {
    PSum& P = psum_of(ph);
    const size_t n = psum_parts(P);
    std::vector<size_t> sz(n);
    psum_sizes(P, sz.data());
    if (n_partitions) *n_partitions = n;
    if (total_terms) {
      size_t t = 0;
      for (size_t v : sz) t += v;
      *total_terms = t;
    }
  });
}

int iqcc_gpu_psum_shard_sizes(iqcc_gpu_psum* ph, size_t* sizes) {
  return guarded([&] { psum_sizes(psum_of(ph), sizes); });
}

int iqcc_gpu_psum_owner(iqcc_gpu_psum* ph, size_t* owner) {
  return guarded([&] { psum_owner(psum_of(ph), owner); });
}

int iqcc_gpu_psum_download_shard(iqcc_gpu_psum* ph, size_t p, uint64_t* rows, double* coeff, size_t cap,
                                 size_t* M) {
  return guarded([&] { *M = psum_download_shard(psum_of(ph), p, rows, coeff, cap); });
}

int iqcc_gpu_psum_gather(iqcc_gpu_psum* ph, uint64_t* rows, double* coeff, size_t cap, size_t* M) {
  return guarded([&] { *M = psum_gather(psum_of(ph), rows, coeff, cap); });
}

int iqcc_gpu_psum_dress(iqcc_gpu_psum* ph, const uint64_t* gen, double cos_tau, double sin_tau, double eps,
                        size_t max_terms, iqcc_message_record* log, size_t log_cap, size_t* n_log,
                        iqcc_compress_stats* cstats, size_t* mask) {
  return guarded([&] {
    psum_dress(psum_of(ph), gen, cos_tau, sin_tau, eps, max_terms, log, log_cap, n_log, cstats, mask);
  });
}

int iqcc_gpu_psum_expect(iqcc_gpu_psum* ph, const double* factors, double* energy) {
  return guarded([&] { *energy = psum_expect(psum_of(ph), factors); });
}

int iqcc_gpu_psum_qmf_energy_gradient(iqcc_gpu_psum* ph, const double* factors, const double* derivs,
                                      double* energy, double* grad) {
  return guarded([&] { *energy = psum_qmf_energy_gradient(psum_of(ph), factors, derivs, grad); });
}

int iqcc_gpu_psum_gradients(iqcc_gpu_psum* ph, const double* factors, const uint64_t* cands, size_t K,
                            int flip_group_only, double* g) {
  return guarded([&] { psum_gradients(psum_of(ph), factors, cands, K, flip_group_only != 0, g); });
}

int iqcc_gpu_psum_rebalance(iqcc_gpu_psum* ph, double threshold, size_t* owner_out) {
  return guarded([&] { psum_rebalance(psum_of(ph), threshold, owner_out); });
}

int iqcc_gpu_parallel_size(iqcc_gpu_sum* h, size_t* total) {
  return guarded([&] {
    need(h);
    *total = parallel_size(h->s);
  });
}

}  // extern "C"
#pragma GCC visibility pop
