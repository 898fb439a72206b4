// multi.cu — bit-wise partitioning across GPUs (one process per GPU, NCCL).
//
// parallel_dress (iqcc/partition.hpp:398-452) with one partition per rank
// (2^m == world, owner a permutation): a term's partition key is the gather
// of its bits at the partition positions (partition.hpp:40-42); survivors
// never move and every product of partition p has key p ^ mask, mask = the
// entangler's key.  So:
//   mask == 0  -> purely local dressing step, no communication;
//   mask != 0  -> each rank orders its products locally (same trie-rank
//                 pipeline), materializes them, swaps them with the rank
//                 owning p ^ mask (pairwise ncclSend/ncclRecv on the engine
//                 stream), and merges its survivors with the received,
//                 already sorted products.
// compress_partitioned (partition.hpp:325-396) runs with allreduced
// histograms and an allgather of the (few) tied words for the canonical
// tie-break.  Energies: per-rank partial sums allgathered and added in rank
// order (reduce_scalar, partition.hpp:233-237).
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "multi.cuh"

namespace iqcc_b200 {

namespace {

struct Comm {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  ull* dev = nullptr;  // small device scratch for collectives
};
Comm g_comm;

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw std::runtime_error(std::string("NCCL error ") + ncclGetErrorString(r) + " at " + what);
}
#define IQCC_NCCL(x) nccl_check((x), #x)

Comm& comm() {
  if (!g_comm.comm) throw std::runtime_error("iqcc_gpu_comm_init has not been called");
  return g_comm;
}

ull* scratch(size_t n) {
  Workspace& ws = workspace();
  return ws.misc3.as<ull>(n);
}

struct NcclReducer : Reducer {
  void sum(ull* vals, size_t n) override {
    Comm& c = comm();
    cudaStream_t st = stream();
    ull* d = workspace().partials.as<ull>(n);
    ull* hp = static_cast<ull*>(host_pinned(n * sizeof(ull)));
    std::memcpy(hp, vals, n * sizeof(ull));
    IQCC_CUDA(cudaMemcpyAsync(d, hp, n * sizeof(ull), cudaMemcpyHostToDevice, st));
    IQCC_NCCL(ncclAllReduce(d, d, n, ncclUint64, ncclSum, c.comm, st));
    d2h_small(hp, d, n * sizeof(ull), st);
    host_sync(st);
    std::memcpy(vals, hp, n * sizeof(ull));
  }
  void sum_device(ull* d, size_t n) override {
    // (a one-kernel allreduce over NVLink mailboxes measured no faster than
    // NCCL here: the time in these collectives is the ranks' skew)
    IQCC_NCCL(ncclAllReduce(d, d, n, ncclUint64, ncclSum, comm().comm, stream()));
  }
  bool allgather_device(const ull* send, ull* recv, size_t n) override {
    IQCC_NCCL(ncclAllGather(send, recv, n, ncclUint64, comm().comm, stream()));
    return true;
  }
  bool can_allgather() const override { return true; }
  int group_size() const override { return g_comm.world; }
  int group_rank() const override { return g_comm.rank; }
  std::vector<ull> gather_keys(const std::vector<ull>& mine, size_t W, size_t* mine_off) override {
    Comm& c = comm();
    cudaStream_t st = stream();
    std::vector<ull> counts(c.world, 0);
    counts[c.rank] = mine.size() / W;
    sum(counts.data(), counts.size());
    size_t mx = 0, off = 0;
    for (int r = 0; r < c.world; ++r) {
      mx = std::max<size_t>(mx, counts[r]);
      if (r < c.rank) off += counts[r];
    }
    *mine_off = off;
    std::vector<ull> all;
    if (mx == 0) return all;
    ull* d = workspace().rbuf_keys.as<ull>((size_t)mx * W * (c.world + 1));
    ull* dm = d + (size_t)mx * W * c.world;
    IQCC_CUDA(cudaMemsetAsync(dm, 0, mx * W * sizeof(ull), st));
    if (!mine.empty())
      IQCC_CUDA(cudaMemcpyAsync(dm, mine.data(), mine.size() * sizeof(ull), cudaMemcpyHostToDevice, st));
    IQCC_NCCL(ncclAllGather(dm, d, mx * W, ncclUint64, c.comm, st));
    std::vector<ull> padded((size_t)mx * W * c.world);
    d2h_small(padded.data(), d, padded.size() * sizeof(ull), st);
    host_sync(st);
    for (int r = 0; r < c.world; ++r)
      all.insert(all.end(), padded.begin() + (size_t)r * mx * W,
                 padded.begin() + (size_t)r * mx * W + counts[r] * W);
    return all;
  }
};

/// Receive buffers in peer-visible memory (CUDA IPC over NVLink).  Every
/// rank owns one buffer of the same agreed capacity `cap` (terms): keys
/// [cap][W] then values [cap].  A sender pushes its sorted products straight
/// into the partner's buffer (no staging copy, no NCCL data transfer), then
/// signals with a one-word NCCL send/recv, which orders the push before the
/// partner's merge.  Reuse is safe: a rank pushes only after the count swap
/// of that step, which the partner posts after its previous merge.
struct P2P {
  bool tried = false, ok = false;
  size_t cap = 0, W = 0;
  char* mine = nullptr;
  std::vector<char*> peer;  // mapping of every rank's buffer (own rank: mine)
};
P2P g_p2p;
size_t g_p2p_last_cap = 0;

// Chunked exchange (the default push): each rank materializes its sorted
// products chunk by chunk into local HBM, the copy engines move each chunk
// into the partner's receive buffer over NVLink (no SM time), and a
// one-thread kernel behind the copy raises the chunk's ready flag in the
// partner's buffer; the partner's merge waits for chunk c's flag only and
// merges chunk c while later chunks are still on the wire.
constexpr int kMaxChunks = 32;
constexpr size_t kChunkAlign = 32 * 1024;  // whole slot-bit scan blocks (PW words)

/// Byte offset of the ready flags (kMaxChunks u32) in a receive buffer.
size_t p2p_flag_off(size_t cap, size_t W) {
  return (cap * (W * 8 + 8) + (cap / 32 + 64) * 4 + 255) & ~(size_t)255;
}

constexpr size_t kP2PTail = 256;  // chunk flags
static_assert(kMaxChunks * sizeof(unsigned) <= kP2PTail, "chunk flags");

struct XState {
  cudaStream_t xst = nullptr;  // copy-engine stream
  std::vector<cudaEvent_t> ev;
  cudaEvent_t done = nullptr;
  unsigned* err = nullptr;  // mapped host word (device view): a ready-flag wait timed out
  unsigned* err_host = nullptr;
  unsigned epoch = 0;       // exchanges so far (same on every rank)
};
XState g_x;

XState& xstate() {
  if (!g_x.xst) {
    IQCC_CUDA(cudaStreamCreateWithFlags(&g_x.xst, cudaStreamNonBlocking));
    g_x.ev.resize(kMaxChunks);
    for (auto& e : g_x.ev) IQCC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    IQCC_CUDA(cudaEventCreateWithFlags(&g_x.done, cudaEventDisableTiming));
    // read by the host after the step's own synchronizations: no extra round trip
    IQCC_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&g_x.err_host), sizeof(unsigned), cudaHostAllocMapped));
    *g_x.err_host = 0;
    IQCC_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&g_x.err), g_x.err_host, 0));
  }
  return g_x;
}

int exchange_chunks() {
  static const int c = [] {
    const char* e = getenv("IQCC_XCHG_CHUNKS");
    const int v = e ? atoi(e) : 4;
    return std::max(1, std::min(v, kMaxChunks));
  }();
  return c;
}

struct KeyWords {
  ull w[8];
};

/// Sender: [A, r_1..r_{C-1}, key(r_1)..key(r_{C-1})] with r_c = c*A/C rounded
/// down to kChunkAlign, key(r) = the r-th sorted product's key (all ones
/// past the end).
__global__ void k_chunk_send(const long long* __restrict__ a_dev, const ull* __restrict__ keys,
                             const unsigned* __restrict__ inv_perm, int W, KeyWords P, int C,
                             ull* __restrict__ out) {
  const int c = threadIdx.x;
  const ull A = a_dev ? (ull)*a_dev : 0ull;
  if (c == 0) out[0] = A;
  if (c < 1 || c >= C) return;
  const ull r = ((A * (ull)c / (ull)C) / kChunkAlign) * kChunkAlign;
  out[c] = r;
  for (int w = 0; w < W; ++w)
    out[C + (size_t)(c - 1) * W + w] = r < A ? keys[(size_t)inv_perm[r] * W + w] ^ P.w[w] : ~0ull;
}

/// Receiver: where the partner's chunk split keys fall in this store
/// (lower bound: a run of equal survivors stays with its product), plus
/// both sides' counts and chunk starts for the host:
/// hb = [A, my r_1..r_{C-1}, nrecv, their r_1..r_{C-1}, a_1..a_{C-1}].
__global__ void k_chunk_bounds(const ull* __restrict__ mine, const ull* __restrict__ recv,
                               const ull* __restrict__ keys, size_t M, int W, int C,
                               ull* __restrict__ hb) {
  const int c = threadIdx.x;
  if (c < C) {
    hb[c] = mine[c];
    hb[C + c] = recv[c];
  }
  if (c < 1 || c >= C) return;
  const ull nrecv = recv[0], r = recv[c];
  size_t a = M;
  if (r < nrecv) {
    const ull* k = recv + C + (size_t)(c - 1) * W;
    size_t lo = 0, hi = M;
    while (lo < hi) {  // first store key >= k
      const size_t mid = (lo + hi) >> 1;
      int cmp = 0;
      for (int w = 0; w < W && cmp == 0; ++w) {
        const ull x = keys[mid * W + w];
        cmp = x < k[w] ? -1 : (x > k[w] ? 1 : 0);
      }
      if (cmp < 0)
        lo = mid + 1;
      else
        hi = mid;
    }
    a = lo;
  }
  hb[2 * C + c - 1] = a;
}

/// Raised behind a chunk's copy (stream order: the copy is complete).
__global__ void k_flag_signal(unsigned* flag, unsigned epoch) {
  __threadfence_system();
  asm volatile("st.release.sys.global.u32 [%0], %1;\n" ::"l"(flag), "r"(epoch) : "memory");
}

/// Blocks the engine stream until the partner raised chunk c's flag; gives
/// up after 60 s (err) rather than hang the device.
__global__ void k_flag_wait(const unsigned* flag, unsigned epoch, unsigned* err) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];\n" : "=r"(v) : "l"(flag) : "memory");
    if ((int)(v - epoch) >= 0) return;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 60ull * 1000000000ull) {
      *(volatile unsigned*)err = 1u;
      return;
    }
    __nanosleep(256);
  }
}

/// A ready-flag wait that gave up means the partner stopped
/// participating: fail loudly (checked after the step's synchronizations).
void check_wait_timeout() {
  if (g_x.err_host && *(volatile unsigned*)g_x.err_host) {
    *g_x.err_host = 0;
    throw std::runtime_error("parallel_dress: the partner's products did not arrive (60 s)");
  }
}

ull allreduce_host(ull v, ncclRedOp_t op) {
  Comm& c = comm();
  cudaStream_t st = stream();
  ull* d = scratch(2);
  ull* hp = static_cast<ull*>(host_pinned(sizeof(ull)));
  *hp = v;
  IQCC_CUDA(cudaMemcpyAsync(d, hp, sizeof(ull), cudaMemcpyHostToDevice, st));
  IQCC_NCCL(ncclAllReduce(d, d, 1, ncclUint64, op, c.comm, st));
  d2h_small(hp, d, sizeof(ull), st);
  host_sync(st);
  return *hp;
}

void p2p_close() {
  for (size_t r = 0; r < g_p2p.peer.size(); ++r)
    if (g_p2p.peer[r] && g_p2p.peer[r] != g_p2p.mine) cudaIpcCloseMemHandle(g_p2p.peer[r]);
  g_p2p.peer.clear();
}

void p2p_free() {
  if (g_p2p.mine) cudaFree(g_p2p.mine);
  g_p2p.mine = nullptr;
  g_p2p.cap = 0;
  g_p2p.ok = false;
}

/// Collective (every rank, same call sequence): make every receive buffer
/// hold at least `need` terms of W words (max over ranks).  Any failure on
/// any rank turns the P2P path off everywhere (NCCL transfers instead).
void p2p_prepare(size_t need, size_t W) {
  Comm& c = comm();
  if (c.world < 2) return;
  static const bool off = getenv("IQCC_NO_P2P") != nullptr;
  if (off || (g_p2p.tried && !g_p2p.ok && g_p2p.cap == 0 && g_p2p.W == (size_t)-1)) return;
  const ull need_g = allreduce_host((ull)need, ncclMax);
  if (g_p2p.ok && need_g <= g_p2p.cap && W == g_p2p.W) return;
  HostScope hs("host_p2p_prepare");
  // a store that outgrew its buffer keeps growing (uncapped dressing, C5):
  // regrow by 2x so the (costly) remap happens every other step at most
  const bool regrow = g_p2p.ok && W == g_p2p.W;
  cudaStream_t st = stream();
  IQCC_CUDA(cudaStreamSynchronize(st));
  p2p_close();
  allreduce_host(0, ncclSum);  // every mapping of the old buffers is closed
  p2p_free();
  g_p2p.tried = true;
  const size_t cap = regrow ? std::max<size_t>(2 * (size_t)need_g, 2 * g_p2p_last_cap) + 1024
                            : (size_t)need_g + need_g / 4 + 1024;
  bool ok = cudaMalloc(&g_p2p.mine, p2p_flag_off(cap, W) + kP2PTail) == cudaSuccess;
  if (ok) ok = cudaMemset(g_p2p.mine + p2p_flag_off(cap, W), 0, kP2PTail) == cudaSuccess;
  cudaIpcMemHandle_t h;
  std::memset(&h, 0, sizeof(h));
  if (ok) ok = cudaIpcGetMemHandle(&h, g_p2p.mine) == cudaSuccess;
  cudaGetLastError();
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  std::vector<ull> all(8 * (size_t)c.world);
  {
    ull* d = workspace().misc3.as<ull>(8 * ((size_t)c.world + 1));
    ull* hp = static_cast<ull*>(host_pinned(8 * ((size_t)c.world + 1) * sizeof(ull)));
    std::memcpy(hp, &h, 64);
    IQCC_CUDA(cudaMemcpyAsync(d + 8 * c.world, hp, 64, cudaMemcpyHostToDevice, st));
    IQCC_NCCL(ncclAllGather(d + 8 * c.world, d, 8, ncclUint64, c.comm, st));
    d2h_small(hp, d, 64 * c.world, st);
    host_sync(st);
    std::memcpy(all.data(), hp, 64 * c.world);
  }
  if (allreduce_host(ok ? 1 : 0, ncclMin) == 1) {
    g_p2p.peer.assign(c.world, nullptr);
    for (int r = 0; r < c.world && ok; ++r) {
      if (r == c.rank) {
        g_p2p.peer[r] = g_p2p.mine;
        continue;
      }
      cudaIpcMemHandle_t hr;
      std::memcpy(&hr, all.data() + 8 * r, 64);
      void* p = nullptr;
      ok = cudaIpcOpenMemHandle(&p, hr, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
      g_p2p.peer[r] = static_cast<char*>(p);
    }
    cudaGetLastError();
  } else {
    ok = false;
  }
  if (allreduce_host(ok ? 1 : 0, ncclMin) == 1) {
    g_p2p.ok = true;
    g_p2p.cap = cap;
    g_p2p_last_cap = cap;
    g_p2p.W = W;
    return;
  }
  if (getenv("IQCC_VERBOSE")) fprintf(stderr, "[p2p] CUDA IPC unavailable: NCCL transfers\n");
  p2p_close();
  p2p_free();
  g_p2p.W = (size_t)-1;  // permanently off
}

size_t key_of_row(const uint64_t* row, uint32_t B, size_t n, size_t m, const size_t* bits) {
  size_t key = 0;
  for (size_t b = 0; b < m; ++b) {
    const size_t p = bits[b];
    const size_t q = p < n ? p : p - n;
    const uint64_t w = row[(p < n ? 0 : B) + q / 64];
    key |= (size_t)((w >> (q % 64)) & 1u) << b;
  }
  return key;
}

}  // namespace

void multi_unique_id(void* out128) {
  ncclUniqueId id;
  IQCC_NCCL(ncclGetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  std::memcpy(out128, &id, 128);
}

void multi_init(const void* uid128, int rank, int world) {
  if (g_comm.comm) throw std::invalid_argument("communicator already initialised");
  if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("comm_init: bad rank/world");
  ncclUniqueId id;
  std::memcpy(&id, uid128, 128);
  IQCC_NCCL(ncclCommInitRank(&g_comm.comm, world, id, rank));
  g_comm.rank = rank;
  g_comm.world = world;
  // NCCL connects point-to-point peers lazily on first use; touch every
  // pair now so no connection setup lands inside a dressing sequence
  if (world > 1) {
    cudaStream_t st = stream();
    ull* d = scratch(2 * (size_t)world);
    IQCC_CUDA(cudaMemsetAsync(d, 0, 2 * (size_t)world * sizeof(ull), st));
    IQCC_NCCL(ncclGroupStart());
    for (int p = 0; p < world; ++p) {
      if (p == rank) continue;
      IQCC_NCCL(ncclSend(d + p, 1, ncclUint64, p, g_comm.comm, st));
      IQCC_NCCL(ncclRecv(d + world + p, 1, ncclUint64, p, g_comm.comm, st));
    }
    IQCC_NCCL(ncclGroupEnd());
    IQCC_NCCL(ncclAllReduce(d, d, 1, ncclUint64, ncclSum, g_comm.comm, st));
    IQCC_NCCL(ncclAllGather(d + rank, d + world, 1, ncclUint64, g_comm.comm, st));
    host_sync(st);
  }
}

void multi_prepare(DeviceStore& s) { p2p_prepare(s.M, 2 * (size_t)s.B); }

void multi_shutdown() {
  if (g_comm.comm) {
    cudaDeviceSynchronize();
    if (g_x.xst) {
      for (auto e : g_x.ev) cudaEventDestroy(e);
      cudaEventDestroy(g_x.done);
      cudaFreeHost(g_x.err_host);
      cudaStreamDestroy(g_x.xst);
      g_x = XState{};
    }
    p2p_close();
    p2p_free();
    g_p2p = P2P{};
    ncclCommDestroy(g_comm.comm);
    g_comm = Comm{};
  }
}

void parallel_dress_step(DeviceStore& s, size_t m, const size_t* bits, const size_t* owner,
                         const uint64_t* gen_row, double cs, double sn, double eps,
                         size_t max_terms, iqcc_exchange_stats* xs, iqcc_compress_stats* cs_out,
                         const uint64_t* next_row, double theta, double exact, bool* spec_failed) {
  Comm& c = comm();
  if (((size_t)1 << m) != (size_t)c.world)
    throw std::invalid_argument("parallel_dress: one partition per rank (2^m == world) required");
  size_t mine = SIZE_MAX;
  for (size_t p = 0; p < ((size_t)1 << m); ++p) {
    if (owner[p] >= (size_t)c.world) throw std::invalid_argument("PartitionMap: owner out of range");
    if (owner[p] == (size_t)c.rank) mine = p;
  }
  if (mine == SIZE_MAX) throw std::invalid_argument("parallel_dress: rank owns no partition");
  const uint32_t Bref = s.n_qubits == 0 ? 1 : (s.n_qubits + 63) / 64;
  std::vector<uint64_t> ref_row(2 * Bref);
  for (uint32_t w = 0; w < Bref; ++w) {
    ref_row[w] = gen_row[w];
    ref_row[Bref + w] = gen_row[s.B + w];
  }
  const size_t mask = key_of_row(ref_row.data(), Bref, s.n_qubits, m, bits);
  const bool want_hist = eps > 0.0 || max_terms != SIZE_MAX;
  if (!want_hist) theta = exact = 0.0;  // no compress follows: every term keeps a slot
  const bool exch = !(mask == 0 || sn == 0.0);
  // host wall time per step kind (each step ends with a synchronize, so it
  // tracks the device time): SURVEY §8(d) C3 reports mask = 0 and mask != 0
  // steps separately
  HostScope step_scope(exch ? "step_exchange" : "step_local");
  const size_t M0 = s.M, L0 = s.logical;
  const Filter F0 = s.filt;
  DressOutcome o;
  iqcc_exchange_stats x{mask, 0, 0, 0, 0};
  size_t nrecv = 0;
  ull* rk = nullptr;
  double* rv = nullptr;
  NcclReducer red;
  struct Hook {  // merges of this step allreduce their counts on the device
    explicit Hook(Reducer* r) { set_merge_reducer(r); }
    ~Hook() { set_merge_reducer(nullptr); }
  } hook(want_hist ? &red : nullptr);
  if (!exch) {
    o = dress_step(s, gen_row, cs, sn, 1e-12, want_hist, eps, next_row, theta);
  } else {
    cudaStream_t st = stream();
    Workspace& ws = workspace();
    // plan, then swap the product counts with the partner straight from
    // device memory: one round trip gives both A and the receive count
    const long long* a_dev = plan_products_async(s, gen_row, cs, sn, theta);
    const int peer = (int)owner[mine ^ mask];
    const size_t W = 2 * s.B;
    static const bool pull = getenv("IQCC_XCHG") && std::string(getenv("IQCC_XCHG")) == "pull";
    // chunked push (every rank decides alike: the P2P state is agreed)
    const int C = (g_p2p.ok && g_p2p.W == W && !pull) ? exchange_chunks() : 1;
    const bool chunked = C > 1;
    // one swap gives A and the receive count (chunked: also both sides'
    // chunk starts and where the partner's chunk keys fall in this store)
    const size_t S = chunked ? (size_t)C + (size_t)(C - 1) * W : 1;
    ull* cnt = scratch(2 * S + 3 * (size_t)C + 8);
    ull* hbd = cnt + 2 * S;
    if (chunked) {
      KeyWords Pw{};
      row_to_device_key(gen_row, s.B, Pw.w);
      k_chunk_send<<<1, 32, 0, st>>>(a_dev, s.keys(), plan_inv_perm(), (int)W, Pw, C, cnt);
    } else if (a_dev) {
      IQCC_CUDA(cudaMemcpyAsync(cnt, a_dev, sizeof(ull), cudaMemcpyDeviceToDevice, st));
    } else {
      IQCC_CUDA(cudaMemsetAsync(cnt, 0, sizeof(ull), st));
    }
    {
      KernelScope ks("exch_count");
      IQCC_NCCL(ncclGroupStart());
      IQCC_NCCL(ncclSend(cnt, S, ncclUint64, peer, c.comm, st));
      IQCC_NCCL(ncclRecv(cnt + S, S, ncclUint64, peer, c.comm, st));
      IQCC_NCCL(ncclGroupEnd());
    }
    std::vector<ull> hb(3 * (size_t)C);
    if (chunked) {
      k_chunk_bounds<<<1, 32, 0, st>>>(cnt, cnt + S, s.keys(), s.M, (int)W, C, hbd);
      ull* hp = static_cast<ull*>(host_pinned((3 * (size_t)C - 1) * sizeof(ull)));
      d2h_small(hp, hbd, (3 * (size_t)C - 1) * sizeof(ull), st);
      host_sync(st);
      std::copy(hp, hp + 3 * C - 1, hb.begin());
    } else {
      ull* hp = static_cast<ull*>(host_pinned(2 * sizeof(ull)));
      d2h_small(hp, cnt, sizeof(ull), st);
      d2h_small(hp + 1, cnt + S, sizeof(ull), st);
      host_sync(st);
      hb[0] = hp[0];
      hb[1] = hp[1];  // (chunked layout: hb[C])
    }
    const size_t A = hb[0];
    nrecv = chunked ? hb[C] : hb[1];
    plan_set_products(A);
    // both ends see the same (A, nrecv) and the same agreed capacity
    const bool p2p = g_p2p.ok && g_p2p.W == W && A <= g_p2p.cap && nrecv <= g_p2p.cap;
    // exchange buffers sized by the shard (products <= terms), so they do
    // not regrow from step to step
    const size_t xcap = std::max<size_t>({A, nrecv, s.M, 1});
    ull* sk = p2p ? nullptr : ws.xbuf_keys.as<ull>(xcap * W);
    double* sv = p2p ? nullptr : ws.xbuf_coef.as<double>(xcap);
    // IQCC_XCHG=pull: each rank writes its sorted products (and the
    // receiver's slot bits) into its OWN peer-visible buffer at HBM speed,
    // and the partner's merge reads them over NVLink while it merges (no
    // separate transfer pass); default: the chunked push (IQCC_XCHG_CHUNKS=1:
    // one SM push of everything, then the merge)
    const unsigned* rbits = nullptr;
    ChunkPlan cp;
    if (p2p && chunked) {
      XState& xs = xstate();
      const unsigned epoch = ++xs.epoch;
      ull* stk = ws.xbuf_keys.as<ull>(std::max<size_t>(A, 1) * W);
      double* stv = ws.xbuf_coef.as<double>(std::max<size_t>(A, 1));
      char* dst = g_p2p.peer[peer];
      ull* dk = reinterpret_cast<ull*>(dst);
      double* dv = reinterpret_cast<double*>(dst + g_p2p.cap * W * 8);
      unsigned* pflag = reinterpret_cast<unsigned*>(dst + p2p_flag_off(g_p2p.cap, W));
      const unsigned* mflag = reinterpret_cast<const unsigned*>(g_p2p.mine + p2p_flag_off(g_p2p.cap, W));
      std::vector<size_t> mr(C + 1);
      mr[0] = 0;
      mr[C] = A;
      for (int k = 1; k < C; ++k) mr[k] = hb[k];
      // IQCC_XCHG_SM=<CTAs>: the chunks leave through SM stores into the
      // partner's buffer (a push kernel with that many CTAs beside the merge)
      // instead of local staging + copy engine
      static const unsigned sm_push = getenv("IQCC_XCHG_SM") ? (unsigned)atoi(getenv("IQCC_XCHG_SM")) : 0u;
      if (sm_push) {
        IQCC_CUDA(cudaEventRecord(xs.ev[0], st));  // the plan is done
        IQCC_CUDA(cudaStreamWaitEvent(xs.xst, xs.ev[0], 0));
      }
      for (int k = 0; k < C && sm_push; ++k) {
        push_products(s, gen_row, sn, dk, dv, mr[k], mr[k + 1], xs.xst, sm_push);
        k_flag_signal<<<1, 1, 0, xs.xst>>>(pflag + k, epoch);
      }
      for (int k = 0; k < C && !sm_push; ++k) {
        // chunk k into local HBM (SMs), then onto the wire (copy engine)
        materialize_products(s, gen_row, sn, stk, stv, mr[k], mr[k + 1], "exchange");
        IQCC_CUDA(cudaEventRecord(xs.ev[k], st));
        IQCC_CUDA(cudaStreamWaitEvent(xs.xst, xs.ev[k], 0));
        if (mr[k + 1] > mr[k]) {
          IQCC_CUDA(cudaMemcpyAsync(dk + mr[k] * W, stk + mr[k] * W, (mr[k + 1] - mr[k]) * W * 8,
                                    cudaMemcpyDeviceToDevice, xs.xst));
          IQCC_CUDA(cudaMemcpyAsync(dv + mr[k], stv + mr[k], (mr[k + 1] - mr[k]) * 8,
                                    cudaMemcpyDeviceToDevice, xs.xst));
        }
        k_flag_signal<<<1, 1, 0, xs.xst>>>(pflag + k, epoch);
      }
      IQCC_CUDA(cudaEventRecord(xs.done, xs.xst));
      rk = reinterpret_cast<ull*>(g_p2p.mine);
      rv = reinterpret_cast<double*>(g_p2p.mine + g_p2p.cap * W * 8);
      cp.C = C;
      cp.a.assign(C + 1, 0);
      cp.r.assign(C + 1, 0);
      for (int k = 1; k < C; ++k) {
        cp.r[k] = hb[C + k];
        cp.a[k] = hb[2 * C + k - 1];
      }
      cp.a[C] = s.M;
      cp.r[C] = nrecv;
      recv_slot_bits_begin(nrecv, theta, C);
      const unsigned* err = xs.err;
      cp.arrive = [&cp, mflag, epoch, err, rv, nrecv, st](int k, const unsigned** qt, size_t* wq) {
        {
          KernelScope ks("exchange");
          k_flag_wait<<<1, 1, 0, st>>>(mflag + k, epoch, const_cast<unsigned*>(err));
        }
        recv_slot_bits_chunk(rv, cp.r[k], cp.r[k + 1], nrecv, k, qt, wq);
      };
    } else if (p2p && pull) {
      char* mine = g_p2p.mine;
      unsigned* mbits = reinterpret_cast<unsigned*>(mine + g_p2p.cap * (W * 8 + 8));
      materialize_products(s, gen_row, sn, reinterpret_cast<ull*>(mine),
                           reinterpret_cast<double*>(mine + g_p2p.cap * W * 8), 0, SIZE_MAX, "exchange", theta,
                           theta != 0.0 ? mbits : nullptr);
      KernelScope ks2("exch_signal");
      char* src = g_p2p.peer[peer];
      rk = reinterpret_cast<ull*>(src);
      rv = reinterpret_cast<double*>(src + g_p2p.cap * W * 8);
      rbits = reinterpret_cast<const unsigned*>(src + g_p2p.cap * (W * 8 + 8));
      // my products are written -> the partner may read them (and its are ready)
      IQCC_NCCL(ncclGroupStart());
      IQCC_NCCL(ncclSend(cnt, 1, ncclUint64, peer, c.comm, st));
      IQCC_NCCL(ncclRecv(cnt + 2, 1, ncclUint64, peer, c.comm, st));
      IQCC_NCCL(ncclGroupEnd());
    } else if (p2p) {
      // the SMs gather the sorted products and write them, tile by tile,
      // straight into the partner's receive buffer over NVLink
      char* dst = g_p2p.peer[peer];
      push_products(s, gen_row, sn, reinterpret_cast<ull*>(dst),
                    reinterpret_cast<double*>(dst + g_p2p.cap * W * 8));
      KernelScope ks2("exch_signal");
      rk = reinterpret_cast<ull*>(g_p2p.mine);
      rv = reinterpret_cast<double*>(g_p2p.mine + g_p2p.cap * W * 8);
      // push done -> the partner may merge (and my own products arrived)
      IQCC_NCCL(ncclGroupStart());
      IQCC_NCCL(ncclSend(cnt, 1, ncclUint64, peer, c.comm, st));
      IQCC_NCCL(ncclRecv(cnt + 2, 1, ncclUint64, peer, c.comm, st));
      IQCC_NCCL(ncclGroupEnd());
    } else {
      materialize_products(s, gen_row, sn, sk, sv);
      rk = ws.rbuf_keys.as<ull>(xcap * W);
      rv = ws.rbuf_coef.as<double>(xcap);
    }
    if (!p2p) {
      KernelScope ks("exchange");
      IQCC_NCCL(ncclGroupStart());
      if (A) {
        IQCC_NCCL(ncclSend(sk, A * W, ncclUint64, peer, c.comm, st));
        IQCC_NCCL(ncclSend(sv, A, ncclFloat64, peer, c.comm, st));
      }
      if (nrecv) {
        IQCC_NCCL(ncclRecv(rk, nrecv * W, ncclUint64, peer, c.comm, st));
        IQCC_NCCL(ncclRecv(rv, nrecv, ncclFloat64, peer, c.comm, st));
      }
      IQCC_NCCL(ncclGroupEnd());
    }
    x.sent_terms = A;
    x.recv_terms = nrecv;
    x.bytes_wire = A * (W * 8 + 8);
    x.bytes_reference = A * (16 + Bref * 16);  // MessageLog formula, partition.hpp:420-422
    if (cp.C > 1) {
      o = merge_products(s, gen_row, cs, sn, 1e-12, want_hist, eps, nrecv, rk, rv, next_row, theta, &cp);
      // the staging buffer is free again once the copies are done; and a
      // timed-out wait means the partner never delivered
      IQCC_CUDA(cudaStreamWaitEvent(st, g_x.done, 0));
      check_wait_timeout();  // (the merge ended with a synchronize)
    } else {
      if (rbits)
        recv_slot_bits_packed(rbits, nrecv, theta);
      else
        recv_slot_bits(rv, nrecv, theta);
      o = merge_products(s, gen_row, cs, sn, 1e-12, want_hist, eps, nrecv, rk, rv, next_row, theta);
    }
  }
  if (xs) *xs = x;
  if (!want_hist) return;  // eps == 0 and no cap: compress_partitioned is a no-op
  // global counts of the step: count_eps, |c| >= theta, identity
  ull glob[3] = {(ull)o.count_eps, (ull)o.n_ge_theta, (ull)(s.has_identity ? 1 : 0)};
  if (o.has_glob)
    std::copy(o.glob, o.glob + 3, glob);
  else
    red.sum(glob, 3);
  double floor_cut = 0.0;  // verified lower bound of the cut (speculation passed)
  if (theta > exact) {
    // the slotted shards compress like the full ones iff the global top
    // `budget` terms are all >= theta and either the compress cuts or no
    // term below theta held a slot (as in the single-device sequence)
    const ull idc = glob[2] ? 1 : 0;
    const ull budget = max_terms - idc;
    const bool ok = glob[1] >= budget && (glob[0] > max_terms || glob[0] == glob[1] + idc);
    if (ok) floor_cut = theta;
    if (!ok) {  // every rank sees the same sums and redoes the step exactly
      dress_undo(s, M0, L0, F0);
      if (!exch) {
        o = dress_step(s, gen_row, cs, sn, 1e-12, want_hist, eps, next_row, exact);
      } else {  // the received products stay; only the slot bits change
        plan_survivors(s, gen_row, cs, sn, exact);
        recv_slot_bits(rv, nrecv, exact);
        o = merge_products(s, gen_row, cs, sn, 1e-12, want_hist, eps, nrecv, rk, rv, next_row, exact);
      }
      glob[0] = o.count_eps;
      glob[1] = o.n_ge_theta;
      glob[2] = s.has_identity ? 1 : 0;
      if (o.has_glob)
        std::copy(o.glob, o.glob + 3, glob);
      else
        red.sum(glob, 3);
      if (spec_failed) *spec_failed = true;
    }
  }
  if (eps > 0.0 || glob[0] > max_terms) {  // compress_partitioned always runs with a cut
    const ull gk[2] = {glob[0], glob[2]};
    CompressResult r =
        compress_store(s, eps, max_terms, true, o.count_eps, cs_out != nullptr, &red, gk, floor_cut);
    if (cs_out) {
      cs_out->dropped_terms += r.dropped_terms;
      cs_out->dropped_weight += r.dropped_weight;
    }
  }
  check_wait_timeout();  // (the compress select ended with a synchronize)
}

void parallel_reserve(DeviceStore& s, size_t terms) { p2p_prepare(std::max(terms, s.M), 2 * (size_t)s.B); }

void parallel_compress_store(DeviceStore& s, double eps, size_t max_terms, iqcc_compress_stats* cs) {
  comm();
  NcclReducer red;
  CompressResult r = compress_store(s, eps, max_terms, false, 0, cs != nullptr, &red);
  if (cs) {
    cs->dropped_terms += r.dropped_terms;
    cs->dropped_weight += r.dropped_weight;
  }
}

double parallel_expect_store(DeviceStore& s, const double* factors) {
  Comm& c = comm();
  const double local = expect_store(s, factors);
  cudaStream_t st = stream();
  double* d = workspace().partials.as<double>(c.world + 1);
  IQCC_CUDA(cudaMemcpyAsync(d + c.world, &local, sizeof(double), cudaMemcpyHostToDevice, st));
  IQCC_NCCL(ncclAllGather(d + c.world, d, 1, ncclFloat64, c.comm, st));
  std::vector<double> parts(c.world);
  d2h_small(parts.data(), d, c.world * sizeof(double), st);
  host_sync(st);
  double e = 0.0;
  for (double v : parts) e += v;  // worker order (reduce_scalar)
  return e;
}

/// Allgather of n doubles per rank; returns [world][n] in rank order.
static std::vector<double> allgather_doubles(const double* local, size_t n) {
  Comm& c = comm();
  cudaStream_t st = stream();
  double* d = workspace().partials.as<double>((c.world + 1) * std::max<size_t>(n, 1));
  IQCC_CUDA(cudaMemcpyAsync(d + c.world * n, local, n * sizeof(double), cudaMemcpyHostToDevice, st));
  IQCC_NCCL(ncclAllGather(d + c.world * n, d, n, ncclFloat64, c.comm, st));
  std::vector<double> parts(c.world * n);
  d2h_small(parts.data(), d, parts.size() * sizeof(double), st);
  host_sync(st);
  return parts;
}

double parallel_qmf_grad_store(DeviceStore& s, const double* factors, const double* derivs, double* grad) {
  Comm& c = comm();
  const size_t n2 = 2 * (size_t)s.n_qubits;
  std::vector<double> local(n2 + 1, 0.0);
  if (s.logical) local[n2] = qmf_grad_store(s, factors, derivs, local.data());
  const auto parts = allgather_doubles(local.data(), n2 + 1);
  for (size_t k = 0; k <= n2; ++k) {
    double v = 0.0;
    for (int w = 0; w < c.world; ++w) v += parts[w * (n2 + 1) + k];  // rank order (reduce_scalar)
    if (k < n2) grad[k] = v;
    else local[n2] = v;
  }
  return local[n2];
}

void parallel_gradients_store(DeviceStore& s, const double* factors, const uint64_t* cands, size_t K,
                              bool flip_only, double* g) {
  Comm& c = comm();
  if (K == 0) return;
  std::vector<double> local(K, 0.0);
  if (s.logical) gradients_store(s, factors, cands, K, flip_only, local.data());
  const auto parts = allgather_doubles(local.data(), K);
  for (size_t k = 0; k < K; ++k) {
    double v = 0.0;
    for (int w = 0; w < c.world; ++w) v += parts[w * K + k];
    g[k] = v;
  }
}

size_t parallel_sum(size_t v) {
  ull a[1] = {(ull)v};
  NcclReducer red;
  red.sum(a, 1);
  return (size_t)a[0];
}

size_t parallel_size(DeviceStore& s) {
  ull v[1] = {(ull)s.logical};
  NcclReducer red;
  red.sum(v, 1);
  return (size_t)v[0];
}

/// Partitioned build_poly_kernels (iqcc/optimizer.hpp:371-422): each rank's
/// h_kernel over its shard, allgathered and combined element by element in
/// worker order from 0.0 (reduce_scalar, partition.hpp:233-237); the
/// tau-independent n_kernel comes from the expansion alone.
void parallel_poly_kernels_store(DeviceStore& s, const double* factors, bool poles, const uint64_t* words,
                                 size_t t, double* hk, double* nk) {
  Comm& c = comm();
  const size_t n = 2 * t * t;
  if (n == 0) return;
  std::vector<double> local(n);
  poly_kernels_store(s, factors, poles, words, t, local.data(), nk, true);
  cudaStream_t st = stream();
  double* d = workspace().partials.as<double>((c.world + 1) * n);
  IQCC_CUDA(cudaMemcpyAsync(d + c.world * n, local.data(), n * sizeof(double), cudaMemcpyHostToDevice, st));
  IQCC_NCCL(ncclAllGather(d + c.world * n, d, n, ncclFloat64, c.comm, st));
  std::vector<double> parts(c.world * n);
  d2h_small(parts.data(), d, parts.size() * sizeof(double), st);
  host_sync(st);
  for (size_t i = 0; i < n; ++i) {
    double v = 0.0;
    for (int w = 0; w < c.world; ++w) v += parts[w * n + i];
    hk[i] = v;
  }
}

}  // namespace iqcc_b200
