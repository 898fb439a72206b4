// psum.cu — the reference's PartitionedSum (iqcc/partition.hpp) held on the
// device: 2^m shards (one per partition id), each a DeviceStore on the GPU
// of its owning worker, driven from ONE API call on the calling host thread.
//
// Execution model.  Every shard gets a host worker thread with its own
// engine context (device, stream, hot-path scratch; capi.cu), created when
// the partitioned sum is built and kept until it is destroyed — the
// reference's run_tasks(kThreaded) (partition.hpp:190-204) with persistent
// threads.  An API call hands every shard thread the same task; collectives
// between shards (compress_partitioned's histograms, counts and tie words)
// are host-side reductions in shard order behind an abortable barrier, so
// the existing device select (compress_store with a Reducer) runs unchanged.
// Shards on one device run concurrently on separate streams; shards on
// different devices exchange products over NVLink (cudaMemcpyPeerAsync).
//
// parallel_dress (partition.hpp:398-452): with mask = the entangler's key on
// the partition bits, survivors stay and products of partition p go to
// p ^ mask.  mask == 0: a local dressing step per shard (no exchange).
// Otherwise every shard plans its products (the sortless trie rank of
// dress.cu), materializes them sorted (key ^ P, +-fl(c sin)), and after a
// barrier merges its survivors with the partner's sorted products — the
// reference's per-destination kway_merge_combine with drop 1e-12.  Then
// compress_partitioned (:325-396): per-shard eps cut plus a global
// max_terms selection, canonical tie-break across shards.  MessageLog
// records are the reference's (:415-424): one per source partition with
// products when mask != 0, bytes = terms * (16 + 16 * blocks).
//
// Worker-order reductions (reduce_scalar, :233-237): parallel_expect sums
// each worker's shards in partition order, then the workers in id order;
// the partitioned QMF gradient and DIS gradients reduce their vectors the
// same way, element by element.
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <exception>
#include <functional>
#include <limits>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/iqcc_b200.h"
#include "engine.cuh"

namespace iqcc_b200 {
namespace {

/// Thrown by a barrier another shard aborted (a secondary failure).
struct ShardAborted : std::runtime_error {
  ShardAborted() : std::runtime_error("partitioned sum: another shard failed") {}
};

/// Generation barrier over the shard threads; abort() releases every waiter
/// with an exception so one failing shard cannot hang the others.
class Barrier {
 public:
  void reset(size_t n) {
    std::lock_guard<std::mutex> lk(mu_);
    n_ = n;
    count_ = 0;
    aborted_ = false;
  }
  void wait() {
    std::unique_lock<std::mutex> lk(mu_);
    if (aborted_) throw ShardAborted();
    const uint64_t g = gen_;
    if (++count_ == n_) {
      count_ = 0;
      ++gen_;
      cv_.notify_all();
      return;
    }
    cv_.wait(lk, [&] { return gen_ != g || aborted_; });
    if (gen_ == g) throw ShardAborted();
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu_);
    aborted_ = true;
    cv_.notify_all();
  }

 private:
  std::mutex mu_;
  std::condition_variable cv_;
  size_t n_ = 1, count_ = 0;
  uint64_t gen_ = 0;
  bool aborted_ = false;
};

struct Shard {
  int device = 0;
  Ctx* ctx = nullptr;  // created, bound and freed by the shard's own thread
  DeviceStore s;
  DevBuf xk, xv;       // this step's sorted products, read by the partner
  DevBuf rk, rv;       // the partner's products copied from another device
  size_t A = 0;        // products exported this step (MessageLog terms)
  DressOutcome o;
  CompressResult cr;
  double e = 0.0;                  // scalar partial (energy)
  std::vector<double> vec;         // vector partial (gradients)
  DeviceStore scratch;             // gather accumulator (shard 0)
};

struct SumSlot {
  std::vector<ull> v;
};

}  // namespace

struct PSum {
  size_t n_qubits = 0, m = 0, n_workers = 1;
  std::vector<size_t> bits, owner;  // owner: partition -> worker
  std::vector<int> devices;         // worker -> device
  std::vector<std::unique_ptr<Shard>> shards;
  // worker pool
  std::vector<std::thread> threads;
  std::mutex mu;
  std::condition_variable cv, done_cv;
  uint64_t gen = 0;
  size_t done = 0;
  bool stop = false;
  std::function<void(size_t)> task;
  std::vector<std::exception_ptr> err;
  Barrier bar;
  // host-side collective slots, one per shard
  std::vector<SumSlot> slots;
  std::vector<std::vector<ull>> key_slots;
  // distribute staging: per device, the full sum uploaded once
  std::vector<DeviceStore*> staging;

  size_t n_parts() const { return shards.size(); }
  int device_of_worker(size_t w) const { return devices[w]; }

  void worker_main(size_t p) {
    uint64_t seen = 0;
    for (;;) {
      std::function<void(size_t)> t;
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return stop || gen != seen; });
        if (stop) break;
        seen = gen;
        t = task;
      }
      try {
        t(p);
      } catch (...) {
        err[p] = std::current_exception();
        bar.abort();
      }
      std::lock_guard<std::mutex> lk(mu);
      if (++done == n_parts()) done_cv.notify_all();
    }
  }

  /// Runs fn(p) on every shard's thread and waits; rethrows the first
  /// failure in shard order.
  void run(std::function<void(size_t)> fn) {
    {
      std::lock_guard<std::mutex> lk(mu);
      task = std::move(fn);
      done = 0;
      err.assign(n_parts(), nullptr);
      bar.reset(n_parts());
      ++gen;
    }
    cv.notify_all();
    std::unique_lock<std::mutex> lk(mu);
    done_cv.wait(lk, [&] { return done == n_parts(); });
    // the first primary failure in shard order (not the aborts it caused)
    std::exception_ptr first;
    for (auto& e : err) {
      if (!e) continue;
      if (!first) first = e;
      try {
        std::rethrow_exception(e);
      } catch (const ShardAborted&) {
        continue;
      } catch (...) {
        std::rethrow_exception(e);
      }
    }
    if (first) std::rethrow_exception(first);
  }

  void start() {
    err.assign(n_parts(), nullptr);
    slots.assign(n_parts(), {});
    key_slots.assign(n_parts(), {});
    for (size_t p = 0; p < n_parts(); ++p) threads.emplace_back([this, p] { worker_main(p); });
    // every thread creates and binds its context on its shard's device
    run([this](size_t p) {
      Shard& sh = *shards[p];
      sh.ctx = ctx_new(sh.device);
      ctx_bind(sh.ctx);
    });
  }

  ~PSum() {
    if (!threads.empty()) {
      try {
        run([this](size_t p) {
          Shard& sh = *shards[p];
          if (!sh.ctx) return;
          ctx_bind(sh.ctx);
          sh.s.free_all();
          sh.scratch.free_all();
          for (DevBuf* b : {&sh.xk, &sh.xv, &sh.rk, &sh.rv}) b->release();
          ctx_free(sh.ctx);
          sh.ctx = nullptr;
        });
      } catch (...) {
      }
      {
        std::lock_guard<std::mutex> lk(mu);
        stop = true;
      }
      cv.notify_all();
      for (auto& t : threads) t.join();
    }
  }
};

namespace {

/// compress_partitioned's collectives across the shard threads: sums in
/// shard order (deterministic), tie words concatenated in shard order.
struct ShardReducer : Reducer {
  PSum* ps;
  size_t rank;
  ShardReducer(PSum* p, size_t r) : ps(p), rank(r) {}
  void sum(ull* vals, size_t n) override {
    ps->slots[rank].v.assign(vals, vals + n);
    ps->bar.wait();
    for (size_t i = 0; i < n; ++i) {
      ull a = 0;
      for (size_t r = 0; r < ps->n_parts(); ++r) a += ps->slots[r].v[i];
      vals[i] = a;
    }
    ps->bar.wait();
  }
  void sum_device(ull* d, size_t n) override {
    std::vector<ull> h(n);
    IQCC_CUDA(cudaMemcpyAsync(h.data(), d, n * sizeof(ull), cudaMemcpyDeviceToHost, stream()));
    IQCC_CUDA(cudaStreamSynchronize(stream()));
    sum(h.data(), n);
    IQCC_CUDA(cudaMemcpyAsync(d, h.data(), n * sizeof(ull), cudaMemcpyHostToDevice, stream()));
    IQCC_CUDA(cudaStreamSynchronize(stream()));
  }
  std::vector<ull> gather_keys(const std::vector<ull>& mine, size_t W, size_t* mine_off) override {
    (void)W;
    ps->key_slots[rank] = mine;
    ps->bar.wait();
    std::vector<ull> all;
    size_t off = 0;
    for (size_t r = 0; r < ps->n_parts(); ++r) {
      if (r == rank) off = all.size() / std::max<size_t>(W, 1);
      all.insert(all.end(), ps->key_slots[r].begin(), ps->key_slots[r].end());
    }
    *mine_off = off;
    ps->bar.wait();
    return all;
  }
};

uint32_t ref_blocks_n(size_t n) { return n == 0 ? 1 : (uint32_t)((n + 63) / 64); }

/// Device-width row of a reference-layout row.
std::vector<uint64_t> widen(const uint64_t* row, uint32_t Bref, uint32_t B) {
  std::vector<uint64_t> r(2 * B, 0);
  for (uint32_t w = 0; w < Bref; ++w) {
    r[w] = row[w];
    r[B + w] = row[Bref + w];
  }
  return r;
}

/// partition_key (partition.hpp:40-42) of a reference-layout row.
size_t key_of(const uint64_t* row, uint32_t Bref, size_t n, const std::vector<size_t>& bits) {
  size_t key = 0;
  for (size_t b = 0; b < bits.size(); ++b) {
    const size_t p = bits[b], q = p < n ? p : p - n;
    const uint64_t w = row[(p < n ? 0 : Bref) + q / 64];
    key |= (size_t)((w >> (q % 64)) & 1u) << b;
  }
  return key;
}

void validate_map(size_t n_qubits, size_t m, const size_t* bits, const size_t* owner, size_t n_workers) {
  if (m > 16) throw std::invalid_argument("partition: at most 16 partition bits");
  if (n_workers < 1) throw std::invalid_argument("make_partition_map: no workers");
  for (size_t b = 0; b < m; ++b)
    if (bits[b] >= 2 * n_qubits) throw std::invalid_argument("PartitionMap: bit position out of range");
  for (size_t p = 0; p < ((size_t)1 << m); ++p)
    if (owner[p] >= n_workers) throw std::invalid_argument("PartitionMap: owner out of range");
}

std::unique_ptr<PSum> make_psum(size_t n_qubits, size_t m, const size_t* bits, const size_t* owner,
                                size_t n_workers, const int* devices) {
  validate_map(n_qubits, m, bits, owner, n_workers);
  int ndev = 0;
  IQCC_CUDA(cudaGetDeviceCount(&ndev));
  auto ps = std::make_unique<PSum>();
  ps->n_qubits = n_qubits;
  ps->m = m;
  ps->n_workers = n_workers;
  ps->bits.assign(bits, bits + m);
  ps->owner.assign(owner, owner + ((size_t)1 << m));
  ps->devices.resize(n_workers);
  for (size_t w = 0; w < n_workers; ++w) {
    ps->devices[w] = devices ? devices[w] : (int)(w % (size_t)std::max(ndev, 1));
    if (ps->devices[w] < 0 || ps->devices[w] >= ndev)
      throw std::invalid_argument("partitioned sum: device id out of range");
  }
  for (size_t p = 0; p < ((size_t)1 << m); ++p) {
    auto sh = std::make_unique<Shard>();
    sh->device = ps->devices[ps->owner[p]];
    ps->shards.push_back(std::move(sh));
  }
  ps->start();
  return ps;
}

/// Owner table of restrict_store that keeps exactly partition p.
std::vector<size_t> identity_owner(size_t m) {
  std::vector<size_t> o((size_t)1 << m);
  for (size_t p = 0; p < o.size(); ++p) o[p] = p;
  return o;
}

/// One parallel_dress step on shard p (its own thread).
void dress_shard(PSum& P, size_t p, const std::vector<uint64_t>& row, double cs, double sn, double eps,
                 size_t max_terms, size_t mask, bool want_stats) {
  Shard& sh = *P.shards[p];
  DeviceStore& s = sh.s;
  const bool want_hist = eps > 0.0 || max_terms != SIZE_MAX;
  // exact output slots: terms under eps cannot survive compress_partitioned
  // (off when drop statistics are requested: they count every dropped term)
  const double theta = want_hist && eps > 0.0 && !want_stats ? eps : 0.0;
  const bool exch = mask != 0 && sn != 0.0;
  sh.A = 0;
  sh.cr = CompressResult{};
  if (!exch) {
    sh.o = dress_step(s, row.data(), cs, sn, 1e-12, want_hist, eps, nullptr, theta);
    sh.A = sn != 0.0 ? sh.o.n_anticommuting : 0;
  } else {
    cudaStream_t st = stream();
    const size_t W = 2 * (size_t)s.B;
    const long long* a_dev = plan_products_async(s, row.data(), cs, sn, theta);
    size_t A = 0;
    if (a_dev) {
      long long* hp = static_cast<long long*>(host_pinned(sizeof(long long)));
      IQCC_CUDA(cudaMemcpyAsync(hp, a_dev, sizeof(long long), cudaMemcpyDeviceToHost, st));
      IQCC_CUDA(cudaStreamSynchronize(st));
      A = (size_t)*hp;
    }
    plan_set_products(A);
    ull* xk = sh.xk.as<ull>(std::max<size_t>(A, 1) * W);
    double* xv = sh.xv.as<double>(std::max<size_t>(A, 1));
    materialize_products(s, row.data(), sn, xk, xv);
    sh.A = A;
    IQCC_CUDA(cudaStreamSynchronize(st));
    P.bar.wait();  // every shard's products are ready
    const Shard& so = *P.shards[p ^ mask];
    const size_t nQ = so.A;
    const ull* qk = static_cast<const ull*>(so.xk.p);
    const double* qv = static_cast<const double*>(so.xv.p);
    if (so.device != sh.device && nQ > 0) {  // NVLink peer copy into this device
      ull* rk = sh.rk.as<ull>(nQ * W);
      double* rv = sh.rv.as<double>(nQ);
      KernelScope ks("exchange");
      IQCC_CUDA(cudaMemcpyPeerAsync(rk, sh.device, qk, so.device, nQ * W * sizeof(ull), st));
      IQCC_CUDA(cudaMemcpyPeerAsync(rv, sh.device, qv, so.device, nQ * sizeof(double), st));
      qk = rk;
      qv = rv;
    }
    recv_slot_bits(qv, nQ, theta);
    sh.o = merge_products(s, row.data(), cs, sn, 1e-12, want_hist, eps, nQ, qk, qv, nullptr, theta);
    P.bar.wait();  // the partner is done reading this shard's products
  }
  if (!want_hist) return;
  ShardReducer red(&P, p);
  ull glob[3] = {(ull)sh.o.count_eps, 0, (ull)(s.has_identity ? 1 : 0)};
  red.sum(glob, 3);
  if (eps > 0.0 || glob[0] > max_terms) {  // compress_partitioned
    const ull gk[2] = {glob[0], glob[2]};
    sh.cr = compress_store(s, eps, max_terms, true, sh.o.count_eps, want_stats, &red, gk, 0.0);
  }
}

/// Worker-order reduction of per-shard values (reduce_scalar over workers,
/// each worker's shards in partition order, partition.hpp:241-254).
double worker_order_sum(const PSum& P, const std::function<double(size_t)>& val) {
  std::vector<double> local(P.n_workers, 0.0);
  for (size_t w = 0; w < P.n_workers; ++w)
    for (size_t p = 0; p < P.n_parts(); ++p)
      if (P.owner[p] == w) local[w] += val(p);
  double s = 0.0;
  for (double v : local) s += v;
  return s;
}

}  // namespace

// ------------------------------------------------------------------ entry
PSum* psum_distribute(size_t n_qubits, const uint64_t* rows, const double* coeff, size_t M,
                                      size_t m, const size_t* bits, const size_t* owner, size_t n_workers,
                                      const int* devices) {
  auto ps = make_psum(n_qubits, m, bits, owner, n_workers, devices);
  PSum& P = *ps;
  const auto ident = identity_owner(m);
  // the lowest shard on each device uploads the whole sum once; every shard
  // on that device keeps its own partition of it (distribute, :208-220)
  P.staging.assign(P.n_parts(), nullptr);
  std::vector<size_t> uploader(P.n_parts());
  for (size_t p = 0; p < P.n_parts(); ++p) {
    uploader[p] = p;
    for (size_t q = 0; q < p; ++q)
      if (P.shards[q]->device == P.shards[p]->device) {
        uploader[p] = q;
        break;
      }
  }
  P.run([&](size_t p) {
    Shard& sh = *P.shards[p];
    if (uploader[p] == p) {
      sh.scratch = DeviceStore{};
      store_upload(sh.scratch, n_qubits, rows, coeff, M, true);
      IQCC_CUDA(cudaStreamSynchronize(stream()));
    }
    P.bar.wait();
    store_clone(P.shards[uploader[p]]->scratch, sh.s);
    restrict_store(sh.s, P.m, P.bits.data(), ident.data(), (int)p);
    IQCC_CUDA(cudaStreamSynchronize(stream()));
    P.bar.wait();
    if (uploader[p] == p) sh.scratch.free_all();
  });
  return ps.release();
}

PSum* psum_from_shards(size_t n_qubits, size_t m, const size_t* bits, const size_t* owner,
                                       size_t n_workers, const int* devices, const uint64_t* const* rows,
                                       const double* const* coeffs, const size_t* sizes) {
  auto ps = make_psum(n_qubits, m, bits, owner, n_workers, devices);
  PSum& P = *ps;
  const auto ident = identity_owner(m);
  P.run([&](size_t p) {
    Shard& sh = *P.shards[p];
    store_upload(sh.s, n_qubits, rows[p], coeffs[p], sizes[p], true);
    // PartitionedSum::validate (:162-172): every term in its own shard
    const size_t before = sh.s.logical;
    restrict_store(sh.s, P.m, P.bits.data(), ident.data(), (int)p);
    if (sh.s.logical != before) throw std::runtime_error("term in wrong shard");
  });
  return ps.release();
}

void psum_destroy(PSum* ps) { delete ps; }

size_t psum_parts(const PSum& P) { return P.n_parts(); }

void psum_sizes(PSum& P, size_t* sizes) {
  for (size_t p = 0; p < P.n_parts(); ++p) sizes[p] = P.shards[p]->s.logical;
}

void psum_owner(const PSum& P, size_t* owner) { std::copy(P.owner.begin(), P.owner.end(), owner); }

size_t psum_download_shard(PSum& P, size_t p, uint64_t* rows, double* coeff, size_t cap) {
  if (p >= P.n_parts()) throw std::invalid_argument("partitioned sum: shard index out of range");
  size_t n = 0;
  P.run([&](size_t q) {
    if (q == p) n = store_download(P.shards[q]->s, rows, coeff, cap, true);
  });
  return n;
}

/// gather (partition.hpp:222-230): the shards are disjoint, so the sorted
/// union is a chain of two-way merges (no coefficient combines); shard 0's
/// thread merges every other shard into its accumulator on its device.
size_t psum_gather(PSum& P, uint64_t* rows, double* coeff, size_t cap) {
  size_t n = 0;
  P.run([&](size_t p) {
    Shard& sh = *P.shards[p];
    store_materialize(sh.s);  // plain sorted live terms (no filter, no dead slots)
    IQCC_CUDA(cudaStreamSynchronize(stream()));
    P.bar.wait();
    if (p == 0) {
      DeviceStore& acc = sh.scratch;
      acc = DeviceStore{};
      store_clone(sh.s, acc);
      const std::vector<uint64_t> zero(2 * acc.B, 0);  // commutes with every word
      const size_t W = 2 * (size_t)acc.B;
      for (size_t q = 1; q < P.n_parts(); ++q) {
        Shard& so = *P.shards[q];
        const size_t nQ = so.s.logical;
        if (nQ == 0) continue;
        const ull* qk = so.s.keys();
        const double* qv = so.s.coef();
        if (so.device != sh.device) {
          ull* rk = sh.rk.as<ull>(nQ * W);
          double* rv = sh.rv.as<double>(nQ);
          IQCC_CUDA(cudaMemcpyPeerAsync(rk, sh.device, qk, so.device, nQ * W * sizeof(ull), stream()));
          IQCC_CUDA(cudaMemcpyPeerAsync(rv, sh.device, qv, so.device, nQ * sizeof(double), stream()));
          qk = rk;
          qv = rv;
        }
        plan_survivors(acc, zero.data(), 1.0, 0.0, 0.0);
        recv_slot_bits(qv, nQ, 0.0);
        merge_products(acc, zero.data(), 1.0, 0.0, 0.0, false, 0.0, nQ, qk, qv);
      }
      n = store_download(acc, rows, coeff, cap, true);
      acc.free_all();
    }
  });
  return n;
}

void psum_dress(PSum& P, const uint64_t* gen, double cs, double sn, double eps, size_t max_terms,
                iqcc_message_record* log, size_t log_cap, size_t* n_log, iqcc_compress_stats* cstats,
                size_t* mask_out) {
  const uint32_t Bref = ref_blocks_n(P.n_qubits);
  bool id = true;
  for (uint32_t w = 0; w < 2 * Bref; ++w) id = id && gen[w] == 0;
  if (id) throw std::invalid_argument("parallel_dress: identity generator");
  if (max_terms < 1) throw std::invalid_argument("compress_partitioned: max_terms < 1");
  const size_t mask = key_of(gen, Bref, P.n_qubits, P.bits);
  const uint32_t B = P.shards.empty() ? 1 : (Bref == 3 ? 4 : Bref);
  const auto row = widen(gen, Bref, B);
  P.run([&](size_t p) { dress_shard(P, p, row, cs, sn, eps, max_terms, mask, cstats != nullptr); });
  size_t nl = 0;
  if (mask != 0)
    for (size_t p = 0; p < P.n_parts(); ++p) {
      const size_t a = P.shards[p]->A;
      if (a == 0) continue;
      if (log && nl < log_cap) log[nl] = iqcc_message_record{p, p ^ mask, a, a * (16 + 2 * (size_t)Bref * 8)};
      ++nl;
    }
  if (n_log) *n_log = nl;
  if (cstats)
    for (size_t p = 0; p < P.n_parts(); ++p) {
      cstats->dropped_terms += P.shards[p]->cr.dropped_terms;
      cstats->dropped_weight += P.shards[p]->cr.dropped_weight;
    }
  if (mask_out) *mask_out = mask;
}

double psum_expect(PSum& P, const double* factors) {
  P.run([&](size_t p) { P.shards[p]->e = expect_store(P.shards[p]->s, factors); });
  return worker_order_sum(P, [&](size_t p) { return P.shards[p]->e; });
}

double psum_qmf_energy_gradient(PSum& P, const double* factors, const double* derivs, double* grad) {
  const size_t n2 = 2 * P.n_qubits;
  P.run([&](size_t p) {
    Shard& sh = *P.shards[p];
    sh.vec.assign(n2, 0.0);
    sh.e = sh.s.logical ? qmf_grad_store(sh.s, factors, derivs, sh.vec.data()) : 0.0;
  });
  for (size_t k = 0; k < n2; ++k) grad[k] = worker_order_sum(P, [&](size_t p) { return P.shards[p]->vec[k]; });
  return worker_order_sum(P, [&](size_t p) { return P.shards[p]->e; });
}

void psum_gradients(PSum& P, const double* factors, const uint64_t* cands, size_t K, bool flip_only, double* g) {
  const uint32_t Bref = ref_blocks_n(P.n_qubits);
  const uint32_t B = Bref == 3 ? 4 : Bref;
  std::vector<uint64_t> wide(std::max<size_t>(K, 1) * 2 * B, 0);
  for (size_t k = 0; k < K; ++k) {
    const auto r = widen(cands + k * 2 * Bref, Bref, B);
    std::copy(r.begin(), r.end(), wide.begin() + k * 2 * B);
  }
  P.run([&](size_t p) {
    Shard& sh = *P.shards[p];
    sh.vec.assign(K, 0.0);
    if (sh.s.logical && K) gradients_store(sh.s, factors, wide.data(), K, flip_only, sh.vec.data());
  });
  for (size_t k = 0; k < K; ++k) g[k] = worker_order_sum(P, [&](size_t p) { return P.shards[p]->vec[k]; });
}

/// rebalance (partition.hpp:457-494) on the shard sizes, then shard
/// migration: a shard whose new owner runs on another device moves there
/// (peer copy on its own thread, which rebinds to a fresh context).
void psum_rebalance(PSum& P, double threshold, size_t* owner_out) {
  if (!(threshold > 1.0)) throw std::invalid_argument("rebalance: threshold must exceed 1");
  std::vector<size_t> sizes(P.n_parts());
  psum_sizes(P, sizes.data());
  std::vector<size_t> own = P.owner;
  for (;;) {
    std::vector<size_t> l(P.n_workers, 0);
    for (size_t p = 0; p < P.n_parts(); ++p) l[own[p]] += sizes[p];
    auto mx = std::max_element(l.begin(), l.end());
    auto mn = std::min_element(l.begin(), l.end());
    const double ratio = *mn == 0 ? std::numeric_limits<double>::infinity() : (double)*mx / (double)*mn;
    if (*mx == 0 || ratio <= threshold) break;
    const size_t donor = mx - l.begin(), receiver = mn - l.begin();
    size_t best = SIZE_MAX, best_size = 0;
    for (size_t p = 0; p < P.n_parts(); ++p) {
      if (own[p] != donor || sizes[p] == 0) continue;
      if (*mn + sizes[p] < *mx && sizes[p] > best_size) {
        best = p;
        best_size = sizes[p];
      }
    }
    if (best == SIZE_MAX) break;
    own[best] = receiver;
  }
  P.owner = own;
  P.run([&](size_t p) {
    Shard& sh = *P.shards[p];
    const int to = P.devices[P.owner[p]];
    if (to == sh.device) return;
    const int from = sh.device;
    Ctx* nc = ctx_new(to);
    Ctx* oc = ctx_bind(nc);
    DeviceStore dst;
    dst.n_qubits = sh.s.n_qubits;
    dst.B = sh.s.B;
    dst.ensure(sh.s.M);
    if (sh.s.M) {
      IQCC_CUDA(cudaMemcpyPeerAsync(dst.keys(), to, sh.s.keys(), from, sh.s.M * 2 * sh.s.B * sizeof(ull), stream()));
      IQCC_CUDA(cudaMemcpyPeerAsync(dst.coef(), to, sh.s.coef(), from, sh.s.M * sizeof(double), stream()));
    }
    IQCC_CUDA(cudaStreamSynchronize(stream()));
    dst.M = sh.s.M;
    dst.filt = sh.s.filt;
    dst.logical = sh.s.logical;
    dst.has_identity = sh.s.has_identity;
    ctx_bind(oc);  // release the old device's buffers under their own context
    sh.s.free_all();
    for (DevBuf* b : {&sh.xk, &sh.xv, &sh.rk, &sh.rv}) b->release();
    sh.scratch.free_all();
    ctx_free(oc);
    ctx_bind(nc);
    sh.ctx = nc;
    sh.s = dst;
    sh.device = to;
  });
  if (owner_out) std::copy(P.owner.begin(), P.owner.end(), owner_out);
}

}  // namespace iqcc_b200
