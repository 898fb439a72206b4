// iqcc_gpu.hpp — drop-in C++ shim: the reference's hot-path API
// (namespace iqcc, /root/reference/proj/include/iqcc/*.hpp) re-exposed as
// iqcc::gpu::* with identical signatures, executed by the B200 engine
// through the C-ABI in iqcc_b200.h.
//
// A reference maintainer switches a call site by qualifying it:
//     iqcc::PauliSum d = iqcc::gpu::dress_single(h, op);        // was iqcc::dress_single
// Exceptions match the reference: std::invalid_argument for precondition
// violations (EINVAL), std::runtime_error otherwise.  Include after the
// reference headers are on the include path (-I <ref>/proj/include) and link
// paper_2603_08883_b200/libiqcc_b200.so.
//
// Host-side numerics stay on the host exactly as in the reference:
// std::cos/std::sin of amplitudes (iqcc/dressing.hpp:203) and the QMF factor
// tables via iqcc::detail::qmf_factor (iqcc/qmf.hpp:56-61), so device results
// are bit-identical.  Sums cross the boundary zero-copy from PauliSum's
// contiguous storage (iqcc/pauli.hpp:373-377).
#pragma once
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <limits>
#include <memory>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "iqcc/dis.hpp"
#include "iqcc/dressing.hpp"
#include "iqcc/optimizer.hpp"
#include "iqcc/partition.hpp"
#include "iqcc/pauli.hpp"
#include "iqcc/qmf.hpp"
#include "iqcc_b200.h"

namespace iqcc::gpu {

namespace detail {

inline void check(int rc) {
  if (rc == IQCC_OK) return;
  const std::string msg = iqcc_gpu_last_error();
  if (rc == IQCC_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

/// Engine context of the calling thread (iqcc_gpu_init binds one per host
/// thread and is idempotent).
inline void ensure_engine(int device = 0) {
  static thread_local const int rc = iqcc_gpu_init(device);
  check(rc);
}

/// Owning device handle.
class Handle {
 public:
  explicit Handle(iqcc_gpu_sum* h = nullptr) : h_(h) {}
  Handle(const Handle&) = delete;
  Handle& operator=(const Handle&) = delete;
  Handle(Handle&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
  ~Handle() {
    if (h_) iqcc_gpu_sum_destroy(h_);
  }
  iqcc_gpu_sum* get() const { return h_; }

 private:
  iqcc_gpu_sum* h_;
};

inline Handle upload(const PauliSum& h) {
  ensure_engine();
  iqcc_gpu_sum* out = nullptr;
  const uint64_t* rows = h.empty() ? nullptr : h.word(0).x.data();
  // PauliSum stores std::complex<double> contiguously (layout-compatible with
  // double[2]); the const accessor returns by value, so reach the storage
  // through the non-const one without modifying it.
  const double* coeff =
      h.empty() ? nullptr : reinterpret_cast<const double*>(&const_cast<PauliSum&>(h).coeff(0));
  check(iqcc_gpu_sum_create(h.n_qubits(), rows, coeff, h.size(), &out));
  return Handle(out);
}

inline PauliSum download(const Handle& d, std::size_t n_qubits) {
  std::size_t n = 0;
  check(iqcc_gpu_sum_size(d.get(), &n));
  const std::size_t B = blocks_for(n_qubits);
  std::vector<uint64_t> rows(std::max<std::size_t>(n, 1) * 2 * B);
  std::vector<double> coeff(std::max<std::size_t>(n, 1) * 2);
  std::size_t got = 0;
  check(iqcc_gpu_sum_download(d.get(), rows.data(), coeff.data(), n, &got));
  PauliSum out(n_qubits);
  out.reserve(got);
  for (std::size_t i = 0; i < got; ++i)
    out.append(PauliView{{rows.data() + i * 2 * B, B}, {rows.data() + i * 2 * B + B, B}},
               Complex(coeff[2 * i], coeff[2 * i + 1]));
  return out;
}

inline PauliSum from_rows(std::size_t n_qubits, const std::vector<uint64_t>& rows,
                          const std::vector<double>& coeff, std::size_t got) {
  const std::size_t B = blocks_for(n_qubits);
  PauliSum out(n_qubits);
  out.reserve(got);
  for (std::size_t i = 0; i < got; ++i)
    out.append(PauliView{{rows.data() + i * 2 * B, B}, {rows.data() + i * 2 * B + B, B}},
               Complex(coeff[2 * i], coeff[2 * i + 1]));
  return out;
}

inline std::vector<double> factor_table(const QmfState& omega) {
  std::vector<double> t(3 * omega.n_qubits());
  for (std::size_t j = 0; j < omega.n_qubits(); ++j) {
    t[3 * j + 0] = iqcc::detail::qmf_factor(omega, j, true, false);   // X
    t[3 * j + 1] = iqcc::detail::qmf_factor(omega, j, false, true);   // Z
    t[3 * j + 2] = iqcc::detail::qmf_factor(omega, j, true, true);    // Y
  }
  return t;
}

inline std::vector<double> deriv_table(const QmfState& omega) {
  std::vector<double> t(6 * omega.n_qubits());
  for (std::size_t j = 0; j < omega.n_qubits(); ++j) {  // iqcc/qmf.hpp:130-143
    const double st = std::sin(omega.theta[j]), ct = std::cos(omega.theta[j]);
    const double sp = std::sin(omega.phi[j]), cp = std::cos(omega.phi[j]);
    const double v[6] = {ct * cp, -st * sp, -st, 0.0, ct * sp, st * cp};
    std::copy(v, v + 6, t.begin() + 6 * j);
  }
  return t;
}

inline std::vector<uint64_t> row_of(PauliView p) {
  std::vector<uint64_t> r(p.x.begin(), p.x.end());
  r.insert(r.end(), p.z.begin(), p.z.end());
  return r;
}

}  // namespace detail

/// A PauliSum kept resident in HBM across many calls (the iQCC loop keeps H
/// on the device; only the final sum comes back).
class DeviceSum {
 public:
  explicit DeviceSum(const PauliSum& h) : n_(h.n_qubits()), d_(detail::upload(h)) {}
  std::size_t n_qubits() const { return n_; }
  std::size_t size() const {
    std::size_t n = 0;
    detail::check(iqcc_gpu_sum_size(d_.get(), &n));
    return n;
  }
  void dress(const DressOp& op, const MergeOptions& opts = {}) {
    if (op.generator.n_qubits() != n_) throw std::invalid_argument("dress_single: mismatched qubit counts");
    const auto row = detail::row_of(op.generator.view());
    detail::check(iqcc_gpu_dress(d_.get(), row.data(), std::cos(op.amplitude), std::sin(op.amplitude),
                                 opts.drop_threshold, nullptr));
  }
  void compress(double epsilon, std::size_t max_terms, CompressStats* stats = nullptr) {
    iqcc_compress_stats s{0, 0.0};
    detail::check(iqcc_gpu_compress(d_.get(), epsilon, max_terms, &s));
    if (stats) {
      stats->dropped_terms += s.dropped_terms;
      stats->dropped_weight += s.dropped_weight;
    }
  }
  void dress_sequence(const Ansatz& a, double epsilon,
                      std::size_t max_terms = std::numeric_limits<std::size_t>::max(),
                      CompressStats* stats = nullptr, const MergeOptions& opts = {}) {
    std::vector<uint64_t> gens;
    std::vector<double> c, s;
    for (std::size_t k = 0; k < a.size(); ++k) {
      if (a.entanglers[k].n_qubits() != n_) throw std::invalid_argument("dress_single: mismatched qubit counts");
      const auto row = detail::row_of(a.entanglers[k].view());
      gens.insert(gens.end(), row.begin(), row.end());
      c.push_back(std::cos(a.tau[k]));
      s.push_back(std::sin(a.tau[k]));
    }
    iqcc_compress_stats st{0, 0.0};
    detail::check(iqcc_gpu_dress_sequence(d_.get(), a.size(), gens.data(), c.data(), s.data(), epsilon,
                                          max_terms, opts.drop_threshold, stats ? &st : nullptr, nullptr));
    if (stats) {
      stats->dropped_terms += st.dropped_terms;
      stats->dropped_weight += st.dropped_weight;
    }
  }
  double expect(const QmfState& omega) {
    const auto t = detail::factor_table(omega);
    double e = 0.0;
    detail::check(iqcc_gpu_expect(d_.get(), t.data(), &e));
    return e;
  }
  /// qcc_energy / qcc_gradient (iqcc/optimizer.hpp:19-77) on device copies.
  double qcc_energy(const QmfState& omega, const Ansatz& a) const {
    std::vector<uint64_t> gens;
    std::vector<double> c, s;
    ansatz_arrays(a, gens, c, s);
    const auto t = detail::factor_table(omega);
    double e = 0.0;
    detail::check(iqcc_gpu_qcc_energy(d_.get(), a.size(), gens.data(), c.data(), s.data(), t.data(), &e));
    return e;
  }
  std::vector<double> qcc_gradient(const QmfState& omega, const Ansatz& a) const {
    std::vector<uint64_t> gens;
    std::vector<double> c, s;
    ansatz_arrays(a, gens, c, s);
    const auto t = detail::factor_table(omega);
    std::vector<double> g(a.size(), 0.0);
    detail::check(iqcc_gpu_qcc_gradient(d_.get(), a.size(), gens.data(), c.data(), s.data(), t.data(), g.data()));
    return g;
  }
  PauliSum download() const { return detail::download(d_, n_); }
  iqcc_gpu_sum* handle() const { return d_.get(); }

 private:
  void ansatz_arrays(const Ansatz& a, std::vector<uint64_t>& gens, std::vector<double>& c,
                     std::vector<double>& s) const {
    for (std::size_t k = 0; k < a.size(); ++k) {
      if (a.entanglers[k].n_qubits() != n_) throw std::invalid_argument("dress_single: mismatched qubit counts");
      const auto row = detail::row_of(a.entanglers[k].view());
      gens.insert(gens.end(), row.begin(), row.end());
      c.push_back(std::cos(a.tau[k]));
      s.push_back(std::sin(a.tau[k]));
    }
  }
  std::size_t n_;
  detail::Handle d_;
};

// ------------------------------------------------------------------ dressing
/// iqcc::dress_single (iqcc/dressing.hpp:197-220).
inline PauliSum dress_single(const PauliSum& h, const DressOp& op, const MergeOptions& opts = {}) {
  if (h.n_qubits() != op.generator.n_qubits())
    throw std::invalid_argument("dress_single: mismatched qubit counts");
  if (op.generator.is_identity()) throw std::invalid_argument("dress_single: identity generator");
  DeviceSum d(h);
  d.dress(op, opts);
  return d.download();
}

/// iqcc::sortless_dress (iqcc/dressing.hpp:228-307): the same sum; the
/// engine never sorts products, so new_stream_sorts is 0 by construction.
inline PauliSum sortless_dress(const PauliSum& h, const DressOp& op, const MergeOptions& opts = {},
                               SortlessStats* stats = nullptr) {
  if (h.n_qubits() != op.generator.n_qubits())
    throw std::invalid_argument("sortless_dress: mismatched qubit counts");
  if (op.generator.is_identity()) throw std::invalid_argument("sortless_dress: identity generator");
  const auto pos = iqcc::detail::support_positions(op.generator.view(), h.n_qubits());
  if (pos.size() > 64) throw std::runtime_error("entangler support exceeds 64 bits; not supported");
  DeviceSum d(h);
  if (stats) {
    // buckets / new-term streams counted on the device (dressing.hpp:248-268);
    // no stream is ever sorted; merge_comparisons (heap compares) stays 0
    *stats = SortlessStats{};
    const auto row = detail::row_of(op.generator.view());
    detail::check(iqcc_gpu_sortless_stats(d.handle(), row.data(), std::sin(op.amplitude), &stats->n_buckets,
                                          &stats->new_term_streams));
  }
  d.dress(op, opts);
  return d.download();
}

/// iqcc::dress_sequence (iqcc/dressing.hpp:311-324), device resident.
inline PauliSum dress_sequence(const PauliSum& h, const Ansatz& ansatz, double epsilon,
                               std::size_t max_terms = std::numeric_limits<std::size_t>::max(),
                               CompressStats* stats = nullptr, const MergeOptions& opts = {}) {
  if (max_terms < 1) throw std::invalid_argument("dress_sequence: max_terms < 1");
  DeviceSum d(h);
  d.dress_sequence(ansatz, epsilon, max_terms, stats, opts);
  return d.download();
}

/// iqcc::compress (iqcc/pauli.hpp:425-474).
inline PauliSum compress(const PauliSum& h, double epsilon, std::size_t max_terms,
                         CompressStats* stats = nullptr) {
  if (epsilon < 0) throw std::invalid_argument("compress: epsilon < 0");
  if (max_terms < 1) throw std::invalid_argument("compress: max_terms < 1");
  DeviceSum d(h);
  d.compress(epsilon, max_terms, stats);
  return d.download();
}

/// iqcc::growth_split (iqcc/dressing.hpp:41-50).
inline GrowthSplit growth_split(const PauliSum& h, PauliView p) {
  DeviceSum d(h);
  const auto row = detail::row_of(p);
  GrowthSplit g;
  detail::check(iqcc_gpu_growth_split(d.handle(), row.data(), &g.n_commuting, &g.n_anticommuting));
  return g;
}

// ------------------------------------------------------------ QMF and DIS
/// iqcc::expect_sum (iqcc/qmf.hpp:83-90).
inline double expect_sum(const QmfState& omega, const PauliSum& h) {
  if (!h.empty() && h.n_qubits() != omega.n_qubits())
    throw std::invalid_argument("expect_sum: mismatched qubit counts");
  if (h.empty()) return 0.0;
  DeviceSum d(h);
  return d.expect(omega);
}

/// iqcc::qcc_energy (iqcc/optimizer.hpp:19-25).
inline double qcc_energy(const PauliSum& h, const QmfState& omega, const Ansatz& ansatz) {
  if (h.empty()) return 0.0;
  DeviceSum d(h);
  return d.qcc_energy(omega, ansatz);
}

/// iqcc::qcc_gradient (iqcc/optimizer.hpp:54-77).
inline std::vector<double> qcc_gradient(const PauliSum& h, const QmfState& omega, const Ansatz& ansatz) {
  if (h.empty()) return std::vector<double>(ansatz.size(), 0.0);
  DeviceSum d(h);
  return d.qcc_gradient(omega, ansatz);
}

/// iqcc::qmf_energy_gradient (iqcc/qmf.hpp:94-148).
inline double qmf_energy_gradient(const PauliSum& h, const QmfState& omega, std::span<double> grad) {
  DeviceSum d(h);
  const auto t = detail::factor_table(omega);
  const auto dt = detail::deriv_table(omega);
  double e = 0.0;
  detail::check(iqcc_gpu_qmf_energy_gradient(d.handle(), t.data(), dt.data(), &e, grad.data()));
  return e;
}

/// iqcc::gradient (iqcc/dis.hpp:39-52).
inline double gradient(const PauliSum& h, const QmfState& omega, PauliView p) {
  if (!h.empty() && h.word(0).x.size() != p.x.size())
    throw std::invalid_argument("gradient: mismatched qubit counts");
  DeviceSum d(h);
  const auto t = detail::factor_table(omega);
  const auto row = detail::row_of(p);
  double g = 0.0;
  detail::check(iqcc_gpu_gradients(d.handle(), t.data(), row.data(), 1, 0, &g));
  return g;
}

/// iqcc::dis_candidates (iqcc/dis.hpp:140-191).  The device screens every
/// flip group; the seeded shuffle of equal-|g| runs uses the same
/// std::mt19937_64 + std::shuffle as the reference (inside the engine).
inline std::vector<RankedGenerator> dis_candidates(const PauliSum& h, const QmfState& omega,
                                                   std::size_t top_k, const DisOptions& opts = {}) {
  if (top_k < 1) throw std::invalid_argument("dis_candidates: top_k < 1");
  DeviceSum d(h);
  const auto t = detail::factor_table(omega);
  const std::size_t B = blocks_for(h.n_qubits());
  const int has_seed = opts.tie_break_seed ? 1 : 0;
  const uint64_t seed = opts.tie_break_seed ? *opts.tie_break_seed : 0;
  std::size_t n = 0;
  detail::check(iqcc_gpu_dis_candidates(d.handle(), t.data(), omega.at_poles(), top_k, opts.screen_threshold,
                                        opts.per_group_cap, has_seed, seed, nullptr, nullptr, 0, &n));
  const std::size_t k = std::min(n, top_k);
  std::vector<uint64_t> rows(std::max<std::size_t>(k, 1) * 2 * B);
  std::vector<double> g(std::max<std::size_t>(k, 1));
  detail::check(iqcc_gpu_dis_candidates(d.handle(), t.data(), omega.at_poles(), top_k, opts.screen_threshold,
                                        opts.per_group_cap, has_seed, seed, rows.data(), g.data(), k, &n));
  std::vector<RankedGenerator> picks;
  for (std::size_t i = 0; i < k; ++i)
    picks.push_back({PauliWord(h.n_qubits(), std::span<const Block>(rows.data() + i * 2 * B, B),
                               std::span<const Block>(rows.data() + i * 2 * B + B, B)),
                     g[i]});
  return picks;
}

/// iqcc::build_poly_kernels (iqcc/optimizer.hpp:340-368).  The expansion
/// (build_poly, optimizer.hpp:219-268) is host data and used as given; the
/// t(t+1)/2 sandwiches and the n_kernel run on the device, bit-identical to
/// the reference whenever one chunk covers the sum (<= 4096 terms or enough
/// pairs to fill the GPU), else equal up to fp64 reassociation of the chunks.
inline PolyKernels build_poly_kernels(const PauliSum& h, const QmfState& omega, const PolyExpansion& ex) {
  const std::size_t t = ex.subsets.size(), n = ex.n_qubits, B = blocks_for(n);
  PauliSum zero(n);
  if (h.empty()) zero.append(PauliWord(n).view(), Complex{});  // h_kernel stays 0
  DeviceSum d(h.empty() ? zero : h);
  const auto tab = detail::factor_table(omega);
  std::vector<uint64_t> words(std::max<std::size_t>(t, 1) * 2 * B);
  for (std::size_t s = 0; s < t; ++s) {
    const auto row = detail::row_of(ex.subsets[s].word.view());
    std::copy(row.begin(), row.end(), words.begin() + s * 2 * B);
  }
  std::vector<double> hk(std::max<std::size_t>(t * t, 1) * 2), nk(hk.size());
  detail::check(iqcc_gpu_poly_kernels(d.handle(), tab.data(), omega.at_poles(), words.data(), t, hk.data(),
                                      nk.data()));
  PolyKernels ker;
  ker.t = t;
  ker.h_kernel.resize(t * t);
  ker.n_kernel.resize(t * t);
  for (std::size_t i = 0; i < t * t; ++i) {
    ker.h_kernel[i] = Complex(hk[2 * i], hk[2 * i + 1]);
    ker.n_kernel[i] = Complex(nk[2 * i], nk[2 * i + 1]);
  }
  return ker;
}

/// iqcc::merge_sums (iqcc/pauli.hpp:383-415): a + b (a first) on shared words,
/// keep_term(opts.drop_threshold) on every output (check_hermitian is moot:
/// the device holds real coefficients).
inline PauliSum merge_sums(const PauliSum& a, const PauliSum& b, const MergeOptions& opts = {}) {
  if (a.n_qubits() != b.n_qubits()) throw std::invalid_argument("merge_sums: mismatched qubit counts");
  DeviceSum da(a), db(b);
  iqcc_gpu_sum* out = nullptr;
  detail::check(iqcc_gpu_merge_sums(da.handle(), db.handle(), opts.drop_threshold, &out));
  return detail::download(detail::Handle(out), a.n_qubits());
}

// ------------------------------------------------------------ partitioning
/// A PartitionedSum (iqcc/partition.hpp:145-173) resident on the GPUs: 2^m
/// device shards, worker w on CUDA device devices[w] (default w % count).
/// One call drives every shard; any m (several partitions per GPU).
class DevicePartitionedSum {
 public:
  DevicePartitionedSum(const PauliSum& h, const PartitionMap& map, std::vector<int> devices = {})
      : map_(map) {
    map.validate();
    if (map.n_qubits != h.n_qubits()) throw std::invalid_argument("distribute: mismatched qubit counts");
    detail::ensure_engine();
    const uint64_t* rows = h.empty() ? nullptr : h.word(0).x.data();
    const double* coeff =
        h.empty() ? nullptr : reinterpret_cast<const double*>(&const_cast<PauliSum&>(h).coeff(0));
    iqcc_gpu_psum* out = nullptr;
    detail::check(iqcc_gpu_psum_distribute(h.n_qubits(), rows, coeff, h.size(), map.partition_bits.size(),
                                           map.partition_bits.data(), map.owner.data(), map.n_workers,
                                           devices.empty() ? nullptr : devices.data(), &out));
    h_ = out;
  }
  explicit DevicePartitionedSum(const PartitionedSum& ph, std::vector<int> devices = {}) : map_(ph.map) {
    ph.map.validate();
    detail::ensure_engine();
    std::vector<const uint64_t*> rows;
    std::vector<const double*> coeffs;
    std::vector<std::size_t> sizes;
    for (const auto& s : ph.shards) {
      rows.push_back(s.empty() ? nullptr : s.word(0).x.data());
      coeffs.push_back(s.empty() ? nullptr : reinterpret_cast<const double*>(&const_cast<PauliSum&>(s).coeff(0)));
      sizes.push_back(s.size());
    }
    if (ph.shards.size() != ph.map.n_partitions()) throw std::invalid_argument("PartitionMap: owner table size");
    iqcc_gpu_psum* out = nullptr;
    detail::check(iqcc_gpu_psum_create_shards(ph.map.n_qubits, ph.map.partition_bits.size(),
                                              ph.map.partition_bits.data(), ph.map.owner.data(),
                                              ph.map.n_workers, devices.empty() ? nullptr : devices.data(),
                                              rows.data(), coeffs.data(), sizes.data(), &out));
    h_ = out;
  }
  DevicePartitionedSum(const DevicePartitionedSum&) = delete;
  DevicePartitionedSum& operator=(const DevicePartitionedSum&) = delete;
  ~DevicePartitionedSum() {
    if (h_) iqcc_gpu_psum_destroy(h_);
  }
  const PartitionMap& map() const { return map_; }
  std::vector<std::size_t> shard_sizes() const {
    std::vector<std::size_t> s(map_.n_partitions());
    detail::check(iqcc_gpu_psum_shard_sizes(h_, s.data()));
    return s;
  }
  std::size_t total_terms() const {
    std::size_t t = 0;
    for (std::size_t v : shard_sizes()) t += v;
    return t;
  }
  /// parallel_dress (iqcc/partition.hpp:398-452), in place.
  void dress(const DressOp& op, double epsilon, std::size_t max_terms = std::numeric_limits<std::size_t>::max(),
             MessageLog* log = nullptr, ParallelDressStats* stats = nullptr) {
    if (map_.n_qubits != op.generator.n_qubits())
      throw std::invalid_argument("parallel_dress: mismatched qubit counts");
    const auto row = detail::row_of(op.generator.view());
    std::vector<iqcc_message_record> recs(map_.n_partitions());
    std::size_t nl = 0, mask = 0;
    iqcc_compress_stats cs{0, 0.0};
    detail::check(iqcc_gpu_psum_dress(h_, row.data(), std::cos(op.amplitude), std::sin(op.amplitude), epsilon,
                                      max_terms, recs.data(), recs.size(), &nl, stats ? &cs : nullptr, &mask));
    if (log)
      for (std::size_t i = 0; i < std::min(nl, recs.size()); ++i)
        log->records.push_back({recs[i].source, recs[i].destination, recs[i].terms, recs[i].bytes});
    if (stats) {
      stats->compress.dropped_terms += cs.dropped_terms;
      stats->compress.dropped_weight += cs.dropped_weight;
      stats->mask = mask;
    }
  }
  double expect(const QmfState& omega) const {
    const auto t = detail::factor_table(omega);
    double e = 0.0;
    detail::check(iqcc_gpu_psum_expect(h_, t.data(), &e));
    return e;
  }
  double qmf_energy_gradient(const QmfState& omega, std::span<double> grad) const {
    const auto t = detail::factor_table(omega);
    const auto dt = detail::deriv_table(omega);
    double e = 0.0;
    detail::check(iqcc_gpu_psum_qmf_energy_gradient(h_, t.data(), dt.data(), &e, grad.data()));
    return e;
  }
  std::vector<double> gradients(const QmfState& omega, const std::vector<PauliWord>& cands,
                                bool flip_group_only = false) const {
    const auto t = detail::factor_table(omega);
    std::vector<uint64_t> rows;
    for (const auto& c : cands) {
      const auto r = detail::row_of(c.view());
      rows.insert(rows.end(), r.begin(), r.end());
    }
    std::vector<double> g(std::max<std::size_t>(cands.size(), 1));
    detail::check(iqcc_gpu_psum_gradients(h_, t.data(), rows.data(), cands.size(), flip_group_only, g.data()));
    g.resize(cands.size());
    return g;
  }
  /// rebalance (iqcc/partition.hpp:457-494) + migration of moved shards.
  PartitionMap rebalance(double threshold) {
    detail::check(iqcc_gpu_psum_rebalance(h_, threshold, map_.owner.data()));
    return map_;
  }
  PauliSum shard(std::size_t p) const {
    const std::size_t n = shard_sizes().at(p), B = blocks_for(map_.n_qubits);
    std::vector<uint64_t> rows(std::max<std::size_t>(n, 1) * 2 * B);
    std::vector<double> coeff(std::max<std::size_t>(n, 1) * 2);
    std::size_t got = 0;
    detail::check(iqcc_gpu_psum_download_shard(h_, p, rows.data(), coeff.data(), n, &got));
    return detail::from_rows(map_.n_qubits, rows, coeff, got);
  }
  /// gather (iqcc/partition.hpp:222-230), merged on the device.
  PauliSum gather() const {
    const std::size_t n = total_terms(), B = blocks_for(map_.n_qubits);
    std::vector<uint64_t> rows(std::max<std::size_t>(n, 1) * 2 * B);
    std::vector<double> coeff(std::max<std::size_t>(n, 1) * 2);
    std::size_t got = 0;
    detail::check(iqcc_gpu_psum_gather(h_, rows.data(), coeff.data(), n, &got));
    return detail::from_rows(map_.n_qubits, rows, coeff, got);
  }
  /// The shards as a reference PartitionedSum on the host.
  PartitionedSum to_host() const {
    PartitionedSum ph;
    ph.map = map_;
    for (std::size_t p = 0; p < map_.n_partitions(); ++p) ph.shards.push_back(shard(p));
    return ph;
  }

 private:
  PartitionMap map_;
  iqcc_gpu_psum* h_ = nullptr;
};

/// iqcc::distribute (iqcc/partition.hpp:208-220) onto the devices.
inline std::unique_ptr<DevicePartitionedSum> distribute(const PauliSum& h, const PartitionMap& map,
                                                        std::vector<int> devices = {}) {
  return std::make_unique<DevicePartitionedSum>(h, map, std::move(devices));
}

/// iqcc::gather of a device partitioned sum.
inline PauliSum gather(const DevicePartitionedSum& ph) { return ph.gather(); }

/// iqcc::parallel_dress (iqcc/partition.hpp:398-452) with the reference's
/// signature: the shards go to the devices, one dressing step runs there
/// (any mode gives the same sum: shards always run concurrently), and the
/// dressed shards come back as a host PartitionedSum.
inline PartitionedSum parallel_dress(const PartitionedSum& ph, const DressOp& op, double epsilon,
                                     std::size_t max_terms = std::numeric_limits<std::size_t>::max(),
                                     MessageLog* log = nullptr, ExecutionMode mode = ExecutionMode::kDeterministic,
                                     ParallelDressStats* stats = nullptr) {
  (void)mode;
  if (ph.map.n_qubits != op.generator.n_qubits())
    throw std::invalid_argument("parallel_dress: mismatched qubit counts");
  if (op.generator.is_identity()) throw std::invalid_argument("parallel_dress: identity generator");
  DevicePartitionedSum d(ph);
  d.dress(op, epsilon, max_terms, log, stats);
  return d.to_host();
}

/// iqcc::parallel_expect (iqcc/partition.hpp:241-254): worker-order reduction.
inline double parallel_expect(const PartitionedSum& ph, const QmfState& omega,
                              ExecutionMode mode = ExecutionMode::kDeterministic) {
  (void)mode;
  DevicePartitionedSum d(ph);
  return d.expect(omega);
}

}  // namespace iqcc::gpu
