// ref_capi.cpp — exposes the UNMODIFIED reference library (header-only C++20
// under /root/reference/proj/include) through oracle_api.h.  TEST
// INFRASTRUCTURE ONLY: compiled here by oracle/Makefile into
// oracle/_ref/libiqcc_ref.so (git-ignored), used to pin the port
// (iqcc_oracle.cpp), to generate tests/golden/, and as the CPU arm of
// bench.py.  No reference source is copied; this file only calls it.
#include <chrono>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>

#include "generators.hpp"
#include "iqcc/dis.hpp"
#include "iqcc/dressing.hpp"
#include "iqcc/io.hpp"
#include "iqcc/optimizer.hpp"
#include "iqcc/oracle.hpp"
#include "iqcc/partition.hpp"
#include "iqcc/pauli.hpp"
#include "iqcc/qmf.hpp"
#include "oracle_api.h"

struct orc_sum {
  iqcc::PauliSum h;
};
struct orc_rng {
  std::mt19937_64 eng;
};

namespace {
thread_local std::string g_err;
thread_local int g_kind = 0;

template <class F>
auto guard(F&& f, decltype(f()) fail) -> decltype(f()) {
  try {
    g_kind = 0;
    return f();
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    g_kind = 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    g_kind = 2;
  }
  return fail;
}

orc_sum* box(iqcc::PauliSum&& h) { return new orc_sum{std::move(h)}; }

iqcc::PauliWord word_of(std::size_t n, const uint64_t* row) {
  std::size_t B = iqcc::blocks_for(n);
  return iqcc::PauliWord(n, std::span<const iqcc::Block>(row, B),
                         std::span<const iqcc::Block>(row + B, B));
}

iqcc::QmfState qmf_of(std::size_t n, const double* th, const double* ph) {
  iqcc::QmfState q(n);
  std::copy(th, th + n, q.theta.begin());
  std::copy(ph, ph + n, q.phi.begin());
  return q;
}

iqcc::PauliSum sum_of(std::size_t n, const uint64_t* rows, const double* coeff, std::size_t M) {
  iqcc::PauliSum h(n);
  std::size_t B = iqcc::blocks_for(n);
  h.reserve(M);
  for (std::size_t i = 0; i < M; ++i)
    h.append(iqcc::PauliView{{rows + i * 2 * B, B}, {rows + i * 2 * B + B, B}},
             iqcc::Complex(coeff[2 * i], coeff[2 * i + 1]));
  return h;
}

iqcc::PartitionMap map_of(std::size_t n, std::size_t m, const size_t* bits, const size_t* owner,
                          std::size_t nw) {
  iqcc::PartitionMap map;
  map.n_qubits = n;
  map.partition_bits.assign(bits, bits + m);
  map.n_workers = nw;
  map.owner.assign(owner, owner + (std::size_t{1} << m));
  return map;
}
}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
int orc_last_error_kind(void) { return g_kind; }
const char* orc_flavor(void) { return "reference"; }

orc_sum* orc_sum_new(size_t n, const uint64_t* rows, const double* coeff, size_t M) {
  return guard([&]() -> orc_sum* { return box(sum_of(n, rows, coeff, M)); }, nullptr);
}

orc_sum* orc_from_terms(size_t n, const uint64_t* rows, const double* coeff, size_t M, double thr,
                        int check, double tol) {
  return guard([&]() -> orc_sum* {
    std::size_t B = iqcc::blocks_for(n);
    std::vector<iqcc::WeightedTerm> t;
    t.reserve(M);
    for (size_t i = 0; i < M; ++i)
      t.push_back({iqcc::Complex(coeff[2 * i], coeff[2 * i + 1]), word_of(n, rows + i * 2 * B)});
    iqcc::MergeOptions o{thr, check != 0, tol};
    return box(iqcc::PauliSum::from_terms(n, std::move(t), o));
  }, nullptr);
}

void orc_sum_free(orc_sum* h) { delete h; }
size_t orc_sum_size(const orc_sum* h) { return h->h.size(); }
size_t orc_sum_qubits(const orc_sum* h) { return h->h.n_qubits(); }
void orc_sum_export(const orc_sum* h, uint64_t* rows, double* coeff) {
  std::size_t B = h->h.blocks();
  for (size_t i = 0; i < h->h.size(); ++i) {
    auto w = h->h.word(i);
    std::copy(w.x.begin(), w.x.end(), rows + i * 2 * B);
    std::copy(w.z.begin(), w.z.end(), rows + i * 2 * B + B);
    coeff[2 * i] = h->h.coeff(i).real();
    coeff[2 * i + 1] = h->h.coeff(i).imag();
  }
}
int orc_sum_is_canonical(const orc_sum* h) { return h->h.is_canonical(); }
int orc_sum_equal(const orc_sum* a, const orc_sum* b) { return a->h == b->h; }

int orc_canonical_compare(size_t n, const uint64_t* a, const uint64_t* b) {
  return iqcc::canonical_compare(word_of(n, a), word_of(n, b));
}
int orc_commutes(size_t n, const uint64_t* a, const uint64_t* b) {
  return iqcc::commutes(word_of(n, a), word_of(n, b));
}
int orc_multiply(size_t n, const uint64_t* a, const uint64_t* b, uint64_t* out) {
  auto p = iqcc::multiply(word_of(n, a), word_of(n, b));
  std::size_t B = iqcc::blocks_for(n);
  std::copy(p.word.x_bits().begin(), p.word.x_bits().end(), out);
  std::copy(p.word.z_bits().begin(), p.word.z_bits().end(), out + B);
  return p.phase_exponent;
}

orc_sum* orc_merge_sums(const orc_sum* a, const orc_sum* b, double thr, int check, double tol) {
  return guard([&]() -> orc_sum* {
    return box(iqcc::merge_sums(a->h, b->h, iqcc::MergeOptions{thr, check != 0, tol}));
  }, nullptr);
}

orc_sum* orc_compress(const orc_sum* h, double eps, size_t max_terms, size_t* dt, double* dw) {
  return guard([&]() -> orc_sum* {
    iqcc::CompressStats st;
    auto out = iqcc::compress(h->h, eps, max_terms, &st);
    if (dt) *dt += st.dropped_terms;
    if (dw) *dw += st.dropped_weight;
    return box(std::move(out));
  }, nullptr);
}

orc_sum* orc_dress_single(const orc_sum* h, const uint64_t* gen, double tau, double thr, int check,
                          double tol) {
  return guard([&]() -> orc_sum* {
    iqcc::DressOp op{word_of(h->h.n_qubits(), gen), tau};
    return box(iqcc::dress_single(h->h, op, iqcc::MergeOptions{thr, check != 0, tol}));
  }, nullptr);
}

orc_sum* orc_sortless_dress(const orc_sum* h, const uint64_t* gen, double tau, double thr,
                            size_t* n_buckets, size_t* new_stream_sorts) {
  return guard([&]() -> orc_sum* {
    iqcc::DressOp op{word_of(h->h.n_qubits(), gen), tau};
    iqcc::SortlessStats st;
    iqcc::MergeOptions o;
    o.drop_threshold = thr;
    auto out = iqcc::sortless_dress(h->h, op, o, &st);
    if (n_buckets) *n_buckets = st.n_buckets;
    if (new_stream_sorts) *new_stream_sorts = st.new_stream_sorts;
    return box(std::move(out));
  }, nullptr);
}

orc_sum* orc_dress_sequence(const orc_sum* h, size_t K, const uint64_t* gens, const double* taus,
                            double eps, size_t max_terms, double drop_thr, size_t* dt, double* dw) {
  return guard([&]() -> orc_sum* {
    iqcc::Ansatz a;
    std::size_t n = h->h.n_qubits(), B = iqcc::blocks_for(n);
    for (size_t k = 0; k < K; ++k) a.push(word_of(n, gens + k * 2 * B), taus[k]);
    iqcc::CompressStats st;
    iqcc::MergeOptions opts;
    opts.drop_threshold = drop_thr;
    auto out = iqcc::dress_sequence(h->h, a, eps, max_terms, &st, opts);
    if (dt) *dt += st.dropped_terms;
    if (dw) *dw += st.dropped_weight;
    return box(std::move(out));
  }, nullptr);
}

void orc_growth_split(const orc_sum* h, const uint64_t* gen, size_t* nc, size_t* na) {
  auto g = iqcc::growth_split(h->h, word_of(h->h.n_qubits(), gen));
  *nc = g.n_commuting;
  *na = g.n_anticommuting;
}

double orc_expect_word(size_t n, const double* th, const double* ph, const uint64_t* w) {
  return iqcc::expect_word(qmf_of(n, th, ph), word_of(n, w));
}
double orc_expect_sum(const double* th, const double* ph, const orc_sum* h) {
  return iqcc::expect_sum(qmf_of(h->h.n_qubits(), th, ph), h->h);
}
double orc_qcc_energy(const orc_sum* h, const double* th, const double* ph, size_t K,
                      const uint64_t* gens, const double* taus) {
  return guard([&]() -> double {
    iqcc::Ansatz a;
    std::size_t n = h->h.n_qubits(), B = iqcc::blocks_for(n);
    for (size_t k = 0; k < K; ++k) a.push(word_of(n, gens + k * 2 * B), taus[k]);
    return iqcc::qcc_energy(h->h, qmf_of(n, th, ph), a);
  }, 0.0);
}
int orc_qcc_gradient(const orc_sum* h, const double* th, const double* ph, size_t K,
                     const uint64_t* gens, const double* taus, double* g) {
  return guard([&]() -> int {
    iqcc::Ansatz a;
    std::size_t n = h->h.n_qubits(), B = iqcc::blocks_for(n);
    for (size_t k = 0; k < K; ++k) a.push(word_of(n, gens + k * 2 * B), taus[k]);
    auto v = iqcc::qcc_gradient(h->h, qmf_of(n, th, ph), a);
    for (size_t k = 0; k < K; ++k) g[k] = v[k];
    return 0;
  }, -1);
}
int orc_poly_kernels(const orc_sum* h, const double* th, const double* ph, size_t N,
                     const uint64_t* ents, size_t k, size_t cap, size_t* t_out, uint64_t* words_out,
                     int* phase_out, double* hk_out, double* nk_out) {
  return guard([&]() -> int {
    std::size_t n = h->h.n_qubits(), B = iqcc::blocks_for(n);
    std::vector<iqcc::PauliWord> e;
    for (size_t j = 0; j < N; ++j) e.push_back(word_of(n, ents + j * 2 * B));
    iqcc::QmfState om = qmf_of(n, th, ph);
    iqcc::PolyExpansion ex = iqcc::build_poly(e, om, k);
    const std::size_t t = ex.subsets.size();
    *t_out = t;
    if (t > cap) throw std::runtime_error("orc_poly_kernels: capacity");
    iqcc::PolyKernels ker = iqcc::build_poly_kernels(h->h, om, ex);
    for (std::size_t s = 0; s < t; ++s) {
      auto v = ex.subsets[s].word.view();
      std::copy(v.x.begin(), v.x.end(), words_out + s * 2 * B);
      std::copy(v.z.begin(), v.z.end(), words_out + s * 2 * B + B);
      phase_out[s] = ex.subsets[s].phase_exponent;
    }
    for (std::size_t i = 0; i < t * t; ++i) {
      hk_out[2 * i] = ker.h_kernel[i].real();
      hk_out[2 * i + 1] = ker.h_kernel[i].imag();
      nk_out[2 * i] = ker.n_kernel[i].real();
      nk_out[2 * i + 1] = ker.n_kernel[i].imag();
    }
    return 0;
  }, -1);
}
double orc_qmf_energy_gradient(const orc_sum* h, const double* th, const double* ph, double* g) {
  std::size_t n = h->h.n_qubits();
  return iqcc::qmf_energy_gradient(h->h, qmf_of(n, th, ph), std::span<double>(g, 2 * n));
}
double orc_gradient(const orc_sum* h, const double* th, const double* ph, const uint64_t* p) {
  std::size_t n = h->h.n_qubits();
  return iqcc::gradient(h->h, qmf_of(n, th, ph), word_of(n, p));
}

size_t orc_dis_candidates(const orc_sum* h, const double* th, const double* ph, size_t top_k,
                          double thr, size_t cap, int has_seed, uint64_t seed, uint64_t* rows_out,
                          double* g_out, size_t out_cap) {
  return guard([&]() -> size_t {
    std::size_t n = h->h.n_qubits(), B = iqcc::blocks_for(n);
    iqcc::DisOptions o;
    o.screen_threshold = thr;
    o.per_group_cap = cap;
    if (has_seed) o.tie_break_seed = seed;
    auto picks = iqcc::dis_candidates(h->h, qmf_of(n, th, ph), top_k, o);
    for (size_t i = 0; i < picks.size() && i < out_cap; ++i) {
      auto& w = picks[i].word;
      std::copy(w.x_bits().begin(), w.x_bits().end(), rows_out + i * 2 * B);
      std::copy(w.z_bits().begin(), w.z_bits().end(), rows_out + i * 2 * B + B);
      g_out[i] = picks[i].gradient;
    }
    return picks.size();
  }, (size_t)-1);
}

size_t orc_flip_groups(const orc_sum* h, size_t* starts_out, size_t out_cap) {
  auto g = iqcc::group_by_flip(h->h);
  for (size_t i = 0; i < g.size() && i < out_cap; ++i) starts_out[i] = g[i].member_terms.front();
  return g.size();
}

double orc_choose_partition_bits(const orc_sum* h, size_t m, size_t* bits_out) {
  return guard([&]() -> double {
    auto c = iqcc::choose_partition_bits(h->h, m);
    std::copy(c.bits.begin(), c.bits.end(), bits_out);
    return c.imbalance;
  }, -1.0);
}

orc_sum* orc_parallel_dress(const orc_sum* h, size_t m, const size_t* bits, const size_t* owner,
                            size_t nw, const uint64_t* gen, double tau, double eps,
                            size_t max_terms, int threaded, size_t* shard_sizes, size_t* log_out,
                            size_t log_cap, size_t* n_log, size_t* mask_out) {
  return guard([&]() -> orc_sum* {
    std::size_t n = h->h.n_qubits();
    auto ph = iqcc::distribute(h->h, map_of(n, m, bits, owner, nw));
    iqcc::MessageLog log;
    iqcc::ParallelDressStats st;
    auto out = iqcc::parallel_dress(
        ph, iqcc::DressOp{word_of(n, gen), tau}, eps, max_terms, &log,
        threaded ? iqcc::ExecutionMode::kThreaded : iqcc::ExecutionMode::kDeterministic, &st);
    for (size_t p = 0; p < out.shards.size(); ++p) shard_sizes[p] = out.shards[p].size();
    for (size_t i = 0; i < log.records.size() && i < log_cap; ++i) {
      log_out[4 * i + 0] = log.records[i].source;
      log_out[4 * i + 1] = log.records[i].destination;
      log_out[4 * i + 2] = log.records[i].terms;
      log_out[4 * i + 3] = log.records[i].bytes;
    }
    *n_log = log.records.size();
    *mask_out = st.mask;
    return box(iqcc::gather(out));
  }, nullptr);
}

double orc_parallel_expect(const orc_sum* h, size_t m, const size_t* bits, const size_t* owner,
                           size_t nw, const double* th, const double* phi) {
  std::size_t n = h->h.n_qubits();
  auto ph = iqcc::distribute(h->h, map_of(n, m, bits, owner, nw));
  return iqcc::parallel_expect(ph, qmf_of(n, th, phi));
}

int orc_rebalance(const orc_sum* h, size_t m, const size_t* bits, size_t* owner, size_t nw,
                  double threshold) {
  return guard([&]() -> int {
    std::size_t n = h->h.n_qubits();
    auto ph = iqcc::distribute(h->h, map_of(n, m, bits, owner, nw));
    auto map = iqcc::rebalance(ph, threshold);
    std::copy(map.owner.begin(), map.owner.end(), owner);
    return 0;
  }, -1);
}

orc_rng* orc_rng_new(uint64_t seed) { return new orc_rng{std::mt19937_64(seed)}; }
void orc_rng_free(orc_rng* r) { delete r; }
uint64_t orc_rng_next(orc_rng* r) { return r->eng(); }
double orc_rng_uniform(orc_rng* r, double lo, double hi) {
  std::uniform_real_distribution<double> d(lo, hi);
  return d(r->eng);
}
void orc_random_word(orc_rng* r, size_t n, int allow_identity, uint64_t* row_out) {
  auto w = orcgen::random_word(r->eng, n, allow_identity != 0);
  std::copy(w.begin(), w.end(), row_out);
}
orc_sum* orc_random_sum(orc_rng* r, size_t n, size_t max_terms) {
  auto t = orcgen::random_terms(r->eng, n, max_terms);
  return orc_from_terms(n, t.rows.data(), t.coeff.data(), t.size(), 1e-12, 1, 1e-10);
}
void orc_random_qmf(orc_rng* r, size_t n, double* th, double* ph) {
  orcgen::random_qmf(r->eng, n, th, ph);
}

orc_sum* orc_gen_mol(size_t n, size_t count, uint64_t seed) {
  return guard([&]() -> orc_sum* {
    auto t = orcgen::mol_terms(n, count, seed);
    std::size_t B = iqcc::blocks_for(n);
    std::vector<size_t> idx(count);
    for (size_t i = 0; i < count; ++i) idx[i] = i;
    auto view = [&](size_t i) {
      const uint64_t* r = &t.rows[i * 2 * B];
      return iqcc::PauliView{{r, B}, {r + B, B}};
    };
    std::sort(idx.begin(), idx.end(), [&](size_t a, size_t b) {
      int c = iqcc::canonical_compare(view(a), view(b));
      return c != 0 ? c < 0 : a < b;
    });
    iqcc::PauliSum s(n);
    s.reserve(count);
    for (size_t r = 0; r < count; ++r) {
      if (r > 0 && iqcc::words_equal(view(idx[r]), view(idx[r - 1]))) continue;
      s.append(view(idx[r]), iqcc::Complex(t.coeff[2 * idx[r]], 0.0));
    }
    return box(std::move(s));
  }, nullptr);
}

double orc_time_dress_sequence(const orc_sum* h, size_t K, const uint64_t* gens, const double* taus,
                               double eps, size_t max_terms, size_t m_bits, int threads,
                               size_t* terms_in_total, size_t* final_size, orc_sum** out) {
  // Reference CPU arm: parallel_dress (kThreaded) per entangler over 2^m_bits
  // partitions; run_tasks uses min(hardware_concurrency, 2^m) std::threads
  // (iqcc/partition.hpp:190-204).  m_bits = 0 -> serial dress_sequence.
  (void)threads;
  std::size_t n = h->h.n_qubits(), B = iqcc::blocks_for(n);
  size_t tin = 0;
  if (m_bits == 0) {
    auto t0 = std::chrono::steady_clock::now();
    iqcc::PauliSum cur = h->h;
    for (size_t k = 0; k < K; ++k) {
      tin += cur.size();
      cur = iqcc::dress_single(cur, iqcc::DressOp{word_of(n, gens + k * 2 * B), taus[k]});
      if (eps > 0.0 || cur.size() > max_terms) cur = iqcc::compress(cur, eps, max_terms);
    }
    auto t1 = std::chrono::steady_clock::now();
    *terms_in_total = tin;
    *final_size = cur.size();
    if (out) *out = box(std::move(cur));
    return std::chrono::duration<double>(t1 - t0).count();
  }
  auto ph = iqcc::distribute(h->h, iqcc::make_partition_map(h->h, m_bits, size_t{1} << m_bits));
  auto t0 = std::chrono::steady_clock::now();
  for (size_t k = 0; k < K; ++k) {
    tin += ph.total_terms();
    ph = iqcc::parallel_dress(ph, iqcc::DressOp{word_of(n, gens + k * 2 * B), taus[k]}, eps,
                              max_terms, nullptr, iqcc::ExecutionMode::kThreaded, nullptr);
  }
  auto t1 = std::chrono::steady_clock::now();
  *terms_in_total = tin;
  *final_size = ph.total_terms();
  if (out) *out = box(iqcc::gather(ph));  // outside the timed region (bench parity digest)
  return std::chrono::duration<double>(t1 - t0).count();
}

/* extras only the reference flavour provides (fixture generation) --------- */
orc_sum* orc_ref_jordan_wigner_fcidump(const char* path, size_t* n_electrons) {
  return guard([&]() -> orc_sum* {
    auto ints = iqcc::read_fcidump(path);
    if (n_electrons) *n_electrons = ints.n_electrons;
    return box(iqcc::jordan_wigner(ints));
  }, nullptr);
}

orc_sum* orc_ref_parse_pauli_file(const char* path) {
  return guard([&]() -> orc_sum* { return box(iqcc::parse_pauli_file(path)); }, nullptr);
}

int orc_ref_write_pauli_file(const orc_sum* h, const char* path) {
  return guard([&]() -> int {
    iqcc::write_pauli_file(h->h, path);
    return 0;
  }, -1);
}

double orc_ref_ground_energy(const orc_sum* h) {
  return guard([&]() -> double { return iqcc::oracle::ground_energy(h->h); }, 0.0);
}

/* One iQCC iteration as composed in SURVEY.md §3.6: DIS top-k at omega,
 * optimize_amplitudes, dress_sequence(eps, max_terms).  Returns the dressed
 * sum; writes the picked entanglers and amplitudes (<= k). */
orc_sum* orc_ref_iqcc_iteration(const orc_sum* h, const double* th, const double* ph, size_t k,
                                double eps, size_t max_terms, uint64_t* gens_out, double* taus_out,
                                size_t* n_picked, double* energy_out) {
  return guard([&]() -> orc_sum* {
    std::size_t n = h->h.n_qubits(), B = iqcc::blocks_for(n);
    auto omega = qmf_of(n, th, ph);
    auto picks = iqcc::dis_candidates(h->h, omega, k);
    *n_picked = picks.size();
    if (picks.empty()) {
      *energy_out = iqcc::expect_sum(omega, h->h);
      return box(iqcc::PauliSum(h->h));
    }
    std::vector<iqcc::PauliWord> ents;
    for (auto& p : picks) ents.push_back(p.word);
    auto amp = iqcc::optimize_amplitudes(h->h, omega, ents);
    iqcc::Ansatz a;
    for (size_t i = 0; i < ents.size(); ++i) {
      a.push(ents[i], amp.tau[i]);
      std::copy(ents[i].x_bits().begin(), ents[i].x_bits().end(), gens_out + i * 2 * B);
      std::copy(ents[i].z_bits().begin(), ents[i].z_bits().end(), gens_out + i * 2 * B + B);
      taus_out[i] = amp.tau[i];
    }
    auto out = iqcc::dress_sequence(h->h, a, eps, max_terms);
    *energy_out = iqcc::expect_sum(omega, out);
    return box(std::move(out));
  }, nullptr);
}

}  // extern "C"
