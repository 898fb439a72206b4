// C++ parity harness: the reference's own functions (namespace iqcc, the
// UNMODIFIED headers) against the drop-in shim (iqcc::gpu, the B200 engine)
// on the reference tests' seeds.  Built by tests/cpp/Makefile where
// /root/reference exists; the binary (tests/cpp/_bin) runs on the GPU box.
// Prints one "ok <name> <cases>" line per check; exits 1 on any mismatch.
#include <cstring>
#include <numbers>
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <random>

#include "iqcc/dressing.hpp"
#include "iqcc/io.hpp"
#include "iqcc/optimizer.hpp"
#include "iqcc/partition.hpp"
#include "iqcc/pauli.hpp"
#include "iqcc/qmf.hpp"
#include "iqcc_b200/iqcc_gpu.hpp"

namespace {
// same semantics as tests/helpers.hpp:74-99 (not included: it needs Eigen)
iqcc::PauliWord rand_word(std::mt19937_64& rng, std::size_t n, bool allow_id) {
  std::uniform_int_distribution<int> letter(0, 3);
  for (;;) {
    iqcc::PauliWord w(n);
    bool any = false;
    for (std::size_t j = 0; j < n; ++j) {
      int l = letter(rng);
      if (l == 1 || l == 3) w.set_x(j);
      if (l == 2 || l == 3) w.set_z(j);
      any = any || l != 0;
    }
    if (any || allow_id) return w;
  }
}
iqcc::PauliSum rand_sum(std::mt19937_64& rng, std::size_t n, std::size_t m) {
  std::uniform_real_distribution<double> coeff(-1.0, 1.0);
  std::vector<iqcc::WeightedTerm> t;
  for (std::size_t k = 0; k < m; ++k) {
    double c = coeff(rng);
    t.push_back({c, rand_word(rng, n, true)});
  }
  return iqcc::PauliSum::from_terms(n, std::move(t));
}
int failures = 0;
void expect(bool ok, const char* what, int i) {
  if (!ok) {
    ++failures;
    std::printf("FAIL %s case %d\n", what, i);
  }
}
}  // namespace

int main(int argc, char** argv) {
  // dress_single, tests/test_dressing.cpp:177-196 seeds
  {
    std::mt19937_64 rng(557);
    std::uniform_real_distribution<double> amp(-3.0, 3.0);
    for (int t = 0; t < 120; ++t) {
      std::size_t n = 2 + t % 7;
      auto h = rand_sum(rng, n, 12 * n);
      iqcc::DressOp op{rand_word(rng, n, false), amp(rng)};
      expect(iqcc::gpu::dress_single(h, op) == iqcc::dress_single(h, op), "dress_single/557", t);
      iqcc::SortlessStats sa, sb;
      expect(iqcc::gpu::sortless_dress(h, op, {}, &sa) == iqcc::sortless_dress(h, op, {}, &sb), "sortless_dress/557", t);
      expect(sa.n_buckets == sb.n_buckets && sa.new_term_streams == sb.new_term_streams &&
                 sa.new_stream_sorts == sb.new_stream_sorts,
             "sortless_stats/557", t);
    }
    std::printf("ok dress_single 120\n");
  }
  // pipeline with truncation, tests/test_partition.cpp:180-208 seeds
  {
    std::mt19937_64 rng(631);
    std::uniform_real_distribution<double> amp(-3.0, 3.0);
    for (int t = 0; t < 40; ++t) {
      std::size_t n = 3 + t % 4;
      auto h = rand_sum(rng, n, 25 * n);
      iqcc::DressOp op{rand_word(rng, n, false), amp(rng)};
      double eps = (t % 3 == 0) ? 1e-3 : 0.0;
      std::size_t mt = (t % 4 == 0) ? 40 : 100000;
      iqcc::Ansatz a;
      a.push(op.generator, op.amplitude);
      iqcc::CompressStats s1, s2;
      expect(iqcc::gpu::dress_sequence(h, a, eps, mt, &s1) == iqcc::dress_sequence(h, a, eps, mt, &s2),
             "dress_sequence/631", t);
      expect(s1.dropped_terms == s2.dropped_terms, "dress_sequence/631 stats", t);
    }
    std::printf("ok dress_sequence 40\n");
  }
  // compress, tests/test_pauli.cpp:157-197
  {
    std::mt19937_64 rng(41);
    for (int t = 0; t < 40; ++t) {
      auto h = rand_sum(rng, 5, 40);
      for (double eps : {0.0, 1e-3, 0.2})
        for (std::size_t mt : {std::size_t{1}, std::size_t{10}, std::size_t{1000}})
          expect(iqcc::gpu::compress(h, eps, mt) == iqcc::compress(h, eps, mt), "compress/41", t);
    }
    std::printf("ok compress 360\n");
  }
  // C1 ingestion path: JW of the shipped FCIDUMP, 3 dressings
  if (argc > 1) {
    auto h = iqcc::jordan_wigner(iqcc::read_fcidump(argv[1]));
    std::mt19937_64 rng(547);
    std::uniform_real_distribution<double> amp(-1.5, 1.5);
    iqcc::Ansatz a;
    for (int k = 0; k < 3; ++k) a.push(rand_word(rng, h.n_qubits(), false), amp(rng));
    expect(iqcc::gpu::dress_sequence(h, a, 0.0) == iqcc::dress_sequence(h, a, 0.0), "h2 sequence", 0);
    std::printf("ok fcidump_sequence 1\n");
  }
  // qcc_energy / qcc_gradient, iqcc/optimizer.hpp:19-77 (tests/test_optimizer.cpp shapes)
  {
    std::mt19937_64 rng(619);
    std::uniform_real_distribution<double> amp(-1.0, 1.0), ang(-3.0, 3.0);
    int cases = 0;
    for (int t = 0; t < 12; ++t) {
      std::size_t n = 3 + t % 5;
      auto h = rand_sum(rng, n, 10 * n);
      iqcc::QmfState om(n);
      for (std::size_t j = 0; j < n; ++j) {
        om.theta[j] = ang(rng);
        om.phi[j] = ang(rng);
      }
      iqcc::Ansatz a;
      for (int k = 0; k < 3; ++k) a.push(rand_word(rng, n, false), amp(rng));
      const double e = iqcc::gpu::qcc_energy(h, om, a), er = iqcc::qcc_energy(h, om, a);
      expect(std::fabs(e - er) <= 1e-10 * std::max(1.0, std::fabs(er)), "qcc_energy/619", t);
      const auto g = iqcc::gpu::qcc_gradient(h, om, a), gr = iqcc::qcc_gradient(h, om, a);
      double scale = 1.0;
      for (double v : gr) scale = std::max(scale, std::fabs(v));
      for (std::size_t k = 0; k < g.size(); ++k)
        expect(std::fabs(g[k] - gr[k]) <= 1e-10 * scale, "qcc_gradient/619", t);
      ++cases;
    }
    std::printf("ok qcc_energy_gradient %d\n", cases);
  }
  // build_poly_kernels, iqcc/optimizer.hpp:340-368 (tests/test_optimizer.cpp:185-230 shapes):
  // bit-identical kernels (each sum fits one chunk)
  {
    std::mt19937_64 rng(757);
    std::uniform_real_distribution<double> ang(-3.0, 3.0);
    int cases = 0;
    for (int t = 0; t < 8; ++t) {
      std::size_t n = 3 + 9 * (t % 4);
      auto h = rand_sum(rng, n, 12 * n);
      iqcc::QmfState om(n);
      for (std::size_t j = 0; j < n; ++j) {
        om.theta[j] = t % 2 ? (j % 3 ? 0.0 : std::numbers::pi) : ang(rng);
        om.phi[j] = t % 2 ? 0.0 : ang(rng);
      }
      std::vector<iqcc::PauliWord> ents;
      for (int k = 0; k < 4; ++k) ents.push_back(rand_word(rng, n, false));
      iqcc::PolyExpansion ex = iqcc::build_poly(ents, om, 2 + t % 3);
      auto a = iqcc::gpu::build_poly_kernels(h, om, ex), b = iqcc::build_poly_kernels(h, om, ex);
      bool same = a.t == b.t;
      for (std::size_t i = 0; same && i < b.t * b.t; ++i)
        same = std::memcmp(&a.h_kernel[i], &b.h_kernel[i], sizeof(iqcc::Complex)) == 0 &&
               std::memcmp(&a.n_kernel[i], &b.n_kernel[i], sizeof(iqcc::Complex)) == 0;
      expect(same, "build_poly_kernels/757", t);
      ++cases;
    }
    std::printf("ok build_poly_kernels %d\n", cases);
  }
  // parallel_dress with the reference's signature, tests/test_partition.cpp:180-208
  // (seed 631): gathered sums AND message logs equal for every worker count
  {
    std::mt19937_64 rng(631);
    std::uniform_real_distribution<double> amp(-3.0, 3.0);
    int cases = 0;
    for (int t = 0; t < 16; ++t) {
      std::size_t n = 3 + t % 4;
      auto h = rand_sum(rng, n, 25 * n);
      iqcc::DressOp op{rand_word(rng, n, false), amp(rng)};
      double eps = (t % 3 == 0) ? 1e-3 : 0.0;
      std::size_t mt = (t % 4 == 0) ? 40 : 100000;
      for (std::size_t workers : {1, 2, 4, 8}) {
        const std::size_t m = workers == 1 ? 2 : 3;
        auto ph = iqcc::distribute(h, iqcc::make_partition_map(h, m, workers));
        iqcc::MessageLog la, lb;
        iqcc::ParallelDressStats sa, sb;
        auto a = iqcc::gpu::parallel_dress(ph, op, eps, mt, &la, iqcc::ExecutionMode::kThreaded, &sa);
        auto b = iqcc::parallel_dress(ph, op, eps, mt, &lb, iqcc::ExecutionMode::kDeterministic, &sb);
        expect(iqcc::gather(a) == iqcc::gather(b), "parallel_dress/631 gather", t);
        bool shards_equal = a.shards.size() == b.shards.size();
        for (std::size_t p = 0; shards_equal && p < a.shards.size(); ++p) shards_equal = a.shards[p] == b.shards[p];
        expect(shards_equal, "parallel_dress/631 shards", t);
        bool logs = la.records.size() == lb.records.size();
        for (std::size_t i = 0; logs && i < la.records.size(); ++i)
          logs = la.records[i].source == lb.records[i].source &&
                 la.records[i].destination == lb.records[i].destination &&
                 la.records[i].terms == lb.records[i].terms && la.records[i].bytes == lb.records[i].bytes;
        expect(logs && la.total_bytes() == lb.total_bytes(), "parallel_dress/631 message log", t);
        expect(sa.mask == sb.mask && sa.compress.dropped_terms == sb.compress.dropped_terms,
               "parallel_dress/631 stats", t);
        ++cases;
      }
    }
    std::printf("ok parallel_dress %d\n", cases);
  }
  // parallel_expect + rebalance (tests/test_partition.cpp:257-309, seeds 647, 653)
  {
    std::mt19937_64 rng(647);
    std::uniform_real_distribution<double> ang(-3.0, 3.0);
    int cases = 0;
    for (int t = 0; t < 8; ++t) {
      auto h = rand_sum(rng, 6, 100);
      iqcc::QmfState om(6);
      for (std::size_t j = 0; j < 6; ++j) {
        om.theta[j] = ang(rng);
        om.phi[j] = ang(rng);
      }
      for (std::size_t workers : {1, 2, 4}) {
        auto ph = iqcc::distribute(h, iqcc::make_partition_map(h, 3, workers));
        const double a = iqcc::gpu::parallel_expect(ph, om), b = iqcc::parallel_expect(ph, om);
        expect(std::fabs(a - b) <= 1e-10 * std::max(1.0, std::fabs(b)), "parallel_expect/647", t);
        ++cases;
      }
    }
    std::mt19937_64 rng2(653);
    auto h = rand_sum(rng2, 6, 160);
    iqcc::PartitionMap map;
    map.n_qubits = 6;
    map.partition_bits = {0, 1, 2};
    map.n_workers = 4;
    map.owner.assign(8, 0);
    auto ph = iqcc::distribute(h, map);
    iqcc::gpu::DevicePartitionedSum d(h, map);
    expect(d.rebalance(1.5).owner == iqcc::rebalance(ph, 1.5).owner, "rebalance/653", 0);
    expect(d.gather() == h, "rebalance/653 gather", 0);
    std::printf("ok parallel_expect_rebalance %d\n", cases + 1);
  }
  // merge_sums, iqcc/pauli.hpp:383-415 (tests/test_pauli.cpp seed 37)
  {
    std::mt19937_64 rng(37);
    for (int t = 0; t < 30; ++t) {
      std::size_t n = 2 + t % 6;
      auto a = rand_sum(rng, n, 40), b = rand_sum(rng, n, 40);
      for (double drop : {1e-12, 0.0, 0.3}) {
        iqcc::MergeOptions o;
        o.drop_threshold = drop;
        expect(iqcc::gpu::merge_sums(a, b, o) == iqcc::merge_sums(a, b, o), "merge_sums/37", t);
      }
    }
    std::printf("ok merge_sums 90\n");
  }
  // dress_sequence forwards MergeOptions (iqcc/dressing.hpp:311-324)
  {
    std::mt19937_64 rng(29);
    std::uniform_real_distribution<double> amp(-1.0, 1.0);
    for (int t = 0; t < 12; ++t) {
      std::size_t n = 4 + t % 5;
      auto h = rand_sum(rng, n, 30 * n);
      iqcc::Ansatz a;
      for (int k = 0; k < 3; ++k) a.push(rand_word(rng, n, false), amp(rng));
      iqcc::MergeOptions o;
      o.drop_threshold = t % 2 ? 0.0 : 0.05;
      expect(iqcc::gpu::dress_sequence(h, a, 0.0, 1000, nullptr, o) == iqcc::dress_sequence(h, a, 0.0, 1000, nullptr, o),
             "dress_sequence merge options", t);
    }
    std::printf("ok dress_sequence_options 12\n");
  }
  // identity generator rejected with std::invalid_argument
  {
    iqcc::PauliSum h(2);
    h.append(iqcc::PauliWord::from_string("XI"), 1.0);
    bool threw = false;
    try {
      iqcc::gpu::dress_single(h, {iqcc::PauliWord(2), 0.5});
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    expect(threw, "identity generator", 0);
    std::printf("ok exceptions 1\n");
  }
  std::printf(failures ? "FAILED %d\n" : "ALL OK\n", failures);
  return failures ? 1 : 0;
}
