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
      expect(iqcc::gpu::sortless_dress(h, op) == iqcc::sortless_dress(h, op), "sortless_dress/557", t);
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
