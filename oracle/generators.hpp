// generators.hpp — seeded input generators shared by both CPU checkers.
// TEST INFRASTRUCTURE ONLY (see oracle_api.h).
//
// The mt19937_64-based generators reproduce the semantics of the reference's
// test helpers (tests/helpers.hpp:74-109): letters drawn iid from
// uniform_int_distribution<int>(0,3) with 0=I 1=X 2=Z 3=Y, identity rejected
// when requested; coefficients from uniform_real_distribution<double>(-1,1)
// drawn BEFORE the word of each term (braced-init order); QMF angles from
// uniform_real_distribution<double>(-3,3), theta then phi per qubit.  Because
// they call the same libstdc++ distributions in the same order, a seed gives
// the same inputs the reference tests see.
#pragma once
#include <cstdint>
#include <random>
#include <vector>

#include "../paper_2603_08883_b200/csrc/gen_mol.h"

namespace orcgen {

inline std::size_t blocks_for(std::size_t n) { return n == 0 ? 1 : (n + 63) / 64; }

/// One word in row layout (x blocks then z blocks).
inline std::vector<std::uint64_t> random_word(std::mt19937_64& rng, std::size_t n,
                                              bool allow_identity) {
  const std::size_t B = blocks_for(n);
  std::uniform_int_distribution<int> letter(0, 3);
  for (;;) {
    std::vector<std::uint64_t> row(2 * B, 0);
    bool any = false;
    for (std::size_t q = 0; q < n; ++q) {
      int l = letter(rng);
      std::uint64_t bit = std::uint64_t{1} << (q % 64);
      if (l == 1 || l == 3) row[q / 64] |= bit;
      if (l == 2 || l == 3) row[B + q / 64] |= bit;
      any = any || l != 0;
    }
    if (any || allow_identity) return row;
  }
}

struct RawTerms {
  std::vector<std::uint64_t> rows;
  std::vector<double> coeff;  // (re, im) pairs
  std::size_t size() const { return coeff.size() / 2; }
};

inline RawTerms random_terms(std::mt19937_64& rng, std::size_t n, std::size_t count) {
  std::uniform_real_distribution<double> coeff(-1.0, 1.0);
  RawTerms t;
  for (std::size_t k = 0; k < count; ++k) {
    double c = coeff(rng);
    auto row = random_word(rng, n, true);
    t.rows.insert(t.rows.end(), row.begin(), row.end());
    t.coeff.push_back(c);
    t.coeff.push_back(0.0);
  }
  return t;
}

inline void random_qmf(std::mt19937_64& rng, std::size_t n, double* theta, double* phi) {
  std::uniform_real_distribution<double> angle(-3.0, 3.0);
  for (std::size_t j = 0; j < n; ++j) {
    theta[j] = angle(rng);
    phi[j] = angle(rng);
  }
}

/// G_mol terms 0..count-1 in generation order (not yet canonical).
inline RawTerms mol_terms(std::size_t n, std::size_t count, std::uint64_t seed) {
  const std::size_t B = blocks_for(n);
  RawTerms t;
  t.rows.resize(count * 2 * B);
  t.coeff.resize(count * 2);
  for (std::size_t k = 0; k < count; ++k) {
    t.coeff[2 * k] = iqcc_gen::mol_term((uint32_t)n, (uint32_t)B, seed, k, &t.rows[k * 2 * B]);
    t.coeff[2 * k + 1] = 0.0;
  }
  return t;
}

}  // namespace orcgen
