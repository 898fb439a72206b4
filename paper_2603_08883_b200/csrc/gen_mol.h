// gen_mol.h — counter-based synthetic "molecular-like" Pauli term generator
// (SURVEY.md §8(d) G_mol).  Term k of G_mol(n, seed) is a pure function of
// (n, seed, k), so the host generator (oracle/, the CPU baseline) and the
// device generator (bench input) produce bit-identical term sets.
//
//   * k == 0 is the identity with coefficient -1.0 (molecular H carries a
//     constant term; it exercises the identity keep rules of
//     iqcc/pauli.hpp:180-184 and :449-456).
//   * otherwise a flip set of size {0,2,4} with probability {.10,.45,.45},
//     X/Y letters on it with an even number of Y (a real Hamiltonian, cf.
//     tests/test_dis.cpp:14-24), Z with p = 1/2 on every other qubit, and a
//     coefficient whose binary exponent is uniform over [-33,-1] with a random
//     52-bit mantissa and sign (log-uniform |c| in [1.16e-10, 1)).
//
// Words use the reference row layout: B x-blocks then B z-blocks, bit j of
// block j/64 is qubit j (iqcc/pauli.hpp:35-120, 373-377).  No transcendental
// functions are used, so host and device agree bit for bit.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define IQCC_HD __host__ __device__ __forceinline__
#else
#define IQCC_HD inline
#endif

namespace iqcc_gen {

struct SplitMix {
  uint64_t s;
  IQCC_HD uint64_t next() {
    s += 0x9E3779B97F4A7C15ull;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
};

IQCC_HD SplitMix term_stream(uint64_t seed, uint64_t k) {
  SplitMix m{seed * 0xD1B54A32D192ED03ull + 0x5851F42D4C957F2Dull};
  m.s ^= k * 0x9E3779B97F4A7C15ull;
  m.next();
  return m;
}

/// Writes term k into row[0..2B) (x blocks then z blocks) and returns its
/// coefficient.  Requires 1 <= n_qubits <= 64*B, B <= 4.
IQCC_HD double mol_term(uint32_t n_qubits, uint32_t B, uint64_t seed,
                        uint64_t k, uint64_t* row) {
  for (uint32_t b = 0; b < 2 * B; ++b) row[b] = 0;
  if (k == 0) return -1.0;
  SplitMix r = term_stream(seed, k);
  uint32_t u = (uint32_t)(r.next() % 100u);
  uint32_t w = u < 10 ? 0u : (u < 55 ? 2u : 4u);
  if (w > n_qubits) w = n_qubits & ~1u;
  uint32_t flips[4] = {0, 0, 0, 0};
  for (uint32_t i = 0; i < w; ++i) {
    for (;;) {
      uint32_t q = (uint32_t)(r.next() % n_qubits);
      bool dup = false;
      for (uint32_t j = 0; j < i; ++j) dup = dup || flips[j] == q;
      if (!dup) { flips[i] = q; break; }
    }
  }
  uint32_t ny = 0;
  uint64_t ybits = r.next();
  for (uint32_t i = 0; i < w; ++i) {
    uint32_t q = flips[i];
    row[q >> 6] |= 1ull << (q & 63);                  // x bit
    bool y = (ybits >> i) & 1u;
    if (i + 1 == w && ((ny + (y ? 1u : 0u)) & 1u)) y = !y;  // even #Y
    if (y) { row[B + (q >> 6)] |= 1ull << (q & 63); ++ny; }
  }
  for (uint32_t b = 0; b < B; ++b) {
    uint64_t valid = (64 * (b + 1) <= n_qubits)
                         ? ~0ull
                         : (n_qubits > 64 * b ? ((1ull << (n_qubits - 64 * b)) - 1) : 0ull);
    uint64_t zr = r.next() & valid & ~row[b];          // Z only off the flip set
    row[B + b] |= zr;
  }
  uint64_t e = 1 + r.next() % 33u;
  uint64_t mant = r.next() >> 12;
  uint64_t sign = r.next() & 1u;
  uint64_t bits = (sign << 63) | ((1023ull - e) << 52) | mant;
  double c;
#if defined(__CUDA_ARCH__)
  c = __longlong_as_double((long long)bits);
#else
  __builtin_memcpy(&c, &bits, 8);
#endif
  return c;
}

}  // namespace iqcc_gen
