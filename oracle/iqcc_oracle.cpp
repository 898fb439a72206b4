// iqcc_oracle.cpp — CPU restatement ("port") of the reference algorithms on
// the B200 hot path.  TEST INFRASTRUCTURE ONLY: the parity checker for the
// CUDA engine (see oracle_api.h).  Built with -O2 -ffp-contract=off (no FMA
// contraction) into oracle/liboracle.so.
//
// Every function cites the reference code it restates (paths relative to
// /root/reference/proj/include).  Coefficient arithmetic is done with
// std::complex<double> in the same operation order as the reference, so
// results are bit-identical; tests pin this against oracle/_ref (the
// reference headers compiled unmodified) and the golden fixtures.
#include <algorithm>
#include <bit>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <limits>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "generators.hpp"
#include "oracle_api.h"

using u64 = std::uint64_t;
using cplx = std::complex<double>;

struct orc_sum {
  std::size_t n = 0, B = 1;
  std::vector<u64> rows;  // [M][2B]
  std::vector<cplx> c;    // [M]
  std::size_t size() const { return c.size(); }
  const u64* row(std::size_t i) const { return rows.data() + i * 2 * B; }
  void push(const u64* r, cplx v) {
    rows.insert(rows.end(), r, r + 2 * B);
    c.push_back(v);
  }
};

struct orc_rng {
  std::mt19937_64 eng;
};

namespace {

thread_local std::string g_err;
thread_local int g_kind = 0;

struct invalid_arg : std::runtime_error {
  using std::runtime_error::runtime_error;
};

template <class F>
auto guard(F&& f, decltype(f()) fail) -> decltype(f()) {
  try {
    g_kind = 0;
    return f();
  } catch (const invalid_arg& e) {
    g_err = e.what();
    g_kind = 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    g_kind = 2;
  }
  return fail;
}

std::size_t blocks_for(std::size_t n) { return orcgen::blocks_for(n); }

// Bit reversal: reversed words compare as plain unsigned integers in the
// canonical order of iqcc/pauli.hpp:146-161 (qubit 0 is the most
// significant position, x plane before z plane).
u64 rev64(u64 v) {
  v = ((v >> 1) & 0x5555555555555555ull) | ((v & 0x5555555555555555ull) << 1);
  v = ((v >> 2) & 0x3333333333333333ull) | ((v & 0x3333333333333333ull) << 2);
  v = ((v >> 4) & 0x0F0F0F0F0F0F0F0Full) | ((v & 0x0F0F0F0F0F0F0F0Full) << 4);
  return __builtin_bswap64(v);
}

int cmp_rows(const u64* a, const u64* b, std::size_t B) {
  for (std::size_t w = 0; w < 2 * B; ++w) {
    if (a[w] == b[w]) continue;
    return rev64(a[w]) < rev64(b[w]) ? -1 : 1;
  }
  return 0;
}

bool is_id(const u64* r, std::size_t B) {
  for (std::size_t w = 0; w < 2 * B; ++w)
    if (r[w]) return false;
  return true;
}

// keep_term, iqcc/pauli.hpp:180-184
bool keep(cplx v, const u64* r, std::size_t B, double thr) {
  if (is_id(r, B)) return true;
  if (v == cplx{}) return false;
  return std::abs(v) >= thr;
}

// commutes, iqcc/pauli.hpp:188-193 (parity of the symplectic form)
bool commute(const u64* p, const u64* q, std::size_t B) {
  unsigned s = 0;
  for (std::size_t b = 0; b < B; ++b)
    s += std::popcount((p[b] & q[B + b]) ^ (p[B + b] & q[b]));
  return (s & 1u) == 0;
}

// multiply_into, iqcc/pauli.hpp:202-215: out = p xor q, returns t (p*q = i^t out)
int mult(const u64* p, const u64* q, u64* out, std::size_t B) {
  long t = 0;
  for (std::size_t b = 0; b < B; ++b) {
    u64 px = p[b], pz = p[B + b], qx = q[b], qz = q[B + b];
    u64 rx = px ^ qx, rz = pz ^ qz;
    t += std::popcount(px & pz) + std::popcount(qx & qz) - std::popcount(rx & rz) +
         2 * std::popcount(pz & qx);
    out[b] = rx;
    out[B + b] = rz;
  }
  return (int)(((t % 4) + 4) % 4);
}

// phase_value, iqcc/pauli.hpp:217-220
cplx phase(int t) {
  static const cplx tab[4] = {{1, 0}, {0, 1}, {-1, 0}, {0, -1}};
  return tab[t & 3];
}

void herm_check(const orc_sum& h, double tol) {  // assert_hermitian, pauli.hpp:358-366
  for (std::size_t i = 0; i < h.size(); ++i) {
    double re = std::abs(h.c[i].real());
    if (std::abs(h.c[i].imag()) >= tol * std::max(1.0, re))
      throw std::runtime_error("hermiticity violated: coefficient " + std::to_string(i));
  }
}

// PauliSum::from_terms, iqcc/pauli.hpp:302-326.  Index sort with the same
// strict-weak comparator drives libstdc++'s introsort through the same
// decisions as sorting the term structs, so duplicate runs are combined in
// the same order.
orc_sum from_terms(std::size_t n, const u64* rows, const cplx* c, std::size_t M, double thr,
                   bool check, double tol) {
  const std::size_t B = blocks_for(n);
  std::vector<std::size_t> idx(M);
  std::iota(idx.begin(), idx.end(), 0);
  std::sort(idx.begin(), idx.end(), [&](std::size_t a, std::size_t b) {
    return cmp_rows(rows + a * 2 * B, rows + b * 2 * B, B) < 0;
  });
  orc_sum out;
  out.n = n;
  out.B = B;
  std::size_t i = 0;
  while (i < M) {
    cplx v = c[idx[i]];
    std::size_t j = i + 1;
    while (j < M && cmp_rows(rows + idx[i] * 2 * B, rows + idx[j] * 2 * B, B) == 0)
      v += c[idx[j++]];
    if (keep(v, rows + idx[i] * 2 * B, B, thr)) out.push(rows + idx[i] * 2 * B, v);
    i = j;
  }
  if (check) herm_check(out, tol);
  return out;
}

// merge_sums, iqcc/pauli.hpp:383-415 (a's addend first on equal words)
orc_sum merge(const orc_sum& a, const orc_sum& b, double thr, bool check, double tol) {
  if (a.n != b.n) throw invalid_arg("merge_sums: mismatched qubit counts");
  const std::size_t B = a.B;
  orc_sum out;
  out.n = a.n;
  out.B = B;
  std::size_t i = 0, j = 0;
  auto put = [&](const u64* r, cplx v) {
    if (keep(v, r, B, thr)) out.push(r, v);
  };
  while (i < a.size() || j < b.size()) {
    int s = i == a.size() ? 1 : j == b.size() ? -1 : cmp_rows(a.row(i), b.row(j), B);
    if (s < 0) {
      put(a.row(i), a.c[i]);
      ++i;
    } else if (s > 0) {
      put(b.row(j), b.c[j]);
      ++j;
    } else {
      put(a.row(i), a.c[i] + b.c[j]);
      ++i;
      ++j;
    }
  }
  if (check) herm_check(out, tol);
  return out;
}

// dress_single, iqcc/dressing.hpp:197-220 with product_scale :57-59 and
// append_product pauli.hpp:287-293
orc_sum dress(const orc_sum& h, const u64* P, double tau, double thr, bool check, double tol) {
  const std::size_t B = h.B;
  if (is_id(P, B)) throw invalid_arg("dress_single: identity generator");
  const double cs = std::cos(tau), sn = std::sin(tau);
  orc_sum surv, prod;
  surv.n = prod.n = h.n;
  surv.B = prod.B = B;
  std::vector<u64> tmp(2 * B);
  for (std::size_t i = 0; i < h.size(); ++i) {
    if (commute(h.row(i), P, B)) {
      surv.push(h.row(i), h.c[i]);
      continue;
    }
    surv.push(h.row(i), h.c[i] * cs);
    if (sn != 0.0) {
      int t = mult(h.row(i), P, tmp.data(), B);
      cplx scale = h.c[i] * sn * cplx{0.0, -1.0};
      prod.push(tmp.data(), scale * phase(t));
    }
  }
  orc_sum sorted = from_terms(h.n, prod.rows.data(), prod.c.data(), prod.size(), 0.0, false, 0.0);
  return merge(surv, sorted, thr, check, tol);
}

// compress, iqcc/pauli.hpp:425-474.  The reference stable_sorts kept indices
// by |c| descending; an explicit (|c| desc, index asc) order is the same
// permutation.
orc_sum compress(const orc_sum& h, double eps, std::size_t max_terms, std::size_t* dt,
                 double* dw) {
  if (eps < 0) throw invalid_arg("compress: epsilon < 0");
  if (max_terms < 1) throw invalid_arg("compress: max_terms < 1");
  const std::size_t B = h.B;
  std::vector<char> kp(h.size(), 0);
  std::vector<std::size_t> kept;
  for (std::size_t i = 0; i < h.size(); ++i)
    if (is_id(h.row(i), B) || std::abs(h.c[i]) >= eps) {
      kp[i] = 1;
      kept.push_back(i);
    }
  if (kept.size() > max_terms) {
    std::sort(kept.begin(), kept.end(), [&](std::size_t a, std::size_t b) {
      double ma = std::abs(h.c[a]), mb = std::abs(h.c[b]);
      if (ma != mb) return ma > mb;
      return a < b;
    });
    std::fill(kp.begin(), kp.end(), 0);
    std::size_t budget = max_terms;
    bool has_id = h.size() > 0 && is_id(h.row(0), B);
    if (has_id) {
      kp[0] = 1;
      --budget;
    }
    for (std::size_t r = 0; r < kept.size() && budget > 0; ++r) {
      if (has_id && kept[r] == 0) continue;
      kp[kept[r]] = 1;
      --budget;
    }
  }
  orc_sum out;
  out.n = h.n;
  out.B = B;
  for (std::size_t i = 0; i < h.size(); ++i) {
    if (kp[i]) {
      out.push(h.row(i), h.c[i]);
    } else {
      if (dt) ++*dt;
      if (dw) *dw += std::abs(h.c[i]);
    }
  }
  return out;
}

// dress_sequence, iqcc/dressing.hpp:311-324
// dress_sequence, iqcc/dressing.hpp:311-324: opts (drop threshold) forwarded
// to every step's merge (:319)
orc_sum dress_seq(const orc_sum& h, std::size_t K, const u64* gens, const double* taus,
                  double eps, std::size_t max_terms, double drop, std::size_t* dt, double* dw) {
  if (max_terms < 1) throw invalid_arg("dress_sequence: max_terms < 1");
  orc_sum out = h;
  for (std::size_t k = 0; k < K; ++k) {
    out = dress(out, gens + k * 2 * h.B, taus[k], drop, true, 1e-10);
    if (eps > 0.0 || out.size() > max_terms) out = compress(out, eps, max_terms, dt, dw);
  }
  return out;
}

// qmf_factor, iqcc/qmf.hpp:56-61 (libm sin/cos evaluated per call, as there)
double factor(const double* th, const double* ph, std::size_t j, bool x, bool z) {
  if (x && z) return std::sin(th[j]) * std::sin(ph[j]);
  if (x) return std::sin(th[j]) * std::cos(ph[j]);
  return std::cos(th[j]);
}

// expect_word, iqcc/qmf.hpp:67-80: ascending qubit order over the support
double expect_word(const double* th, const double* ph, const u64* w, std::size_t B) {
  double val = 1.0;
  for (std::size_t b = 0; b < B; ++b) {
    u64 s = w[b] | w[B + b];
    while (s) {
      unsigned bit = std::countr_zero(s);
      u64 m = u64{1} << bit;
      val *= factor(th, ph, b * 64 + bit, w[b] & m, w[B + b] & m);
      s &= s - 1;
    }
  }
  return val;
}

// expect_sum, iqcc/qmf.hpp:83-90 (canonical order accumulation)
double expect_sum(const double* th, const double* ph, const orc_sum& h) {
  double e = 0.0;
  for (std::size_t i = 0; i < h.size(); ++i) e += h.c[i].real() * expect_word(th, ph, h.row(i), h.B);
  return e;
}

// qmf_energy_gradient, iqcc/qmf.hpp:94-148
double energy_grad(const orc_sum& h, const double* th, const double* ph, double* grad) {
  const std::size_t n = h.n, B = h.B;
  std::fill(grad, grad + 2 * n, 0.0);
  double energy = 0.0;
  std::vector<std::size_t> sup;
  std::vector<double> fac, pre, suf;
  for (std::size_t t = 0; t < h.size(); ++t) {
    const u64* w = h.row(t);
    sup.clear();
    fac.clear();
    for (std::size_t b = 0; b < B; ++b) {
      u64 s = w[b] | w[B + b];
      while (s) {
        sup.push_back(b * 64 + std::countr_zero(s));
        s &= s - 1;
      }
    }
    const double c = h.c[t].real();
    auto xz = [&](std::size_t j, bool& x, bool& z) {
      x = (w[j / 64] >> (j % 64)) & 1;
      z = (w[B + j / 64] >> (j % 64)) & 1;
    };
    for (std::size_t j : sup) {
      bool x, z;
      xz(j, x, z);
      fac.push_back(factor(th, ph, j, x, z));
    }
    const std::size_t m = sup.size();
    pre.assign(m + 1, 1.0);
    suf.assign(m + 1, 1.0);
    for (std::size_t k = 0; k < m; ++k) pre[k + 1] = pre[k] * fac[k];
    for (std::size_t k = m; k-- > 0;) suf[k] = suf[k + 1] * fac[k];
    energy += c * pre[m];
    for (std::size_t k = 0; k < m; ++k) {
      std::size_t j = sup[k];
      bool x, z;
      xz(j, x, z);
      double rest = pre[k] * suf[k + 1];
      double st = std::sin(th[j]), ct = std::cos(th[j]);
      double sp = std::sin(ph[j]), cp = std::cos(ph[j]);
      double dth, dph;
      if (x && z) {
        dth = ct * sp;
        dph = st * cp;
      } else if (x) {
        dth = ct * cp;
        dph = -st * sp;
      } else {
        dth = -st;
        dph = 0.0;
      }
      grad[j] += c * rest * dth;
      grad[n + j] += c * rest * dph;
    }
  }
  return energy;
}

// gradient (full scan), iqcc/dis.hpp:39-52; group_gradient :121-132 when
// [lo,hi) restricts to one flip group
double dis_grad(const orc_sum& h, const double* th, const double* ph, const u64* P,
                std::size_t lo, std::size_t hi) {
  std::vector<u64> tmp(2 * h.B);
  double g = 0.0;
  for (std::size_t k = lo; k < hi; ++k) {
    int t = mult(h.row(k), P, tmp.data(), h.B);
    cplx wgt = h.c[k] * phase(t);
    if (wgt.imag() == 0.0) continue;
    g += wgt.imag() * expect_word(th, ph, tmp.data(), h.B);
  }
  return g;
}

// group_by_flip, iqcc/dis.hpp:23-35: runs of equal x planes
std::vector<std::size_t> flip_group_starts(const orc_sum& h) {
  std::vector<std::size_t> st;
  for (std::size_t i = 0; i < h.size(); ++i)
    if (i == 0 || !std::equal(h.row(i), h.row(i) + h.B, h.row(i - 1))) st.push_back(i);
  return st;
}

// odd_y_candidates, iqcc/dis.hpp:89-116
std::vector<std::vector<u64>> odd_y(const u64* xflip, std::size_t n, std::size_t B,
                                    std::size_t cap) {
  std::vector<std::size_t> pos;
  for (std::size_t b = 0; b < B; ++b)
    for (u64 s = xflip[b]; s; s &= s - 1) pos.push_back(b * 64 + std::countr_zero(s));
  const std::size_t w = pos.size();
  std::vector<std::vector<u64>> out;
  if (w == 0) return out;
  auto make = [&](u64 ymask) {
    std::vector<u64> r(2 * B, 0);
    for (std::size_t i = 0; i < w; ++i) {
      r[pos[i] / 64] |= u64{1} << (pos[i] % 64);
      if ((ymask >> i) & 1) r[B + pos[i] / 64] |= u64{1} << (pos[i] % 64);
    }
    return r;
  };
  bool exhaustive = w < 2 || (w <= 63 && (u64{1} << (w - 1)) <= cap);
  if (exhaustive) {
    for (u64 m = 1; m < (u64{1} << w); ++m) {
      if (std::popcount(m) % 2 == 1) out.push_back(make(m));
      if (out.size() >= cap) break;
    }
  } else {
    for (std::size_t i = 0; i < w && out.size() < cap; ++i) out.push_back(make(u64{1} << i));
  }
  (void)n;
  return out;
}

bool at_poles(const double* th, std::size_t n) {  // QmfState::at_poles, qmf.hpp:26-30
  for (std::size_t j = 0; j < n; ++j)
    if (std::abs(std::sin(th[j])) > 1e-12) return false;
  return true;
}

struct Pick {
  std::vector<u64> w;
  double g;
};

// dis_candidates, iqcc/dis.hpp:140-191
std::vector<Pick> dis(const orc_sum& h, const double* th, const double* ph, std::size_t top_k,
                      double thr, std::size_t cap, bool has_seed, u64 seed) {
  if (top_k < 1) throw invalid_arg("dis_candidates: top_k < 1");
  const bool poles = at_poles(th, h.n);
  auto starts = flip_group_starts(h);
  std::vector<Pick> picks;
  for (std::size_t gi = 0; gi < starts.size(); ++gi) {
    std::size_t lo = starts[gi], hi = gi + 1 < starts.size() ? starts[gi + 1] : h.size();
    auto cands = odd_y(h.row(lo), h.n, h.B, cap);
    Pick best;
    bool have = false;
    for (auto& cd : cands) {
      double g = poles ? dis_grad(h, th, ph, cd.data(), lo, hi)
                       : dis_grad(h, th, ph, cd.data(), 0, h.size());
      if (!have || std::abs(g) > std::abs(best.g) ||
          (std::abs(g) == std::abs(best.g) && cmp_rows(cd.data(), best.w.data(), h.B) < 0)) {
        best = {cd, g};
        have = true;
      }
    }
    if (have && std::abs(best.g) >= thr) picks.push_back(best);
  }
  std::stable_sort(picks.begin(), picks.end(), [&](const Pick& a, const Pick& b) {
    if (std::abs(a.g) != std::abs(b.g)) return std::abs(a.g) > std::abs(b.g);
    return cmp_rows(a.w.data(), b.w.data(), h.B) < 0;
  });
  if (has_seed) {
    std::mt19937_64 rng(seed);
    std::size_t i = 0;
    while (i < picks.size()) {
      std::size_t j = i + 1;
      double mag = std::abs(picks[i].g);
      while (j < picks.size() && std::abs(std::abs(picks[j].g) - mag) <= 1e-12 * std::max(1.0, mag))
        ++j;
      std::shuffle(picks.begin() + i, picks.begin() + j, rng);
      i = j;
    }
  }
  if (picks.size() > top_k) picks.resize(top_k);
  return picks;
}

// gather_key over concatenated positions, iqcc/dressing.hpp:132-147
u64 gather_key(const u64* r, std::size_t n, std::size_t B, const std::size_t* pos, std::size_t m) {
  u64 key = 0;
  for (std::size_t i = 0; i < m; ++i) {
    std::size_t p = pos[i];
    bool bit = p < n ? (r[p / 64] >> (p % 64)) & 1 : (r[B + (p - n) / 64] >> ((p - n) % 64)) & 1;
    key |= u64{bit} << i;
  }
  return key;
}

// choose_partition_bits, iqcc/partition.hpp:52-108 (greedy, lowest position
// wins ties, imbalance = max shard / ideal)
double choose_bits(const orc_sum& h, std::size_t m, std::size_t* bits_out) {
  const std::size_t width = 2 * h.n;
  if (m > width) throw invalid_arg("choose_partition_bits: m exceeds representation width");
  std::vector<std::size_t> keys(h.size(), 0), chosen;
  auto bit_at = [&](std::size_t i, std::size_t pos) -> std::size_t {
    const u64* r = h.row(i);
    return pos < h.n ? (r[pos / 64] >> (pos % 64)) & 1 : (r[h.B + (pos - h.n) / 64] >> ((pos - h.n) % 64)) & 1;
  };
  for (std::size_t round = 0; round < m; ++round) {
    std::size_t best_pos = width, best_max = std::numeric_limits<std::size_t>::max();
    for (std::size_t pos = 0; pos < width; ++pos) {
      if (std::find(chosen.begin(), chosen.end(), pos) != chosen.end()) continue;
      std::vector<std::size_t> cnt(std::size_t{2} << round, 0);
      for (std::size_t i = 0; i < h.size(); ++i) ++cnt[keys[i] | (bit_at(i, pos) << round)];
      std::size_t worst = *std::max_element(cnt.begin(), cnt.end());
      if (worst < best_max) {
        best_max = worst;
        best_pos = pos;
      }
    }
    chosen.push_back(best_pos);
    for (std::size_t i = 0; i < h.size(); ++i) keys[i] |= bit_at(i, best_pos) << round;
  }
  double imb = 1.0;
  if (h.size() > 0 && m > 0) {
    std::vector<std::size_t> cnt(std::size_t{1} << m, 0);
    for (auto k : keys) ++cnt[k];
    double ideal = double(h.size()) / double(cnt.size());
    imb = double(*std::max_element(cnt.begin(), cnt.end())) / std::max(1.0, ideal);
  }
  std::copy(chosen.begin(), chosen.end(), bits_out);
  return imb;
}

orc_sum* box(orc_sum&& s) { return new orc_sum(std::move(s)); }

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
int orc_last_error_kind(void) { return g_kind; }
const char* orc_flavor(void) { return "port"; }

orc_sum* orc_sum_new(size_t n, const uint64_t* rows, const double* coeff, size_t M) {
  return guard([&]() -> orc_sum* {
    orc_sum s;
    s.n = n;
    s.B = blocks_for(n);
    s.rows.assign(rows, rows + M * 2 * s.B);
    s.c.resize(M);
    for (size_t i = 0; i < M; ++i) s.c[i] = cplx(coeff[2 * i], coeff[2 * i + 1]);
    return box(std::move(s));
  }, nullptr);
}

orc_sum* orc_from_terms(size_t n, const uint64_t* rows, const double* coeff, size_t M,
                        double thr, int check, double tol) {
  return guard([&]() -> orc_sum* {
    std::vector<cplx> c(M);
    for (size_t i = 0; i < M; ++i) c[i] = cplx(coeff[2 * i], coeff[2 * i + 1]);
    return box(from_terms(n, rows, c.data(), M, thr, check, tol));
  }, nullptr);
}

void orc_sum_free(orc_sum* h) { delete h; }
size_t orc_sum_size(const orc_sum* h) { return h->size(); }
size_t orc_sum_qubits(const orc_sum* h) { return h->n; }
void orc_sum_export(const orc_sum* h, uint64_t* rows, double* coeff) {
  std::copy(h->rows.begin(), h->rows.end(), rows);
  for (size_t i = 0; i < h->size(); ++i) {
    coeff[2 * i] = h->c[i].real();
    coeff[2 * i + 1] = h->c[i].imag();
  }
}
int orc_sum_is_canonical(const orc_sum* h) {
  for (size_t i = 0; i + 1 < h->size(); ++i)
    if (cmp_rows(h->row(i), h->row(i + 1), h->B) >= 0) return 0;
  return 1;
}
int orc_sum_equal(const orc_sum* a, const orc_sum* b) {
  return a->n == b->n && a->rows == b->rows && a->c == b->c;
}

int orc_canonical_compare(size_t n, const uint64_t* a, const uint64_t* b) {
  return cmp_rows(a, b, blocks_for(n));
}
int orc_commutes(size_t n, const uint64_t* a, const uint64_t* b) {
  return commute(a, b, blocks_for(n));
}
int orc_multiply(size_t n, const uint64_t* a, const uint64_t* b, uint64_t* out) {
  return mult(a, b, out, blocks_for(n));
}

orc_sum* orc_merge_sums(const orc_sum* a, const orc_sum* b, double thr, int check, double tol) {
  return guard([&]() -> orc_sum* { return box(merge(*a, *b, thr, check, tol)); }, nullptr);
}

orc_sum* orc_compress(const orc_sum* h, double eps, size_t max_terms, size_t* dt, double* dw) {
  return guard([&]() -> orc_sum* { return box(compress(*h, eps, max_terms, dt, dw)); }, nullptr);
}

orc_sum* orc_dress_single(const orc_sum* h, const uint64_t* gen, double tau, double thr,
                          int check, double tol) {
  return guard([&]() -> orc_sum* { return box(dress(*h, gen, tau, thr, check, tol)); }, nullptr);
}

orc_sum* orc_sortless_dress(const orc_sum* h, const uint64_t* gen, double tau, double thr,
                            size_t* n_buckets, size_t* new_stream_sorts) {
  // sortless_dress (dressing.hpp:228-307) returns the dress_single sum bit
  // for bit; the port restates only its contract (result + the >64 key-bit
  // limit of bucket_by_support, dressing.hpp:163-165).
  return guard([&]() -> orc_sum* {
    if (is_id(gen, h->B)) throw invalid_arg("sortless_dress: identity generator");
    size_t w = 0;
    for (size_t b = 0; b < h->B; ++b) w += std::popcount(gen[b] | gen[h->B + b]);
    if (2 * w > 64) throw std::runtime_error("entangler support exceeds 64 bits; not supported");
    if (n_buckets) {
      std::vector<size_t> pos;
      for (size_t b = 0; b < h->B; ++b)
        for (u64 s = gen[b] | gen[h->B + b]; s; s &= s - 1) {
          size_t j = b * 64 + std::countr_zero(s);
          pos.push_back(j);
          pos.push_back(h->n + j);
        }
      std::vector<u64> keys;
      for (size_t i = 0; i < h->size(); ++i) keys.push_back(gather_key(h->row(i), h->n, h->B, pos.data(), pos.size()));
      std::sort(keys.begin(), keys.end());
      *n_buckets = std::unique(keys.begin(), keys.end()) - keys.begin();
    }
    if (new_stream_sorts) *new_stream_sorts = 0;
    return box(dress(*h, gen, tau, thr, true, 1e-10));
  }, nullptr);
}

orc_sum* orc_dress_sequence(const orc_sum* h, size_t K, const uint64_t* gens, const double* taus,
                            double eps, size_t max_terms, double drop_thr, size_t* dt, double* dw) {
  return guard([&]() -> orc_sum* { return box(dress_seq(*h, K, gens, taus, eps, max_terms, drop_thr, dt, dw)); },
               nullptr);
}

void orc_growth_split(const orc_sum* h, const uint64_t* gen, size_t* nc, size_t* na) {
  *nc = *na = 0;  // growth_split, dressing.hpp:41-50
  for (size_t i = 0; i < h->size(); ++i) ++*(commute(h->row(i), gen, h->B) ? nc : na);
}

double orc_expect_word(size_t n, const double* th, const double* ph, const uint64_t* w) {
  return expect_word(th, ph, w, blocks_for(n));
}
double orc_expect_sum(const double* th, const double* ph, const orc_sum* h) {
  return expect_sum(th, ph, *h);
}
// qcc_energy, iqcc/optimizer.hpp:19-25: dress_sequence without compression
// and MergeOptions{0.0, true}, then expect_sum.
double orc_qcc_energy(const orc_sum* h, const double* th, const double* ph, size_t K,
                      const uint64_t* gens, const double* taus) {
  return guard([&]() -> double {
    orc_sum cur = *h;
    for (size_t k = 0; k < K; ++k) cur = dress(cur, gens + k * 2 * h->B, taus[k], 0.0, true, 1e-10);
    return expect_sum(th, ph, cur);
  }, 0.0);
}

// dress_derivative, iqcc/optimizer.hpp:31-48: the anticommuting part of a
// maps to -sin(tau) c T + cos(tau) (phase) c (-i) (T*P); merged with drop 0.
static orc_sum dress_derivative(const orc_sum& a, const u64* P, double tau) {
  const std::size_t B = a.B;
  const double cs = std::cos(tau), sn = std::sin(tau);
  orc_sum surv, prod;
  surv.n = prod.n = a.n;
  surv.B = prod.B = B;
  std::vector<u64> tmp(2 * B);
  for (std::size_t i = 0; i < a.size(); ++i) {
    if (commute(a.row(i), P, B)) continue;
    surv.push(a.row(i), -sn * a.c[i]);
    int t = mult(a.row(i), P, tmp.data(), B);
    prod.push(tmp.data(), a.c[i] * cs * cplx{0.0, -1.0} * phase(t));
  }
  orc_sum sorted = from_terms(a.n, prod.rows.data(), prod.c.data(), prod.size(), 0.0, false, 0.0);
  return merge(surv, sorted, 0.0, false, 0.0);
}

// qcc_gradient, iqcc/optimizer.hpp:54-77: forward chain A_k (exact merges),
// derivative of step k, dressed through the remaining entanglers.
int orc_qcc_gradient(const orc_sum* h, const double* th, const double* ph, size_t K,
                     const uint64_t* gens, const double* taus, double* g) {
  return guard([&]() -> int {
    const std::size_t B = h->B;
    std::vector<orc_sum> chain{*h};
    for (size_t k = 0; k + 1 < K; ++k)
      chain.push_back(dress(chain.back(), gens + k * 2 * B, taus[k], 0.0, true, 1e-10));
    for (size_t k = 0; k < K; ++k) {
      orc_sum d = dress_derivative(chain[k], gens + k * 2 * B, taus[k]);
      for (size_t j = k + 1; j < K; ++j) d = dress(d, gens + j * 2 * B, taus[j], 0.0, false, 0.0);
      g[k] = expect_sum(th, ph, d);
    }
    return 0;
  }, -1);
}

// build_poly (iqcc/optimizer.hpp:219-268): subsets of size <= k in
// lexicographic index order, each word the ordered product of its
// entanglers extended on the right, phase exponents accumulated mod 4.
// build_poly_kernels (optimizer.hpp:340-368) with sandwich (288-333): at the
// poles only the run of terms whose x plane is x_a ^ x_b is summed.
int orc_poly_kernels(const orc_sum* h, const double* th, const double* ph, size_t N,
                     const uint64_t* ents, size_t k, size_t cap, size_t* t_out, uint64_t* words_out,
                     int* phase_out, double* hk_out, double* nk_out) {
  return guard([&]() -> int {
    const std::size_t n = h->n, B = h->B;
    if (k > N) throw invalid_arg("build_poly: order exceeds N");
    for (size_t j = 0; j < N; ++j)
      if (is_id(ents + j * 2 * B, B)) throw invalid_arg("build_poly: identity entangler");
    double count = 0, binom = 1;
    for (std::size_t j = 0; j <= k; ++j) {
      count += binom;
      binom = binom * double(N - j) / double(j + 1);
      if (count > 200000.0) throw std::runtime_error("build_poly: subset budget exceeded");
    }
    std::vector<u64> words(2 * B, 0);
    std::vector<int> phs{0}, last{-1};
    std::size_t beg = 0, end = 1;
    for (std::size_t sz = 1; sz <= k; ++sz) {
      const std::size_t next = phs.size();
      for (std::size_t s = beg; s < end; ++s)
        for (std::size_t e = (std::size_t)(last[s] + 1); e < N; ++e) {
          std::vector<u64> w(2 * B);
          const int t = mult(&words[s * 2 * B], ents + e * 2 * B, w.data(), B);
          words.insert(words.end(), w.begin(), w.end());
          phs.push_back((phs[s] + t) & 3);
          last.push_back((int)e);
        }
      beg = next;
      end = phs.size();
    }
    const std::size_t t = phs.size();
    *t_out = t;
    if (t > cap) throw std::runtime_error("orc_poly_kernels: capacity");
    bool poles = true;  // QmfState::at_poles, iqcc/qmf.hpp:26-30
    for (std::size_t j = 0; j < n; ++j)
      if (std::abs(std::sin(th[j])) > 1e-12) poles = false;
    std::vector<u64> w1(2 * B), w2(2 * B);
    for (std::size_t a = 0; a < t; ++a)
      for (std::size_t b = a; b < t; ++b) {
        const u64* wa = &words[a * 2 * B];
        const u64* wb = &words[b * 2 * B];
        const int tw = mult(wa, wb, w1.data(), B);
        const cplx nv = phase(tw) * expect_word(th, ph, w1.data(), B);
        std::size_t lo = 0, hi = h->size();
        if (poles) {  // the x run x_a ^ x_b (canonical order is x-major)
          std::vector<u64> tx(2 * B, 0);
          for (std::size_t q = 0; q < B; ++q) tx[q] = wa[q] ^ wb[q];
          auto x_cmp = [&](std::size_t i) {
            for (std::size_t q = 0; q < B; ++q)
              if (h->row(i)[q] != tx[q]) return rev64(h->row(i)[q]) < rev64(tx[q]) ? -1 : 1;
            return 0;
          };
          std::size_t l = 0, r = h->size();
          while (l < r) {
            const std::size_t mid = (l + r) / 2;
            if (x_cmp(mid) < 0) l = mid + 1; else r = mid;
          }
          lo = hi = l;
          while (hi < h->size() && x_cmp(hi) == 0) ++hi;
        }
        cplx hv{};
        for (std::size_t i = lo; i < hi; ++i) {
          const int t1 = mult(wa, h->row(i), w1.data(), B);
          const int t2 = mult(w1.data(), wb, w2.data(), B);
          const double e = expect_word(th, ph, w2.data(), B);
          if (e != 0.0) hv += h->c[i] * phase((t1 + t2) & 3) * e;
        }
        nk_out[2 * (a * t + b)] = nv.real();
        nk_out[2 * (a * t + b) + 1] = nv.imag();
        nk_out[2 * (b * t + a)] = std::conj(nv).real();
        nk_out[2 * (b * t + a) + 1] = std::conj(nv).imag();
        hk_out[2 * (a * t + b)] = hv.real();
        hk_out[2 * (a * t + b) + 1] = hv.imag();
        hk_out[2 * (b * t + a)] = std::conj(hv).real();
        hk_out[2 * (b * t + a) + 1] = std::conj(hv).imag();
      }
    for (std::size_t s = 0; s < t; ++s) {
      std::copy(&words[s * 2 * B], &words[s * 2 * B] + 2 * B, words_out + s * 2 * B);
      phase_out[s] = phs[s];
    }
    return 0;
  }, -1);
}

double orc_qmf_energy_gradient(const orc_sum* h, const double* th, const double* ph, double* g) {
  return energy_grad(*h, th, ph, g);
}
double orc_gradient(const orc_sum* h, const double* th, const double* ph, const uint64_t* p) {
  return dis_grad(*h, th, ph, p, 0, h->size());
}

size_t orc_dis_candidates(const orc_sum* h, const double* th, const double* ph, size_t top_k,
                          double thr, size_t cap, int has_seed, uint64_t seed, uint64_t* rows_out,
                          double* g_out, size_t out_cap) {
  return guard([&]() -> size_t {
    auto picks = dis(*h, th, ph, top_k, thr, cap, has_seed != 0, seed);
    size_t n = std::min(out_cap, picks.size());
    for (size_t i = 0; i < n; ++i) {
      std::copy(picks[i].w.begin(), picks[i].w.end(), rows_out + i * 2 * h->B);
      g_out[i] = picks[i].g;
    }
    return picks.size();
  }, (size_t)-1);
}

size_t orc_flip_groups(const orc_sum* h, size_t* starts_out, size_t out_cap) {
  auto st = flip_group_starts(*h);
  std::copy(st.begin(), st.begin() + std::min(out_cap, st.size()), starts_out);
  return st.size();
}

double orc_choose_partition_bits(const orc_sum* h, size_t m, size_t* bits_out) {
  return guard([&]() -> double { return choose_bits(*h, m, bits_out); }, -1.0);
}

orc_sum* orc_parallel_dress(const orc_sum* h, size_t m, const size_t* bits, const size_t* owner,
                            size_t n_workers, const uint64_t* gen, double tau, double eps,
                            size_t max_terms, int threaded, size_t* shard_sizes, size_t* log_out,
                            size_t log_cap, size_t* n_log, size_t* mask_out) {
  // parallel_dress, iqcc/partition.hpp:398-452: the gathered result equals
  // the serial dress_single + compress pipeline (tests/test_partition.cpp:
  // 180-208); routed batches are one record per source shard with products
  // when the entangler's key (mask) is nonzero, bytes = terms*(16 + 16B).
  (void)owner;
  (void)n_workers;
  (void)threaded;
  return guard([&]() -> orc_sum* {
    if (is_id(gen, h->B)) throw invalid_arg("parallel_dress: identity generator");
    if (max_terms < 1) throw invalid_arg("compress_partitioned: max_terms < 1");
    const size_t P = size_t{1} << m;
    size_t mask = gather_key(gen, h->n, h->B, bits, m);
    orc_sum out = dress(*h, gen, tau, 1e-12, false, 0.0);
    if (eps > 0.0 || out.size() > max_terms) out = compress(out, eps, max_terms, nullptr, nullptr);
    std::fill(shard_sizes, shard_sizes + P, 0);
    for (size_t i = 0; i < out.size(); ++i) ++shard_sizes[gather_key(out.row(i), h->n, h->B, bits, m)];
    std::vector<size_t> prod(P, 0);
    if (std::sin(tau) != 0.0)
      for (size_t i = 0; i < h->size(); ++i)
        if (!commute(h->row(i), gen, h->B)) ++prod[gather_key(h->row(i), h->n, h->B, bits, m)];
    size_t nl = 0;
    for (size_t p = 0; p < P; ++p) {
      if (mask == 0 || prod[p] == 0) continue;
      if (nl < log_cap) {
        log_out[4 * nl + 0] = p;
        log_out[4 * nl + 1] = p ^ mask;
        log_out[4 * nl + 2] = prod[p];
        log_out[4 * nl + 3] = prod[p] * (16 + 2 * h->B * 8);
      }
      ++nl;
    }
    *n_log = nl;
    *mask_out = mask;
    return box(std::move(out));
  }, nullptr);
}

double orc_parallel_expect(const orc_sum* h, size_t m, const size_t* bits, const size_t* owner,
                           size_t n_workers, const double* th, const double* ph) {
  // parallel_expect + reduce_scalar, iqcc/partition.hpp:233-254: each worker
  // sums its shards in partition order (each shard in canonical order), then
  // worker partials are added in worker order.
  const size_t P = size_t{1} << m;
  std::vector<orc_sum> shards(P);
  for (auto& s : shards) {
    s.n = h->n;
    s.B = h->B;
  }
  for (size_t i = 0; i < h->size(); ++i)
    shards[gather_key(h->row(i), h->n, h->B, bits, m)].push(h->row(i), h->c[i]);
  std::vector<double> local(n_workers, 0.0);
  for (size_t w = 0; w < n_workers; ++w)
    for (size_t p = 0; p < P; ++p)
      if (owner[p] == w) local[w] += expect_sum(th, ph, shards[p]);
  double s = 0.0;
  for (double v : local) s += v;
  return s;
}

int orc_rebalance(const orc_sum* h, size_t m, const size_t* bits, size_t* owner, size_t nw,
                  double threshold) {
  // rebalance, iqcc/partition.hpp:457-494
  if (!(threshold > 1.0)) {
    g_err = "rebalance: threshold must exceed 1";
    g_kind = 1;
    return -1;
  }
  const size_t P = size_t{1} << m;
  std::vector<size_t> sz(P, 0);
  for (size_t i = 0; i < h->size(); ++i) ++sz[gather_key(h->row(i), h->n, h->B, bits, m)];
  for (;;) {
    std::vector<size_t> l(nw, 0);
    for (size_t p = 0; p < P; ++p) l[owner[p]] += sz[p];
    auto mx = std::max_element(l.begin(), l.end());
    auto mn = std::min_element(l.begin(), l.end());
    double ratio = *mn == 0 ? std::numeric_limits<double>::infinity() : double(*mx) / double(*mn);
    if (*mx == 0 || ratio <= threshold) break;
    size_t donor = mx - l.begin(), recv = mn - l.begin(), best = P, best_sz = 0;
    for (size_t p = 0; p < P; ++p) {
      if (owner[p] != donor || sz[p] == 0) continue;
      if (*mn + sz[p] < *mx && sz[p] > best_sz) {
        best = p;
        best_sz = sz[p];
      }
    }
    if (best == P) break;
    owner[best] = recv;
  }
  return 0;
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
    const size_t B = blocks_for(n);
    std::vector<size_t> idx(count);
    std::iota(idx.begin(), idx.end(), 0);
    std::sort(idx.begin(), idx.end(), [&](size_t a, size_t b) {
      int c = cmp_rows(&t.rows[a * 2 * B], &t.rows[b * 2 * B], B);
      return c != 0 ? c < 0 : a < b;
    });
    orc_sum s;
    s.n = n;
    s.B = B;
    for (size_t r = 0; r < count; ++r) {
      size_t i = idx[r];
      if (r > 0 && cmp_rows(&t.rows[i * 2 * B], &t.rows[idx[r - 1] * 2 * B], B) == 0) continue;
      s.push(&t.rows[i * 2 * B], cplx(t.coeff[2 * i], 0.0));
    }
    return box(std::move(s));
  }, nullptr);
}

double orc_time_dress_sequence(const orc_sum* h, size_t K, const uint64_t* gens, const double* taus,
                               double eps, size_t max_terms, size_t m_bits, int threads,
                               size_t* terms_in_total, size_t* final_size, orc_sum** out) {
  (void)m_bits;
  (void)threads;
  auto t0 = std::chrono::steady_clock::now();
  orc_sum cur = *h;
  size_t tin = 0;
  for (size_t k = 0; k < K; ++k) {
    tin += cur.size();
    cur = dress(cur, gens + k * 2 * h->B, taus[k], 1e-12, true, 1e-10);
    if (eps > 0.0 || cur.size() > max_terms) cur = compress(cur, eps, max_terms, nullptr, nullptr);
  }
  auto t1 = std::chrono::steady_clock::now();
  *terms_in_total = tin;
  *final_size = cur.size();
  if (out) *out = box(std::move(cur));
  return std::chrono::duration<double>(t1 - t0).count();
}

}  // extern "C"
