/* oracle_api.h — C interface shared by the two CPU checkers in oracle/.
 *
 * TEST INFRASTRUCTURE ONLY.  Two shared libraries export exactly these
 * symbols:
 *   oracle/liboracle.so        — iqcc_oracle.cpp, our restatement ("port") of
 *                                 the reference algorithms, citing file:line;
 *   oracle/_ref/libiqcc_ref.so — ref_capi.cpp compiled against the UNMODIFIED
 *                                 reference headers under /root/reference
 *                                 (built here only; never shipped).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm load them.  The product (paper_2603_08883_b200/) never does.
 *
 * Layout (identical to iqcc::PauliSum storage, iqcc/pauli.hpp:373-377):
 *   rows  : [M][2B] uint64, x blocks then z blocks, bit j%64 of block j/64 = qubit j
 *   coeff : [M][2]  double, (re, im)
 * Errors: functions returning a handle return NULL and set orc_last_error();
 * the error kind is 1 = invalid_argument, 2 = runtime_error.
 */
#ifndef IQCC_ORACLE_API_H
#define IQCC_ORACLE_API_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_sum orc_sum;
typedef struct orc_rng orc_rng;

const char* orc_last_error(void);
int orc_last_error_kind(void);
const char* orc_flavor(void); /* "port" or "reference" */

/* container ------------------------------------------------------------ */
orc_sum* orc_sum_new(size_t n_qubits, const uint64_t* rows, const double* coeff, size_t M);
orc_sum* orc_from_terms(size_t n_qubits, const uint64_t* rows, const double* coeff, size_t M,
                        double drop_thr, int check_herm, double herm_tol);
void orc_sum_free(orc_sum* h);
size_t orc_sum_size(const orc_sum* h);
size_t orc_sum_qubits(const orc_sum* h);
void orc_sum_export(const orc_sum* h, uint64_t* rows, double* coeff);
int orc_sum_is_canonical(const orc_sum* h);
int orc_sum_equal(const orc_sum* a, const orc_sum* b);

/* algebra (iqcc/pauli.hpp) ---------------------------------------------- */
int orc_canonical_compare(size_t n_qubits, const uint64_t* a, const uint64_t* b);
int orc_commutes(size_t n_qubits, const uint64_t* a, const uint64_t* b);
int orc_multiply(size_t n_qubits, const uint64_t* a, const uint64_t* b, uint64_t* out);
orc_sum* orc_merge_sums(const orc_sum* a, const orc_sum* b, double drop_thr, int check_herm,
                        double herm_tol);
orc_sum* orc_compress(const orc_sum* h, double eps, size_t max_terms, size_t* dropped_terms,
                      double* dropped_weight);

/* dressing (iqcc/dressing.hpp) ------------------------------------------ */
orc_sum* orc_dress_single(const orc_sum* h, const uint64_t* gen, double tau, double drop_thr,
                          int check_herm, double herm_tol);
orc_sum* orc_sortless_dress(const orc_sum* h, const uint64_t* gen, double tau, double drop_thr,
                            size_t* n_buckets, size_t* new_stream_sorts);
orc_sum* orc_dress_sequence(const orc_sum* h, size_t K, const uint64_t* gens, const double* taus,
                            double eps, size_t max_terms, double drop_thr, size_t* dropped_terms,
                            double* dropped_weight);
void orc_growth_split(const orc_sum* h, const uint64_t* gen, size_t* n_comm, size_t* n_anti);

/* QMF / DIS (iqcc/qmf.hpp, iqcc/dis.hpp) --------------------------------- */
double orc_expect_word(size_t n_qubits, const double* theta, const double* phi, const uint64_t* w);
double orc_expect_sum(const double* theta, const double* phi, const orc_sum* h);
double orc_qmf_energy_gradient(const orc_sum* h, const double* theta, const double* phi,
                               double* grad2n);
double orc_gradient(const orc_sum* h, const double* theta, const double* phi, const uint64_t* p);
/* returns #picks written (<= out_cap); rows_out [cap][2B], g_out [cap] */
size_t orc_dis_candidates(const orc_sum* h, const double* theta, const double* phi,
                          size_t top_k, double screen_thr, size_t per_group_cap,
                          int has_seed, uint64_t seed, uint64_t* rows_out, double* g_out,
                          size_t out_cap);
size_t orc_flip_groups(const orc_sum* h, size_t* starts_out, size_t out_cap);

/* variational energy and amplitude gradient (iqcc/optimizer.hpp:19-77) ---- */
double orc_qcc_energy(const orc_sum* h, const double* theta, const double* phi, size_t K,
                      const uint64_t* gens, const double* taus);
int orc_qcc_gradient(const orc_sum* h, const double* theta, const double* phi, size_t K,
                     const uint64_t* gens, const double* taus, double* grad_out);

/* build_poly + build_poly_kernels (iqcc/optimizer.hpp:219-368): expansion of
 * the N entanglers ents [N][2B] to order k (subset budget 200000); t_out =
 * subset count, words_out [cap][2B] and phase_out [cap] the subsets in
 * build_poly order, hk_out / nk_out [cap*cap][2] the kernels (row stride
 * t).  Returns 0, or -1 on error (orc_last_error). */
int orc_poly_kernels(const orc_sum* h, const double* theta, const double* phi, size_t N,
                     const uint64_t* ents, size_t k, size_t cap, size_t* t_out, uint64_t* words_out,
                     int* phase_out, double* hk_out, double* nk_out);

/* partitioning (iqcc/partition.hpp) --------------------------------------- */
double orc_choose_partition_bits(const orc_sum* h, size_t m, size_t* bits_out);
/* Runs distribute -> parallel_dress -> gather.  shard_sizes_out[2^m];
 * log_out rows of 4 size_t (source, destination, terms, bytes); returns gathered sum. */
orc_sum* orc_parallel_dress(const orc_sum* h, size_t m, const size_t* bits, const size_t* owner,
                            size_t n_workers, const uint64_t* gen, double tau, double eps,
                            size_t max_terms, int threaded, size_t* shard_sizes_out,
                            size_t* log_out, size_t log_cap, size_t* n_log, size_t* mask_out);
double orc_parallel_expect(const orc_sum* h, size_t m, const size_t* bits, const size_t* owner,
                           size_t n_workers, const double* theta, const double* phi);
/* rebalance: owner_inout[2^m] updated in place */
int orc_rebalance(const orc_sum* h, size_t m, const size_t* bits, size_t* owner_inout,
                  size_t n_workers, double threshold);

/* generators ------------------------------------------------------------- */
orc_rng* orc_rng_new(uint64_t seed);
void orc_rng_free(orc_rng* r);
uint64_t orc_rng_next(orc_rng* r);
double orc_rng_uniform(orc_rng* r, double lo, double hi);
void orc_random_word(orc_rng* r, size_t n_qubits, int allow_identity, uint64_t* row_out);
orc_sum* orc_random_sum(orc_rng* r, size_t n_qubits, size_t max_terms);
void orc_random_qmf(orc_rng* r, size_t n_qubits, double* theta, double* phi);
orc_sum* orc_gen_mol(size_t n_qubits, size_t n_terms, uint64_t seed);

/* timing helpers for bench.py's CPU arm (threads = 0 -> hardware) --------- */
double orc_time_dress_sequence(const orc_sum* h, size_t K, const uint64_t* gens,
                               const double* taus, double eps, size_t max_terms, size_t m_bits,
                               int threads, size_t* terms_in_total, size_t* final_size,
                               orc_sum** out /* nullable: the final sum (gathered) */);

#ifdef __cplusplus
}
#endif
#endif
