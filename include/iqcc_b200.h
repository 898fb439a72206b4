/* iqcc_b200.h — C-ABI of the B200 engine for the iQCC dressing hot path
 * (arXiv 2603.08883).  Plain pointers and sizes only; no torch or CUDA types.
 *
 * The reference (/root/reference/proj, header-only C++20) has no FFI; its
 * boundary is the C++ API in namespace iqcc.  Each entry point below names
 * the reference function it replaces.  The C++ shim
 * include/iqcc_b200/iqcc_gpu.hpp re-exposes these with the reference's exact
 * signatures (iqcc::gpu::dress_single, ...), rethrowing the same exception
 * types from the status codes.
 *
 * Host data layout at this boundary is the reference's PauliSum storage
 * (iqcc/pauli.hpp:373-377): rows [M][2B] uint64 (x blocks then z blocks,
 * bit j%64 of block j/64 = qubit j), coefficients [M][2] double (re, im),
 * canonical order (iqcc/pauli.hpp:146-161), duplicate free.  Coefficients
 * must be real (im == 0): JW Hamiltonians and everything dressing produces
 * from them are; nonzero im is rejected with
 * IQCC_EINVAL rather than silently dropped.
 *
 * Device layout: per sum one array of key rows [M][2B]
 * uint64 holding the bit-REVERSED words (so canonical order is plain
 * lexicographic unsigned order) and one fp64 coefficient array [M].
 *
 * Status codes: 0 ok; IQCC_EINVAL ~ std::invalid_argument;
 * IQCC_ERUNTIME ~ std::runtime_error; IQCC_ECUDA / IQCC_ENOMEM device errors.
 * iqcc_gpu_last_error() returns the message of the last failure on the
 * calling thread.  Handles are not thread safe; one host thread per device.
 */
#ifndef IQCC_B200_H
#define IQCC_B200_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum {
  IQCC_OK = 0,
  IQCC_EINVAL = 1,
  IQCC_ERUNTIME = 2,
  IQCC_ECUDA = 3,
  IQCC_ENOMEM = 4
};

typedef struct iqcc_gpu_sum iqcc_gpu_sum;

/* ---- engine ---------------------------------------------------------- */
const char* iqcc_gpu_last_error(void);
/* Binds the calling thread to `device` and creates the engine context.
 * Contexts are per host thread (own stream, scratch, block cache and
 * page-locked staging); a handle is used from the thread that created it.
 * Several threads, each with its own context, run their calls concurrently
 * on one device (bench.py's e2e keeps three upload/dress/download calls in
 * flight this way). */
int iqcc_gpu_init(int device);
/* Run all engine work on an existing cudaStream_t (e.g. torch's current
 * stream) instead of the engine's own; NULL restores the default. */
int iqcc_gpu_set_stream(void* cuda_stream);
/* Releases the calling thread's context (device memory, caches, staging). */
int iqcc_gpu_finalize(void);
/* Number of engine kernel launches so far (bench.py's gpu_launches). */
uint64_t iqcc_gpu_launch_count(void);
/* Per-kernel CUDA-event timing (off by default): enable, then query the
 * accumulated milliseconds and launch count of a kernel family by name
 * ("merge", "classify", "rank", "partition", "select", "expect", ...). */
int iqcc_gpu_profile_enable(int on);
int iqcc_gpu_profile_get(const char* name, double* total_ms, uint64_t* launches);
int iqcc_gpu_profile_reset(void);
/* Algorithmic bytes attributed to a family while profiling is enabled
 * ("merge": (M_in + M_out) * (16B + 8) per dressing step). */
int iqcc_gpu_profile_bytes(const char* name, double* bytes);

/* ---- sums (replace iqcc::PauliSum storage, iqcc/pauli.hpp:245-378) ---- */
/* Upload a canonical real PauliSum from HOST buffers (reference layout). */
int iqcc_gpu_sum_create(size_t n_qubits, const uint64_t* rows, const double* coeff, size_t M,
                        iqcc_gpu_sum** out);
/* Same, from DEVICE buffers in the reference layout. */
int iqcc_gpu_sum_create_device(size_t n_qubits, const uint64_t* d_rows, const double* d_coeff,
                               size_t M, iqcc_gpu_sum** out);
/* Synthetic G_mol(n, n_terms, seed) built on the device (
 * generator in paper_2603_08883_b200/csrc/gen_mol.h).  Bench input only. */
int iqcc_gpu_sum_generate_mol(size_t n_qubits, size_t n_terms, uint64_t seed, iqcc_gpu_sum** out);
int iqcc_gpu_sum_clone(const iqcc_gpu_sum* h, iqcc_gpu_sum** out);
int iqcc_gpu_sum_destroy(iqcc_gpu_sum* h);
int iqcc_gpu_sum_qubits(const iqcc_gpu_sum* h, size_t* n_qubits);
/* Logical term count (PauliSum::size). */
int iqcc_gpu_sum_size(iqcc_gpu_sum* h, size_t* M);
/* Download in canonical order into HOST buffers of capacity `cap` terms
 * (rows [cap][2B], coeff [cap][2]); *M receives the term count. */
int iqcc_gpu_sum_download(iqcc_gpu_sum* h, uint64_t* rows, double* coeff, size_t cap, size_t* M);
/* Same into DEVICE buffers. */
int iqcc_gpu_sum_download_device(iqcc_gpu_sum* h, uint64_t* d_rows, double* d_coeff, size_t cap,
                                 size_t* M);

/* Inspection: copy the PHYSICAL device store (bit-reversed key rows [M][2B'],
 * B' in {1,2,4}; raw coefficients incl. dead-slot NaNs) to host buffers. */
int iqcc_gpu_sum_raw(iqcc_gpu_sum* h, uint64_t* keys, double* coeff, size_t cap, size_t* M);

/* ---- Pauli text files and the FCIDUMP ingest (iqcc/io.hpp) ------------- */
/* parse_pauli_file (io.hpp:31-87): '#' comments, `# qubits: N`, one
 * `<coefficient> <letters>` term per line (qubit 0 leftmost); the same
 * grammar and "path:line: ..." errors (IQCC_ERUNTIME).  Letters become rows
 * on the device; duplicates are combined on the device (from_terms,
 * pauli.hpp:302-326, drop 1e-12) in file order. */
int iqcc_gpu_read_pauli_file(const char* path, iqcc_gpu_sum** out);
/* write_pauli_file (io.hpp:90-101): "# qubits: N" then "%.17g <letters>" in
 * canonical order; letter strings rendered on the device chunk by chunk
 * while the host writes the previous chunk. */
int iqcc_gpu_write_pauli_file(iqcc_gpu_sum* h, const char* path);
/* jordan_wigner(read_fcidump(path)) (io.hpp:154-276): integrals parsed on the
 * host, the ladder-operator expansion and from_terms on the device.
 * *n_electrons (nullable) receives NELEC.  Equal words are combined in
 * emission order (the reference's std::sort leaves that order unspecified:
 * a word with >= 3 contributions may differ in its last bits). */
int iqcc_gpu_jordan_wigner_fcidump(const char* path, size_t* n_electrons, iqcc_gpu_sum** out);

/* ---- dressing (iqcc/dressing.hpp) ------------------------------------- */
typedef struct {
  size_t n_in;             /* logical terms before the step */
  size_t n_anticommuting;  /* terms whose product was generated */
  size_t n_out;            /* logical terms after the step (and compress) */
} iqcc_dress_stats;

typedef struct {
  size_t dropped_terms;   /* CompressStats, iqcc/pauli.hpp:417-420 */
  double dropped_weight;
} iqcc_compress_stats;

/* In place H <- dress_single(H, {gen, tau}, {drop_thr, ...})
 * (iqcc/dressing.hpp:197-220).  cos_tau/sin_tau are std::cos/std::sin of
 * the amplitude evaluated by the HOST (glibc) so coefficients are
 * bit-identical to the reference.  gen: one row [2B]; identity -> EINVAL. */
int iqcc_gpu_dress(iqcc_gpu_sum* h, const uint64_t* gen, double cos_tau, double sin_tau,
                   double drop_thr, iqcc_dress_stats* stats);
/* In place H <- compress(H, eps, max_terms) (iqcc/pauli.hpp:425-474). */
int iqcc_gpu_compress(iqcc_gpu_sum* h, double eps, size_t max_terms, iqcc_compress_stats* stats);
/* In place dress_sequence (iqcc/dressing.hpp:311-324): K entanglers in
 * order, compress(eps, max_terms) after each step when eps > 0 or the size
 * exceeds max_terms.  gens [K][2B].  drop_thr = MergeOptions::drop_threshold
 * (iqcc/pauli.hpp:236-240), forwarded to every step's merge as the reference
 * does (dressing.hpp:319); check_hermitian is moot for real sums.
 * *terms_in_total (optional) receives the sum of the logical input sizes of
 * the K steps.  On failure the handle's contents are unspecified (partly
 * dressed); destroy or re-upload it. */
int iqcc_gpu_dress_sequence(iqcc_gpu_sum* h, size_t K, const uint64_t* gens, const double* cos_tau,
                            const double* sin_tau, double eps, size_t max_terms, double drop_thr,
                            iqcc_compress_stats* stats, size_t* terms_in_total /* nullable */);
/* SortlessStats of sortless_dress (iqcc/dressing.hpp:182-189, 248-305) for
 * dressing h by gen with sin(tau) = sin_tau: n_buckets = support buckets
 * (bucket_by_support, :159-177), new_term_streams = anticommuting buckets
 * when sin_tau != 0, else 0.  The device never sorts products, so
 * new_stream_sorts is 0; merge_comparisons (the reference's heap k-way merge
 * compare count) has no device counterpart and is reported as 0.
 * > 64 support bits -> IQCC_ERUNTIME as the reference throws. */
int iqcc_gpu_sortless_stats(iqcc_gpu_sum* h, const uint64_t* gen, double sin_tau, size_t* n_buckets,
                            size_t* new_term_streams);
/* growth_split (iqcc/dressing.hpp:41-50). */
int iqcc_gpu_growth_split(iqcc_gpu_sum* h, const uint64_t* gen, size_t* n_commuting,
                          size_t* n_anticommuting);

/* ---- QMF energy / gradient, DIS (iqcc/qmf.hpp, iqcc/dis.hpp) ----------- */
/* factors [n][3] = per qubit (X, Z, Y) single-qubit expectations evaluated
 * on the host exactly as qmf_factor (iqcc/qmf.hpp:56-61). */
int iqcc_gpu_expect(iqcc_gpu_sum* h, const double* factors, double* energy);
/* qmf_energy_gradient (iqcc/qmf.hpp:94-148).  derivs [n][6] =
 * (dth_X, dph_X, dth_Z, dph_Z, dth_Y, dph_Y) from the host's sin/cos.
 * grad receives 2n values (theta block then phi block). */
int iqcc_gpu_qmf_energy_gradient(iqcc_gpu_sum* h, const double* factors, const double* derivs,
                                 double* energy, double* grad);
/* qcc_energy (iqcc/optimizer.hpp:19-25): <omega| U^dag H U |omega> through
 * the fully dressed Hamiltonian (no compression, merges drop exact zeros),
 * for K entanglers gens [K][2B] with host cos/sin of the amplitudes. */
int iqcc_gpu_qcc_energy(iqcc_gpu_sum* h, size_t K, const uint64_t* gens, const double* cos_tau,
                        const double* sin_tau, const double* factors, double* energy);
/* qcc_gradient (iqcc/optimizer.hpp:54-77): dE/dtau_k for every k (grad [K]);
 * step k's derivative (dress_derivative, :31-48) dressed through the rest. */
int iqcc_gpu_qcc_gradient(iqcc_gpu_sum* h, size_t K, const uint64_t* gens, const double* cos_tau,
                          const double* sin_tau, const double* factors, double* grad);
/* gradient (iqcc/dis.hpp:39-52) for K candidate generators [K][2B];
 * flip_group_only != 0 restricts each sum to the candidate's flip group
 * (group_gradient, iqcc/dis.hpp:121-132, exact at poles). */
int iqcc_gpu_gradients(iqcc_gpu_sum* h, const double* factors, const uint64_t* cands, size_t K,
                       int flip_group_only, double* g);
/* build_poly_kernels (iqcc/optimizer.hpp:340-368) for the t subset words
 * [t][2B] of a build_poly expansion (optimizer.hpp:219-268, host side):
 * h_kernel[a][b] = sum_k C_k <W_a P_k W_b> and n_kernel[a][b] = <W_a W_b>,
 * both [t][t][2] (re, im).  at_poles != 0 (QmfState::at_poles) restricts
 * each sum to the x run x_a ^ x_b as sandwich does (optimizer.hpp:288-333). */
int iqcc_gpu_poly_kernels(iqcc_gpu_sum* h, const double* factors, int at_poles, const uint64_t* words,
                          size_t t, double* h_kernel, double* n_kernel);
/* dis_candidates (iqcc/dis.hpp:140-191).  Picks are ranked by (|g| desc,
 * canonical); when has_seed, runs of equal |g| are reshuffled with
 * std::mt19937_64(seed) + std::shuffle exactly as the reference does.
 * Writes min(top_k, cap) picks; *n_picks gets the count before truncation. */
int iqcc_gpu_dis_candidates(iqcc_gpu_sum* h, const double* factors, int at_poles, size_t top_k,
                            double screen_thr, size_t per_group_cap, int has_seed, uint64_t seed,
                            uint64_t* rows_out, double* g_out, size_t cap, size_t* n_picks);

/* ---- bit-wise partitioning across GPUs (iqcc/partition.hpp) ------------ */
/* choose_partition_bits (iqcc/partition.hpp:52-108) computed on the device. */
int iqcc_gpu_choose_partition_bits(iqcc_gpu_sum* h, size_t m, size_t* bits_out,
                                   double* imbalance);
/* Keep only terms whose partition key (gather of `bits`) is owned by
 * `rank` under owner[2^m] (distribute, iqcc/partition.hpp:208-220). */
int iqcc_gpu_sum_restrict(iqcc_gpu_sum* h, size_t m, const size_t* bits, const size_t* owner,
                          int rank);
/* NCCL: 128-byte ncclUniqueId from rank 0, then every rank joins. */
int iqcc_gpu_nccl_unique_id(void* out128);
int iqcc_gpu_comm_init(const void* uid128, int rank, int world);
int iqcc_gpu_comm_destroy(void);
typedef struct {
  size_t mask;            /* entangler key on the partition bits */
  size_t sent_terms;      /* products shipped to the partner rank */
  size_t recv_terms;
  size_t bytes_wire;      /* sent_terms * (16B + 8) device wire bytes */
  size_t bytes_reference; /* sent_terms * (16 + 16B), MessageLog formula */
} iqcc_exchange_stats;
/* One parallel_dress step (iqcc/partition.hpp:398-452) over the
 * communicator: local products whose key flips route to the rank owning
 * key ^ mask; compress_partitioned semantics (:325-396) across ranks. */
int iqcc_gpu_parallel_dress(iqcc_gpu_sum* h, size_t m, const size_t* bits, const size_t* owner,
                            const uint64_t* gen, double cos_tau, double sin_tau, double eps,
                            size_t max_terms, iqcc_exchange_stats* xstats,
                            iqcc_compress_stats* cstats);
/* dress_sequence (iqcc/dressing.hpp:311-324) over parallel_dress steps
 * (partition.hpp:398-452): K entanglers gens[K][2B] with cos/sin of their
 * angles, compress_partitioned(eps, max_terms) after each.  Keeps the
 * store's classify metadata across steps (no per-step classify pass).
 * xstats: NULL or K records; terms_in_total: NULL or the logical input
 * size summed over the K steps and all ranks. */
int iqcc_gpu_parallel_dress_sequence(iqcc_gpu_sum* h, size_t m, const size_t* bits,
                                     const size_t* owner, size_t K, const uint64_t* gens,
                                     const double* cos_tau, const double* sin_tau, double eps,
                                     size_t max_terms, iqcc_exchange_stats* xstats,
                                     iqcc_compress_stats* cstats, size_t* terms_in_total);
/* Collective: reserve every rank's NVLink receive buffer for shards of up
 * to `terms` terms (a store about to grow uncapped maps its peer buffers
 * once instead of at every growth step). */
int iqcc_gpu_parallel_reserve(iqcc_gpu_sum* h, size_t terms);
/* compress_partitioned (iqcc/partition.hpp:325-396) alone, collective:
 * keep identity or |c| >= eps; over max_terms globally, the global top
 * max_terms - 1 by |c| with the canonical tie-break across ranks. */
int iqcc_gpu_parallel_compress(iqcc_gpu_sum* h, double eps, size_t max_terms, iqcc_compress_stats* cstats);
/* Partitioned energy: local expect + allreduce (parallel_expect, :241-254). */
int iqcc_gpu_parallel_expect(iqcc_gpu_sum* h, const double* factors, double* energy);
/* Partitioned build_poly_kernels (iqcc/optimizer.hpp:371-422): local
 * sandwiches over this rank's shard, allgathered over NCCL and summed in
 * worker order; same arguments as iqcc_gpu_poly_kernels, collective. */
int iqcc_gpu_parallel_poly_kernels(iqcc_gpu_sum* h, const double* factors, int at_poles, const uint64_t* words,
                                   size_t t, double* h_kernel, double* n_kernel);
/* Total logical terms over all ranks. */
int iqcc_gpu_parallel_size(iqcc_gpu_sum* h, size_t* total);

/* ---- partitioned sums driven from one host thread (iqcc/partition.hpp) --
 * iqcc_gpu_psum = the reference's PartitionedSum (:145-173) held on the
 * device: 2^m shards, shard p owned by worker owner[p], worker w running on
 * CUDA device devices[w] (NULL: w % device count).  One call drives every
 * shard (one engine context and host worker thread per shard inside the
 * handle, like run_tasks(kThreaded), :190-204); products cross devices over
 * NVLink.  Any m (overpartitioning: several partitions per worker/GPU). */
typedef struct iqcc_gpu_psum iqcc_gpu_psum;
typedef struct {
  size_t source;      /* partition id, MessageRecord (:135-140) */
  size_t destination;
  size_t terms;
  size_t bytes;       /* terms * (sizeof(Complex) + 2 * blocks * 8), :419-422 */
} iqcc_message_record;
/* distribute (:208-220): a canonical real host sum -> shards by partition key. */
int iqcc_gpu_psum_distribute(size_t n_qubits, const uint64_t* rows, const double* coeff, size_t M,
                             size_t m, const size_t* bits, const size_t* owner, size_t n_workers,
                             const int* devices /* nullable */, iqcc_gpu_psum** out);
/* From existing host shards (a reference PartitionedSum): rows[p]/coeffs[p]
 * of sizes[p] terms; a term outside its shard -> IQCC_ERUNTIME ("term in
 * wrong shard", PartitionedSum::validate :162-172). */
int iqcc_gpu_psum_create_shards(size_t n_qubits, size_t m, const size_t* bits, const size_t* owner,
                                size_t n_workers, const int* devices, const uint64_t* const* rows,
                                const double* const* coeffs, const size_t* sizes, iqcc_gpu_psum** out);
int iqcc_gpu_psum_destroy(iqcc_gpu_psum* ph);
/* n_partitions = 2^m; total = total_terms() (:147-151). */
int iqcc_gpu_psum_info(iqcc_gpu_psum* ph, size_t* n_partitions, size_t* total_terms);
int iqcc_gpu_psum_shard_sizes(iqcc_gpu_psum* ph, size_t* sizes /* [2^m] */);
int iqcc_gpu_psum_owner(iqcc_gpu_psum* ph, size_t* owner /* [2^m] */);
int iqcc_gpu_psum_download_shard(iqcc_gpu_psum* ph, size_t p, uint64_t* rows, double* coeff, size_t cap,
                                 size_t* M);
/* gather (:222-230): the canonical union of the shards into host buffers. */
int iqcc_gpu_psum_gather(iqcc_gpu_psum* ph, uint64_t* rows, double* coeff, size_t cap, size_t* M);
/* In place ph <- parallel_dress(ph, {gen, tau}, eps, max_terms, log, mode,
 * stats) (:398-452) with host cos/sin of tau.  log: NULL or log_cap records;
 * *n_log receives the record count (records past log_cap are dropped);
 * cstats accumulate ParallelDressStats::compress; *mask = stats->mask. */
int iqcc_gpu_psum_dress(iqcc_gpu_psum* ph, const uint64_t* gen, double cos_tau, double sin_tau, double eps,
                        size_t max_terms, iqcc_message_record* log, size_t log_cap, size_t* n_log,
                        iqcc_compress_stats* cstats, size_t* mask);
/* parallel_expect (:241-254): worker-order reduction of the shard energies. */
int iqcc_gpu_psum_expect(iqcc_gpu_psum* ph, const double* factors, double* energy);
/* qmf_energy_gradient (iqcc/qmf.hpp:94-148) over the shards, energy and 2n
 * gradients reduced in worker order like parallel_expect. */
int iqcc_gpu_psum_qmf_energy_gradient(iqcc_gpu_psum* ph, const double* factors, const double* derivs,
                                      double* energy, double* grad);
/* DIS gradients (iqcc/dis.hpp:39-52, group_gradient :121-132) of K candidate
 * words over the shards, reduced in worker order. */
int iqcc_gpu_psum_gradients(iqcc_gpu_psum* ph, const double* factors, const uint64_t* cands, size_t K,
                            int flip_group_only, double* g);
/* rebalance (:457-494) + migration of every shard whose new owner runs on
 * another device; owner_out (nullable) receives the new map. */
int iqcc_gpu_psum_rebalance(iqcc_gpu_psum* ph, double threshold, size_t* owner_out);

/* merge_sums (iqcc/pauli.hpp:383-415) of two device sums into a new one
 * (a's coefficient first on shared words, keep_term with drop_thr). */
int iqcc_gpu_merge_sums(iqcc_gpu_sum* a, iqcc_gpu_sum* b, double drop_thr, iqcc_gpu_sum** out);

/* Partitioned gradients over the one-process-per-GPU communicator: local
 * values allgathered and summed in rank order (reduce_scalar, :233-237). */
int iqcc_gpu_parallel_qmf_energy_gradient(iqcc_gpu_sum* h, const double* factors, const double* derivs,
                                          double* energy, double* grad);
int iqcc_gpu_parallel_gradients(iqcc_gpu_sum* h, const double* factors, const uint64_t* cands, size_t K,
                                int flip_group_only, double* g);

#ifdef __cplusplus
}
#endif
#endif
