// multi.cuh — bit-wise partitioning across GPUs (one process per GPU, NCCL).
#pragma once
#include "../../include/iqcc_b200.h"
#include "engine.cuh"

namespace iqcc_b200 {
void multi_unique_id(void* out128);
void multi_init(const void* uid128, int rank, int world);
void multi_shutdown();
/// Collective at the start of every partitioned call: (re)size the CUDA IPC
/// receive buffers of the NVLink product push to the largest shard.
void multi_prepare(DeviceStore& s);
void parallel_dress_step(DeviceStore& s, size_t m, const size_t* bits, const size_t* owner,
                         const uint64_t* gen_row, double cs, double sn, double eps,
                         size_t max_terms, iqcc_exchange_stats* xs, iqcc_compress_stats* cs_out,
                         const uint64_t* next_row = nullptr, double theta = 0.0,
                         double exact = 0.0, bool* spec_failed = nullptr);
/// Sum of a host value over the ranks (one allreduce).
size_t parallel_sum(size_t v);
double parallel_expect_store(DeviceStore& s, const double* factors);
/// compress_partitioned (iqcc/partition.hpp:325-396) on its own: global
/// counts and histograms allreduced, canonical tie-break across ranks.
void parallel_compress_store(DeviceStore& s, double eps, size_t max_terms, iqcc_compress_stats* cs);
/// Collective: size every rank's NVLink receive buffer for shards of up to
/// `terms` terms now (mapping a peer buffer costs ~1 s per 10 GB, so a
/// store that will grow uncapped reserves once instead of regrowing).
void parallel_reserve(DeviceStore& s, size_t terms);
/// Partitioned QMF energy + 2n gradients and DIS gradients of K candidates:
/// local values allgathered, summed element by element in rank order.
double parallel_qmf_grad_store(DeviceStore& s, const double* factors, const double* derivs, double* grad);
void parallel_gradients_store(DeviceStore& s, const double* factors, const uint64_t* cands, size_t K,
                              bool flip_only, double* g);
size_t parallel_size(DeviceStore& s);
}  // namespace iqcc_b200
