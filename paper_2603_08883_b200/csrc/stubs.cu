#include <stdexcept>
#include "multi.cuh"
namespace iqcc_b200 {
[[noreturn]] static void ni(const char* w) { throw std::runtime_error(std::string(w) + ": not implemented yet"); }
double expect_store(DeviceStore&, const double*) { ni("expect"); }
double qmf_grad_store(DeviceStore&, const double*, const double*, double*) { ni("qmf"); }
void gradients_store(DeviceStore&, const double*, const uint64_t*, size_t, bool, double*) { ni("gradients"); }
size_t dis_store(DeviceStore&, const double*, bool, size_t, double, size_t, std::vector<uint64_t>&, std::vector<double>&) { ni("dis"); }
double choose_bits_store(DeviceStore&, size_t, size_t*) { ni("choose_bits"); }
void restrict_store(DeviceStore&, size_t, const size_t*, const size_t*, int) { ni("restrict"); }
void multi_unique_id(void*) { ni("nccl"); }
void multi_init(const void*, int, int) { ni("nccl"); }
void multi_shutdown() {}
void parallel_dress_step(DeviceStore&, size_t, const size_t*, const size_t*, const uint64_t*, double, double, double, size_t, iqcc_exchange_stats*, iqcc_compress_stats*) { ni("parallel_dress"); }
double parallel_expect_store(DeviceStore&, const double*) { ni("parallel_expect"); }
size_t parallel_size(DeviceStore&) { ni("parallel_size"); }
}
