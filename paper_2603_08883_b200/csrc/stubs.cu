#include <stdexcept>
#include "multi.cuh"
namespace iqcc_b200 {
[[noreturn]] static void ni(const char* w) { throw std::runtime_error(std::string(w) + ": not implemented yet"); }
void multi_unique_id(void*) { ni("nccl"); }
void multi_init(const void*, int, int) { ni("nccl"); }
void multi_shutdown() {}
void parallel_dress_step(DeviceStore&, size_t, const size_t*, const size_t*, const uint64_t*, double, double, double, size_t, iqcc_exchange_stats*, iqcc_compress_stats*) { ni("parallel_dress"); }
double parallel_expect_store(DeviceStore&, const double*) { ni("parallel_expect"); }
size_t parallel_size(DeviceStore&) { ni("parallel_size"); }
}
