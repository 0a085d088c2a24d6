// common.cuh — shared internals of libsperm.so (product code; never used by oracle/).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/sperm.h"

namespace sperm {

// CRT primes: the 8 largest primes below 2^31 (all > 2^30), descending.
constexpr uint32_t kPrimes[SPERM_KMAX] = {2147483647u, 2147483629u, 2147483587u, 2147483579u,
                                          2147483563u, 2147483549u, 2147483543u, 2147483497u};

// error reporting (thread-local message, see host.cpp)
int set_error(int code, const std::string& msg);
int cuda_check(cudaError_t e, const char* what);
#define SPERM_CUDA(call)                                  \
  do {                                                    \
    cudaError_t e_ = (call);                              \
    if (e_ != cudaSuccess) return ::sperm::cuda_check(e_, #call); \
  } while (0)
#define SPERM_LAUNCH_CHECK(what)                          \
  do {                                                    \
    cudaError_t e_ = cudaGetLastError();                  \
    if (e_ != cudaSuccess) return ::sperm::cuda_check(e_, what); \
  } while (0)

// kernel timing registry (host.cpp)
struct TimingScope {
  TimingScope(const char* name, cudaStream_t s);
  ~TimingScope();
  const char* name_;
  cudaStream_t s_;
  void* ev0_;
  void* ev1_;
};

int sm_count();
void keep_pool_memory();  // keep the default mempool's memory between calls (host.cu)
void count_launch(int k = 1);  // own-kernel launch counter (sperm_launch_count)

}  // namespace sperm
