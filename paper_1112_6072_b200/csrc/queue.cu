// queue.cu — a box-wide work queue for the improved Step 3 across GPUs: "each job goes to the
// currently least loaded processor", realised as dynamic claims of
// chunks of the estimate order from ONE 64-bit counter in rank 0's device memory.  Peers map it
// with CUDA IPC (cudaIpcOpenMemHandle) and claim with a system-scope atomicAdd over NVLink /
// NVSwitch — no host round trip through a TCP store per claim.
#include <cstring>

#include "common.cuh"

namespace sperm {
namespace {

// one thread: start = atomicAdd(counter, chunk) on the (possibly peer-mapped) counter
__global__ void queue_claim_kernel(unsigned long long* counter, unsigned long long chunk,
                                   unsigned long long* out) {
  *out = atomicAdd_system(counter, chunk);
}

}  // namespace
}  // namespace sperm

using namespace sperm;

static_assert(sizeof(cudaIpcMemHandle_t) <= SPERM_QUEUE_HANDLE_BYTES, "IPC handle size");

extern "C" int sperm_queue_create(void** d_counter, void* h_handle) {
  if (!d_counter || !h_handle) return set_error(SPERM_ERR_ARG, "sperm_queue_create: NULL argument");
  *d_counter = nullptr;
  unsigned long long* c = nullptr;
  SPERM_CUDA(cudaMalloc((void**)&c, sizeof(unsigned long long)));
  cudaError_t e = cudaMemset(c, 0, sizeof(unsigned long long));
  cudaIpcMemHandle_t h;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, c);
  if (e != cudaSuccess) {
    cudaFree(c);
    return cuda_check(e, "sperm_queue_create");
  }
  memset(h_handle, 0, SPERM_QUEUE_HANDLE_BYTES);
  memcpy(h_handle, &h, sizeof(h));
  *d_counter = c;
  return SPERM_OK;
}

extern "C" int sperm_queue_open(const void* h_handle, void** d_counter) {
  if (!d_counter || !h_handle) return set_error(SPERM_ERR_ARG, "sperm_queue_open: NULL argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, h_handle, sizeof(h));
  void* p = nullptr;
  SPERM_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  *d_counter = p;
  return SPERM_OK;
}

extern "C" int sperm_queue_claim(void* d_counter, int64_t chunk, void* d_scratch, int64_t* h_start, void* stream) {
  if (!d_counter || !d_scratch || !h_start || chunk < 1) return set_error(SPERM_ERR_ARG, "sperm_queue_claim: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  count_launch();
  queue_claim_kernel<<<1, 1, 0, st>>>((unsigned long long*)d_counter, (unsigned long long)chunk,
                                      (unsigned long long*)d_scratch);
  SPERM_LAUNCH_CHECK("queue_claim_kernel");
  unsigned long long v = 0;
  SPERM_CUDA(cudaMemcpyAsync(&v, d_scratch, sizeof(v), cudaMemcpyDeviceToHost, st));
  SPERM_CUDA(cudaStreamSynchronize(st));
  *h_start = (int64_t)v;
  return SPERM_OK;
}

extern "C" int sperm_queue_close(void* d_counter, int owner) {
  if (!d_counter) return SPERM_OK;
  SPERM_CUDA(owner ? cudaFree(d_counter) : cudaIpcCloseMemHandle(d_counter));
  return SPERM_OK;
}
