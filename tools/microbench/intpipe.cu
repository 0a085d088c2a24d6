// Integer / FP32 pipe throughput microbenchmark for sm_100a (B200).
// Measures warp-instruction throughput of IMAD (32-bit mul), IMAD.WIDE (32x32->64),
// IMAD.HI, IADD3, LOP3, FMUL, and a Montgomery modmul chain, each with 8
// independent dependency chains per thread so latency is hidden.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096
#define CH 8

__global__ void k_imad(uint32_t* out, uint32_t seed) {
  uint32_t a[CH]; uint32_t m = seed | 1u;
#pragma unroll
  for (int c = 0; c < CH; ++c) a[c] = threadIdx.x + c * 7 + seed;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = a[c] * m + (uint32_t)c;
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s ^= a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_imul(uint32_t* out, uint32_t seed) {
  uint32_t a[CH]; uint32_t m = seed | 1u;
#pragma unroll
  for (int c = 0; c < CH; ++c) a[c] = threadIdx.x + c * 7 + seed;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = a[c] * m;
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s ^= a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_wide(uint64_t* out, uint32_t seed) {
  uint32_t a[CH]; uint64_t acc[CH]; uint32_t m = seed | 1u;
#pragma unroll
  for (int c = 0; c < CH; ++c) { a[c] = threadIdx.x + c * 7 + seed; acc[c] = 0; }
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) { uint64_t t = (uint64_t)a[c] * m; a[c] = (uint32_t)(t >> 32) ^ (uint32_t)t; }
  }
  uint64_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s ^= a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_iadd(uint32_t* out, uint32_t seed) {
  uint32_t a[CH]; uint32_t m = seed | 1u;
#pragma unroll
  for (int c = 0; c < CH; ++c) a[c] = threadIdx.x + c * 7 + seed;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = a[c] + m + a[(c + 1) % CH];
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s ^= a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_fmul(float* out, float seed) {
  float a[CH]; float m = seed;
#pragma unroll
  for (int c = 0; c < CH; ++c) a[c] = threadIdx.x + c * 7 + seed;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = a[c] * m;
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma(float* out, float seed) {
  float a[CH]; float m = seed; float b = seed * 0.5f;
#pragma unroll
  for (int c = 0; c < CH; ++c) a[c] = threadIdx.x + c * 7 + seed;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = a[c] * m + b;
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dfma(double* out, double seed) {
  double a[CH]; double m = seed; double b = seed * 0.5;
#pragma unroll
  for (int c = 0; c < CH; ++c) a[c] = threadIdx.x + c * 7 + seed;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = a[c] * m + b;
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// Montgomery multiply a*b*2^-32 mod p, p < 2^31 odd, pinv = -p^-1 mod 2^32
__device__ __forceinline__ uint32_t mont(uint32_t a, uint32_t b, uint32_t p, uint32_t pinv) {
  uint64_t t = (uint64_t)a * b;
  uint32_t m = (uint32_t)t * pinv;
  uint64_t u = (t + (uint64_t)m * p) >> 32;
  uint32_t r = (uint32_t)u;
  return r >= p ? r - p : r;
}
__global__ void k_mont(uint32_t* out, uint32_t seed, uint32_t p, uint32_t pinv) {
  uint32_t a[CH]; uint32_t m = seed % p;
#pragma unroll
  for (int c = 0; c < CH; ++c) a[c] = (threadIdx.x + c * 7 + seed) % p;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = mont(a[c], m, p, pinv);
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s ^= a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// Mersenne 2^31-1 reduction of a 62-bit product
__device__ __forceinline__ uint32_t mersmul(uint32_t a, uint32_t b) {
  uint64_t t = (uint64_t)a * b;
  uint32_t r = ((uint32_t)t & 0x7fffffffu) + (uint32_t)(t >> 31);
  return r >= 0x7fffffffu ? r - 0x7fffffffu : r;
}
__global__ void k_mers(uint32_t* out, uint32_t seed) {
  uint32_t a[CH]; uint32_t m = seed % 0x7fffffffu;
#pragma unroll
  for (int c = 0; c < CH; ++c) a[c] = (threadIdx.x + c * 7 + seed) % 0x7fffffffu;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = mersmul(a[c], m);
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s ^= a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}


// signed Montgomery (Seiler): a,b in (-p,p), p < 2^31 odd, pinv = p^-1 mod 2^32; result in (-p,p) = a*b*2^-32
__device__ __forceinline__ int32_t smont(int32_t a, int32_t b, int32_t p, int32_t pinv) {
  int64_t t = (int64_t)a * b;
  int32_t m = (int32_t)t * pinv;
  int32_t h = __mulhi(m, p);
  return (int32_t)(t >> 32) - h;
}
__global__ void k_smont(int32_t* out, int32_t seed, int32_t p, int32_t pinv) {
  int32_t a[CH]; int32_t m = seed % p;
#pragma unroll
  for (int c = 0; c < CH; ++c) a[c] = (threadIdx.x + c * 7 + seed) % p;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = smont(a[c], m, p, pinv);
  }
  int32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s ^= a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_imadhi(uint32_t* out, uint32_t seed) {
  uint32_t a[CH]; uint32_t m = seed | 1u;
#pragma unroll
  for (int c = 0; c < CH; ++c) a[c] = threadIdx.x + c * 7 + seed;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) a[c] = __umulhi(a[c], m) + (uint32_t)c;
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s ^= a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// mixed: 1 IMAD + 1 IADD3 + 1 LOP3 per chain step (pipe balance probe)
__global__ void k_mix(uint32_t* out, uint32_t seed) {
  uint32_t a[CH]; uint32_t m = seed | 1u;
#pragma unroll
  for (int c = 0; c < CH; ++c) a[c] = threadIdx.x + c * 7 + seed;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) { uint32_t x = a[c] * m; x = x + a[(c+1)%CH] + m; a[c] = x ^ (a[(c+3)%CH] & 0x5555u); }
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s ^= a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
void run(const char* name, F launch, double ops_per_thread_iter) {
  int blocks = 148 * 8, threads = 256;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) launch(blocks, threads);
  cudaEventRecord(e0);
  const int R = 10;
  for (int r = 0; r < R; ++r) launch(blocks, threads);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = (double)blocks * threads * ITERS * CH * ops_per_thread_iter * R;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double per_clk_sm = ops / (ms * 1e-3) / (148.0 * clk * 1e3);
  printf("%-10s %10.3f Tops/s  %7.2f lane-ops/clk/SM (at max clock %d MHz)\n", name, ops / (ms * 1e-3) / 1e12, per_clk_sm, clk / 1000);
}

int main() {
  void* buf; cudaMalloc(&buf, 148 * 8 * 256 * 8);
  uint32_t p = 2147483629u; uint32_t inv = 1; for (int i = 0; i < 5; ++i) inv *= 2 - p * inv; uint32_t pinv = (uint32_t)(-(int32_t)inv);
  run("imad", [&](int b, int t) { k_imad<<<b, t>>>((uint32_t*)buf, 12345u); }, 1.0);
  run("imul", [&](int b, int t) { k_imul<<<b, t>>>((uint32_t*)buf, 12345u); }, 1.0);
  run("wide", [&](int b, int t) { k_wide<<<b, t>>>((uint64_t*)buf, 12345u); }, 1.0);
  run("iadd3", [&](int b, int t) { k_iadd<<<b, t>>>((uint32_t*)buf, 12345u); }, 1.0);
  run("fmul", [&](int b, int t) { k_fmul<<<b, t>>>((float*)buf, 1.0001f); }, 1.0);
  run("ffma", [&](int b, int t) { k_ffma<<<b, t>>>((float*)buf, 1.0001f); }, 1.0);
  run("dfma", [&](int b, int t) { k_dfma<<<b, t>>>((double*)buf, 1.0001); }, 1.0);
  run("mont", [&](int b, int t) { k_mont<<<b, t>>>((uint32_t*)buf, 12345u, p, pinv); }, 1.0);
  { int32_t ps = 2147483629; int32_t iv = 1; for (int i = 0; i < 5; ++i) iv *= 2 - ps * iv;
    run("smont", [&](int b, int t) { k_smont<<<b, t>>>((int32_t*)buf, 12345, ps, iv); }, 1.0); }
  run("imadhi", [&](int b, int t) { k_imadhi<<<b, t>>>((uint32_t*)buf, 12345u); }, 1.0);
  run("mix3", [&](int b, int t) { k_mix<<<b, t>>>((uint32_t*)buf, 12345u); }, 3.0);
  run("mersenne", [&](int b, int t) { k_mers<<<b, t>>>((uint32_t*)buf, 12345u); }, 1.0);
  cudaError_t err = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(err));
  return err != cudaSuccess;
}
