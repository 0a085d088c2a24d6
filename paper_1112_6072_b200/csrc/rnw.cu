// rnw.cu — batched R-NW (Ryser / Nijenhuis-Wilf, Gray-code order)
// leaf permanents in exact multi-prime modular arithmetic, sm_100a.
//
//   per(A) = (-1)^(n-1) 2^(1-n) sum_{t=0}^{2^(n-1)-1} (-1)^t prod_i w_i(g(t))
//   w_i(S) = 2 a_{i,n-1} - sum_j a_ij + 2 sum_{j in S} a_ij        (doubled NW row sums)
//   g(t)   = t ^ (t >> 1); going from t-1 to t flips Gray bit / column ctz(t).
//
// Work decomposition: a work item is (leaf, chunk) where a chunk is
// 32 lanes x 2^m consecutive terms; lane l of a chunk owns t in [t0, t0 + 2^m) with
// t0 = (chunk*32 + l) * 2^m.  Because every lane's range is aligned to 2^m, the flipped
// column ctz(t) = ctz(t - t0) is the same in all 32 lanes at every step (warp-uniform
// shared-memory broadcast of the column).  A persistent grid pulls work items from one
// atomic counter in the given leaf order (improved Step 3).
//
// Per term: the row-sum vector w[NP] lives in registers (static indexing: the column
// update is dense over NP rows, 4 rows per 128-bit broadcast load); rows are multiplied
// in groups of G inside exact int32 (|group| < 2^30 is guaranteed by the per-leaf bound
// pass), then the NP/G group values are chained with signed Montgomery multiplication
// modulo each of the leaf's k primes.  Terms are summed exactly (int64 per lane), reduced
// mod p per chunk and added to the leaf's uint64 accumulator (exact, order-independent).
#include <algorithm>
#include <cmath>

#include "common.cuh"

namespace sperm {
namespace {

constexpr int kRnwThreads = 256;  // 8 warps per CTA
constexpr int kMaxLaneBits = 14;  // terms per lane <= 2^14

struct PrimeSet {
  int32_t p[SPERM_KMAX];
  int32_t pinv[SPERM_KMAX];  // p^-1 mod 2^32
  uint32_t r2[SPERM_KMAX];   // unused by the kernels (kept for layout stability)
};

PrimeSet make_primes() {
  PrimeSet s;
  for (int q = 0; q < SPERM_KMAX; ++q) {
    uint32_t p = kPrimes[q];
    uint32_t inv = p;  // Newton: inv = p^-1 mod 2^32 (p*p = 1 mod 8 start)
    for (int it = 0; it < 5; ++it) inv *= 2u - p * inv;
    s.p[q] = (int32_t)p;
    s.pinv[q] = (int32_t)inv;
    s.r2[q] = 0;
  }
  return s;
}

// Signed Montgomery product (a*b*2^-32 mod p) for |a|,|b| < p < 2^31; result in (-p, p).
__device__ __forceinline__ int32_t smont(int32_t a, int32_t b, int32_t p, int32_t pinv) {
  int64_t t = (int64_t)a * b;
  int32_t m = (int32_t)t * pinv;
  return (int32_t)(t >> 32) - __mulhi(m, p);
}

template <int NP>
struct Layout {
  static constexpr int kPos = 0;                                  // dpos[col][NP]
  static constexpr int kNeg = ((NP * NP + 31) / 32) * 32 + 16;    // dneg[col][NP], bank-shifted
  static constexpr int kW0 = kNeg + NP * NP;                      // w0[NP]
  static constexpr int kWords = ((kW0 + NP + 3) / 4) * 4;         // per warp, 16-byte aligned
};

// ----------------------------------------------------------------------------- prep
// One warp per leaf: row / column abs sums -> number of primes k and group size G.
__global__ void rnw_prep_kernel(const int32_t* __restrict__ mats, int n, int NP, int64_t count,
                                const int64_t* __restrict__ coef, int min_primes,
                                int2* __restrict__ meta, int* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  const int64_t leaf = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (leaf >= count) return;
  const int32_t* a = mats + leaf * (int64_t)n * n;
  __shared__ int64_t srow[8][SPERM_NMAX];
  int64_t* R = srow[threadIdx.x >> 5];
  double lr = 0.0, lc = 0.0;
  bool zero = false, range_bad = false;
  for (int i = lane; i < n; i += 32) {
    int64_t r = 0, c = 0;
    for (int j = 0; j < n; ++j) {
      r += llabs((long long)a[i * n + j]);
      c += llabs((long long)a[j * n + i]);
    }
    R[i] = r;
    if (r == 0 || c == 0) zero = true;
    if (r >= (1ll << 30)) range_bad = true;
    if (r > 0) lr += log2((double)r);
    if (c > 0) lc += log2((double)c);
  }
  for (int o = 16; o; o >>= 1) {
    lr += __shfl_xor_sync(0xffffffffu, lr, o);
    lc += __shfl_xor_sync(0xffffffffu, lc, o);
  }
  zero = __any_sync(0xffffffffu, zero);
  range_bad = __any_sync(0xffffffffu, range_bad);
  __syncwarp();
  if (lane == 0) {
    if (range_bad) atomicOr(err, 1);
    double lb = zero ? -1.0 : fmin(lr, lc);
    int64_t cf = coef ? coef[leaf] : 1;
    if (cf == 0) lb = -1.0;
    else if (lb >= 0.0) lb += log2(fabs((double)cf));
    // need prod p_q > 2 * bound; each p_q > 2^30.99999; margin for log2 rounding
    double need = lb + 1.0 + 1e-6 * fabs(lb) + 1e-6;
    int k = min_primes;
    while (k <= SPERM_KMAX && 30.99999 * k <= need) ++k;
    if (k > SPERM_KMAX) {
      atomicOr(err, 2);
      k = SPERM_KMAX;
    }
    // largest group size G in {8,4,2,1} with every group product of row bounds < 2^30
    int G = 1;
    for (int g = 8; g >= 2; g >>= 1) {
      bool ok = true;
      for (int s = 0; s < NP && ok; s += g) {
        int64_t prod = 1;
        for (int r = s; r < s + g; ++r) {
          int64_t b = r < n ? R[r] : 1;
          if (b == 0) { prod = 0; break; }
          if (prod > ((1ll << 30) - 1) / b) { ok = false; break; }
          prod *= b;
        }
        if (prod >= (1ll << 30)) ok = false;
      }
      if (ok) { G = g; break; }
    }
    meta[leaf] = make_int2(k, G);
  }
}

// ----------------------------------------------------------------------------- main
template <int NP, int G>
__device__ __forceinline__ void term_product(const int32_t (&w)[NP], int k, const PrimeSet& ps,
                                             int32_t (&out)[SPERM_KMAX]) {
  constexpr int NG = NP / G;
  int32_t gp[NG];
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    int32_t x = w[g * G];
#pragma unroll
    for (int r = 1; r < G; ++r) x *= w[g * G + r];
    gp[g] = x;
  }
#pragma unroll
  for (int q = 0; q < SPERM_KMAX; ++q) {
    if (q < k) {
      int32_t pr = gp[0];
#pragma unroll
      for (int g = 1; g < NG; ++g) pr = smont(pr, gp[g], ps.p[q], ps.pinv[q]);
      out[q] = pr;
    }
  }
}

// Runs one lane's 2^m terms starting at t0 (t0 a multiple of 2^m, m >= 1).
template <int NP, int G>
__device__ __forceinline__ void lane_range(int32_t (&w)[NP], const int32_t* __restrict__ sm, int m,
                                        uint64_t t0, int k, const PrimeSet& ps,
                                        int64_t (&acc)[SPERM_KMAX]) {
  using L = Layout<NP>;
  int32_t d0[NP];
#pragma unroll
  for (int v = 0; v < NP / 4; ++v) {
    int4 d = reinterpret_cast<const int4*>(sm + L::kPos)[v];
    d0[4 * v] = d.x; d0[4 * v + 1] = d.y; d0[4 * v + 2] = d.z; d0[4 * v + 3] = d.w;
  }
  int32_t pe[SPERM_KMAX], po[SPERM_KMAX];
  const uint32_t steps = 1u << m;
  for (uint32_t u = 0; u < steps; u += 2) {
    if (u) {
      const int j = __ffs(u) - 1;  // >= 1, warp-uniform
      const bool add = !(((t0 + u) >> (j + 1)) & 1ull);
      const int4* col = reinterpret_cast<const int4*>(sm + (add ? L::kPos : L::kNeg) + j * NP);
#pragma unroll
      for (int v = 0; v < NP / 4; ++v) {
        int4 d = col[v];
        w[4 * v] += d.x; w[4 * v + 1] += d.y; w[4 * v + 2] += d.z; w[4 * v + 3] += d.w;
      }
    }
    term_product<NP, G>(w, k, ps, pe);
    // odd step t0+u+1 flips column 0: added iff bit 1 of t0+u+1 is 0
    if (!(((t0 + u + 1) >> 1) & 1ull)) {
#pragma unroll
      for (int i = 0; i < NP; ++i) w[i] += d0[i];
    } else {
#pragma unroll
      for (int i = 0; i < NP; ++i) w[i] -= d0[i];
    }
    term_product<NP, G>(w, k, ps, po);
#pragma unroll
    for (int q = 0; q < SPERM_KMAX; ++q)
      if (q < k) acc[q] += (int64_t)pe[q] - (int64_t)po[q];
  }
}

template <int NP>
__global__ void __launch_bounds__(kRnwThreads) rnw_main_kernel(
    const int32_t* __restrict__ mats, int n, int m, int cbits, const int32_t* __restrict__ order,
    const int2* __restrict__ meta, unsigned long long* __restrict__ queue, uint64_t total_items,
    unsigned long long* __restrict__ leaf_acc, PrimeSet ps) {
  using L = Layout<NP>;
  extern __shared__ int4 smem4[];
  const int lane = threadIdx.x & 31;
  int32_t* sm = reinterpret_cast<int32_t*>(smem4) + (threadIdx.x >> 5) * L::kWords;
  const uint64_t T = 1ull << (n - 1);
  int64_t cur_leaf = -1;
  while (true) {
    unsigned long long item = 0;
    if (lane == 0) item = atomicAdd(queue, 1ull);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= total_items) break;
    const int64_t slot = (int64_t)(item >> cbits);
    const uint64_t chunk = item & ((1ull << cbits) - 1);
    const int64_t leaf = order ? (int64_t)order[slot] : slot;
    const int2 mt = meta[leaf];
    const int k = mt.x, G = mt.y;
    if (leaf != cur_leaf) {
      __syncwarp();
      const int32_t* a = mats + leaf * (int64_t)n * n;
      // dpos[j][i] = 2 a_ij, dneg = -dpos (columns j < n-1); rows >= n are padding (0)
      for (int e = lane; e < NP * NP; e += 32) {
        const int j = e / NP, i = e % NP;
        const int32_t v = (j < n - 1 && i < n) ? 2 * a[i * n + j] : 0;
        sm[L::kPos + e] = v;
        sm[L::kNeg + e] = -v;
      }
      for (int i = lane; i < NP; i += 32) {
        int32_t w0 = 1;
        if (i < n) {
          int32_t s = 0;
          for (int j = 0; j < n; ++j) s += a[i * n + j];
          w0 = 2 * a[i * n + n - 1] - s;
        }
        sm[L::kW0 + i] = w0;
      }
      __syncwarp();
      cur_leaf = leaf;
    }
    const uint64_t t0 = ((chunk << 5) + (uint64_t)lane) << m;
    int64_t acc[SPERM_KMAX];
#pragma unroll
    for (int q = 0; q < SPERM_KMAX; ++q) acc[q] = 0;
    if (t0 < T) {
      int32_t w[NP];
#pragma unroll
      for (int i = 0; i < NP; ++i) w[i] = sm[L::kW0 + i];
      const uint64_t g0 = t0 ^ (t0 >> 1);
      for (int j = (m > 0 ? m - 1 : 0); j < n - 1; ++j) {
        if ((g0 >> j) & 1ull) {
#pragma unroll
          for (int i = 0; i < NP; ++i) w[i] += sm[L::kPos + j * NP + i];
        }
      }
      if (m == 0) {  // one term per lane (tiny leaves)
        int32_t pr[SPERM_KMAX];
        switch (G) {
          case 8: term_product<NP, 8>(w, k, ps, pr); break;
          case 4: term_product<NP, 4>(w, k, ps, pr); break;
          case 2: term_product<NP, 2>(w, k, ps, pr); break;
          default: term_product<NP, 1>(w, k, ps, pr); break;
        }
        const bool neg = t0 & 1ull;
#pragma unroll
        for (int q = 0; q < SPERM_KMAX; ++q)
          if (q < k) acc[q] = neg ? -(int64_t)pr[q] : (int64_t)pr[q];
      } else {
        switch (G) {
          case 8: lane_range<NP, 8>(w, sm, m, t0, k, ps, acc); break;
          case 4: lane_range<NP, 4>(w, sm, m, t0, k, ps, acc); break;
          case 2: lane_range<NP, 2>(w, sm, m, t0, k, ps, acc); break;
          default: lane_range<NP, 1>(w, sm, m, t0, k, ps, acc); break;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < SPERM_KMAX; ++q) {
      if (q < k) {
        int64_t v = acc[q];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) {
          int64_t r = v % ps.p[q];
          if (r < 0) r += ps.p[q];
          atomicAdd(leaf_acc + leaf * SPERM_KMAX + q, (unsigned long long)r);
        }
      }
    }
  }
}

// ----------------------------------------------------------------------------- finalize
__device__ __forceinline__ uint64_t powmod(uint64_t b, uint64_t e, uint64_t p) {
  uint64_t r = 1 % p;
  b %= p;
  while (e) {
    if (e & 1) r = r * b % p;
    b = b * b % p;
    e >>= 1;
  }
  return r;
}

__global__ void rnw_finalize_kernel(int n, int NP, int64_t count, const int2* __restrict__ meta,
                                    const unsigned long long* __restrict__ leaf_acc,
                                    const int64_t* __restrict__ coef, const int32_t* __restrict__ job,
                                    uint32_t* __restrict__ leaf_res, int32_t* __restrict__ leaf_k,
                                    unsigned long long* __restrict__ job_acc, int64_t num_jobs) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= count * SPERM_KMAX) return;
  const int64_t leaf = idx / SPERM_KMAX;
  const int q = (int)(idx % SPERM_KMAX);
  const int2 mt = meta[leaf];
  const int k = mt.x, G = mt.y;
  if (q == 0 && leaf_k) leaf_k[leaf] = k;
  if (q >= k) {
    if (leaf_res) leaf_res[idx] = 0u;
    return;
  }
  // the primes of kPrimes (common.cuh), replicated for device code
  const uint32_t primes[SPERM_KMAX] = {2147483647u, 2147483629u, 2147483587u, 2147483579u,
                                       2147483563u, 2147483549u, 2147483543u, 2147483497u};
  const uint64_t pq = primes[q];
  uint64_t val;
  if (n == 0) {
    val = 1;
  } else {
    const uint64_t S = (uint64_t)(leaf_acc[leaf * SPERM_KMAX + q] % pq);
    const int NG = NP / G;
    const uint64_t inv2 = (pq + 1) / 2;
    uint64_t f = powmod(inv2, (uint64_t)(n - 1), pq);
    f = f * powmod(((uint64_t)1 << 32) % pq, (uint64_t)(NG - 1), pq) % pq;
    if ((n - 1) & 1) f = (pq - f) % pq;
    val = S * f % pq;
  }
  int64_t cf = coef ? coef[leaf] : 1;
  int64_t cm = cf % (int64_t)pq;
  if (cm < 0) cm += (int64_t)pq;
  val = val * (uint64_t)cm % pq;
  if (leaf_res) leaf_res[idx] = (uint32_t)val;
  if (job_acc) {
    atomicAdd(job_acc + (job ? (int64_t)job[leaf] : 0) * SPERM_KMAX + q, (unsigned long long)val);
    if (job) atomicAdd(job_acc + num_jobs * SPERM_KMAX + q, (unsigned long long)val);  // total row
  }
}

__global__ void reduce_mod_kernel(const unsigned long long* __restrict__ acc, int64_t rows,
                                  uint32_t* __restrict__ out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= rows * SPERM_KMAX) return;
  const uint32_t primes[SPERM_KMAX] = {2147483647u, 2147483629u, 2147483587u, 2147483579u,
                                       2147483563u, 2147483549u, 2147483543u, 2147483497u};
  out[idx] = (uint32_t)(acc[idx] % primes[idx % SPERM_KMAX]);
}

template <int NP>
int launch_main(const int32_t* mats, int n, int m, int cbits, const int32_t* order, const int2* meta,
                unsigned long long* queue, uint64_t total, unsigned long long* leaf_acc, cudaStream_t st) {
  using L = Layout<NP>;
  const size_t smem = (size_t)L::kWords * 4 * (kRnwThreads / 32);
  static bool attr_done = false;  // per process; single device per process in this framework
  if (!attr_done) {
    SPERM_CUDA(cudaFuncSetAttribute(rnw_main_kernel<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
    attr_done = true;
  }
  int per_sm = 0;
  SPERM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rnw_main_kernel<NP>, kRnwThreads, smem));
  if (per_sm < 1) per_sm = 1;
  uint64_t grid = (uint64_t)sm_count() * per_sm;
  const uint64_t warps_needed = total;
  const uint64_t blocks_needed = (warps_needed + kRnwThreads / 32 - 1) / (kRnwThreads / 32);
  if (grid > blocks_needed) grid = blocks_needed;
  if (grid < 1) grid = 1;
  TimingScope ts("rnw", st);
  rnw_main_kernel<NP><<<(unsigned)grid, kRnwThreads, smem, st>>>(mats, n, m, cbits, order, meta, queue, total,
                                                                 leaf_acc, make_primes());
  SPERM_LAUNCH_CHECK("rnw_main_kernel");
  return SPERM_OK;
}

}  // namespace
}  // namespace sperm

using namespace sperm;

extern "C" double sperm_rnw_terms(int n, int64_t count) {
  if (n <= 0) return (double)count;
  return (double)count * std::ldexp(1.0, n - 1);
}

extern "C" int sperm_reduce_mod(const uint64_t* d_acc, int64_t rows, uint32_t* d_out, void* stream) {
  if (rows < 0 || (rows > 0 && (!d_acc || !d_out))) return set_error(SPERM_ERR_ARG, "sperm_reduce_mod: bad args");
  if (rows == 0) return SPERM_OK;
  const int64_t tot = rows * SPERM_KMAX;
  reduce_mod_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      (const unsigned long long*)d_acc, rows, d_out);
  SPERM_LAUNCH_CHECK("reduce_mod_kernel");
  return SPERM_OK;
}

extern "C" int sperm_permanent(const int32_t* d_mats, int n, int64_t count, const int64_t* d_coef,
                               const int32_t* d_order, const int32_t* d_job, int64_t num_jobs,
                               int min_primes, uint32_t* d_leaf_res, int32_t* d_leaf_k,
                               uint64_t* d_job_acc, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 0 || n > SPERM_NMAX) return set_error(SPERM_ERR_ARG, "sperm_permanent: n out of range [0, 48]");
  if (count < 0) return set_error(SPERM_ERR_ARG, "sperm_permanent: count < 0");
  if (min_primes < 1 || min_primes > SPERM_KMAX)
    return set_error(SPERM_ERR_ARG, "sperm_permanent: min_primes out of range");
  if (count == 0) return SPERM_OK;
  if (n > 0 && !d_mats) return set_error(SPERM_ERR_ARG, "sperm_permanent: d_mats is NULL");
  if (d_job_acc && d_job && num_jobs <= 0) return set_error(SPERM_ERR_ARG, "sperm_permanent: num_jobs");
  const int NP = n <= 8 ? 8 : ((n + 7) / 8) * 8;

  int2* meta = nullptr;
  unsigned long long* leaf_acc = nullptr;
  unsigned long long* queue = nullptr;
  int* err = nullptr;
  SPERM_CUDA(cudaMallocAsync((void**)&meta, sizeof(int2) * count, st));
  SPERM_CUDA(cudaMallocAsync((void**)&leaf_acc, sizeof(unsigned long long) * count * SPERM_KMAX, st));
  SPERM_CUDA(cudaMallocAsync((void**)&queue, sizeof(unsigned long long) + sizeof(int) * 4, st));
  err = reinterpret_cast<int*>(queue + 1);
  SPERM_CUDA(cudaMemsetAsync(leaf_acc, 0, sizeof(unsigned long long) * count * SPERM_KMAX, st));
  SPERM_CUDA(cudaMemsetAsync(queue, 0, sizeof(unsigned long long) + sizeof(int) * 4, st));
  int rc = SPERM_OK;
  auto cleanup = [&]() {
    cudaFreeAsync(meta, st);
    cudaFreeAsync(leaf_acc, st);
    cudaFreeAsync(queue, st);
  };
  {
    TimingScope ts("rnw_prep", st);
    const int64_t threads = count * 32;
    rnw_prep_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(d_mats, n, NP, count, d_coef,
                                                                       min_primes, meta, err);
  }
  cudaError_t le = cudaGetLastError();
  if (le != cudaSuccess) { cleanup(); return cuda_check(le, "rnw_prep_kernel"); }
  int herr = 0;
  le = cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (le == cudaSuccess) le = cudaStreamSynchronize(st);
  if (le != cudaSuccess) { cleanup(); return cuda_check(le, "rnw_prep readback"); }
  if (herr & 1) { cleanup(); return set_error(SPERM_ERR_RANGE, "sperm_permanent: a row abs sum is >= 2^30"); }
  if (herr & 2) { cleanup(); return set_error(SPERM_ERR_PRIMES, "sperm_permanent: bound needs > 8 primes"); }

  if (n > 0) {
    const int tb = n - 1;  // log2 of the number of terms
    int m = std::max(0, std::min(kMaxLaneBits, tb - 5 - 6));
    int cbits = std::max(0, tb - 5 - m);
    const uint64_t total = (uint64_t)count << cbits;
    switch (NP) {
      case 8: rc = launch_main<8>(d_mats, n, m, cbits, d_order, meta, queue, total, leaf_acc, st); break;
      case 16: rc = launch_main<16>(d_mats, n, m, cbits, d_order, meta, queue, total, leaf_acc, st); break;
      case 24: rc = launch_main<24>(d_mats, n, m, cbits, d_order, meta, queue, total, leaf_acc, st); break;
      case 32: rc = launch_main<32>(d_mats, n, m, cbits, d_order, meta, queue, total, leaf_acc, st); break;
      case 40: rc = launch_main<40>(d_mats, n, m, cbits, d_order, meta, queue, total, leaf_acc, st); break;
      case 48: rc = launch_main<48>(d_mats, n, m, cbits, d_order, meta, queue, total, leaf_acc, st); break;
      default: rc = set_error(SPERM_ERR_ARG, "sperm_permanent: unsupported order");
    }
    if (rc != SPERM_OK) { cleanup(); return rc; }
  }
  {
    TimingScope ts("rnw_finalize", st);
    const int64_t tot = count * SPERM_KMAX;
    rnw_finalize_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(
        n, NP, count, meta, leaf_acc, d_coef, d_job, d_leaf_res, d_leaf_k,
        (unsigned long long*)d_job_acc, num_jobs);
  }
  le = cudaGetLastError();
  cleanup();
  if (le != cudaSuccess) return cuda_check(le, "rnw_finalize_kernel");
  return rc;
}
