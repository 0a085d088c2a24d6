// kklll.cu — Algorithm KKLLL: approximate permanents used as the
// job weights of the improved Step 3.
//
// Per (job, trial): n <= 32 one warp with B in shared memory (kklll_warp_kernel), n >= 48 one warp
// over the front of the sparse job matrix (kklll_front_kernel), else one CTA with B in shared
// memory (kklll_smem_kernel, also the frontal kernel's fallback).
//   Step 1: B_ij = 0 where a_ij = 0, else the cube root of unity w_r, r = root_index(
//           trial_key(seed, id, trial), i, j)  (counter-based SplitMix64; K1)
//   Step 2: X = |det B|^2 by LU with partial pivoting (first maximal |b_ik|^2), every real
//           operation a single IEEE round-to-nearest fp64 op in a fixed order with no
//           contraction (__dmul_rn/__dadd_rn/__dsub_rn; quotients correctly rounded, see
//           div_by; K2), so the value equals the reference evaluation bit for bit.
// The estimate is the trial-order sum of X divided by N (K3).
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace sperm {
namespace {

constexpr int kKNmax = 112;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t trial_key(uint64_t seed, uint64_t job, uint64_t trial) {
  const uint64_t h = mix64(seed + 0x9E3779B97F4A7C15ull * (job + 1));
  return mix64(h ^ (trial * 0xD1B54A32D192ED03ull));
}
__device__ __forceinline__ int root_index(uint64_t key, uint64_t i, uint64_t j) {
  const uint64_t h = mix64(key ^ ((i << 32) | j));
  return (int)(((h >> 32) * 3ull) >> 32);
}

// RN(a / d) for the step's pivot magnitude d > 0, given y = RN(1/d) (one __drcp_rn per
// elimination step instead of a full division per multiplier): q0 = RN(a y) is within one ulp
// of a/d, r = a - q0 d is exact (FMA), and RN(q0 + r y) is the correctly rounded quotient
// (Markstein's theorem), i.e. the same double as the reference's a / d.  The theorem needs no
// over/underflow in the intermediates: with |a| and d both in [2^-450, 2^450], a*y, q0 and the
// quotient stay in [2^-901, 2^901], far from overflow and from the subnormal range, so q0 has no
// double rounding; d_ok (warp-uniform) and the |a| range select the plain IEEE division
// otherwise.  A zero numerator returns a * y, which keeps the sign of a / d.
__device__ __forceinline__ bool div_range_ok(double v) {
  const double av = fabs(v);
  return av >= 0x1p-450 && av <= 0x1p450;
}
__device__ __forceinline__ double div_by(double a, double d, double y, bool d_ok) {
  if (!d_ok || (a != 0.0 && !div_range_ok(a))) return __ddiv_rn(a, d);
  const double q0 = __dmul_rn(a, y);
  if (a == 0.0) return q0;
  const double r = __fma_rn(-q0, d, a);
  return __fma_rn(r, y, q0);
}


// Shared-memory-resident variant for 32 < n <= 112: one 256-thread CTA per trial, B row-major
// in shared memory (16-byte complex entries), several trials (CTAs) per SM so one trial's
// pivot search and barriers overlap the others' updates.  Per elimination step: warp 0 finds the
// pivot (first maximal |b_ik|^2 over rows k..n-1, the oracle's rule on physically swapped rows),
// the rows k and p are swapped (columns >= k: earlier columns hold spent multipliers), the
// multipliers l_i go to a shared vector (one reciprocal per step + Markstein, div_by), and
// the m x m trailing block is updated by all threads (thread = (row group, column): contiguous
// 16-byte accesses, the multiplier a broadcast).  Same operations in the same order as the
// oracle on every entry, so X is bit-identical.  Updates by a zero pivot-row entry u = 0 are
// skipped (the pivot row is sparse until fill-in): every b_ij - l_i * 0 is b_ij up to the sign
// of a zero, and a zero's sign never reaches a pivot magnitude |b|^2, a nonzero sum or the
// product of the d_k — so X is bit-identical with the update skipped.
// pivot of column k (rows >= k): first row with maximal re^2 + im^2 — per lane ascending with a
// strict >, then a (larger value, then smaller row) butterfly; lane 0 publishes it, and the last
// row of the column holding a nonzero entry (the multipliers below it are zero)
__device__ __forceinline__ void pivot_reduce(double bm, int bi, int last, int lane, double& s_d, int& s_p,
                                             int& s_last) {
  for (int o = 16; o; o >>= 1) {
    const double om = __shfl_xor_sync(0xffffffffu, bm, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (om > bm || (om == bm && oi < bi)) { bm = om; bi = oi; }
  }
  last = __reduce_max_sync(0xffffffffu, last);
  if (lane == 0) {
    s_d = bm;
    s_p = bi;
    s_last = last;
  }
}
__device__ __forceinline__ void pivot_scan(const double2* b, int ns, int n, int k, int lane, double& s_d,
                                           int& s_p, int& s_last) {
  double bm = -1.0;
  int bi = n, last = -1;
  for (int i = k + lane; i < n; i += 32) {
    const double2 v = b[i * ns + k];
    const double mg = __dadd_rn(__dmul_rn(v.x, v.x), __dmul_rn(v.y, v.y));
    if (mg > bm) { bm = mg; bi = i; }
    if (v.x != 0.0 || v.y != 0.0) last = i;
  }
  pivot_reduce(bm, bi, last, lane, s_d, s_p, s_last);
}

// Per elimination step only rows k+1..rmax are updated, rmax = the last row with a nonzero entry
// in column k (every multiplier below it is zero; warp 0 finds it in the pivot search), and
// columns whose pivot-row entry u_j is zero are skipped.  A skipped entry b_ij - l_i u_j with
// l_i = 0 or u_j = 0 equals b_ij up to the sign of a zero, which never reaches |b|^2, a nonzero
// sum or the d_k, so X stays bit-identical while the work follows the band of the sparse job
// matrices (their fill-in stays near the diagonal) instead of the full (n-k)^2 trailing block.
// (Measured: an exact last-nonzero-column bound of the pivot row, found by a warp reduction and
// a shared atomic in the exchange phase, doubled the step time — that phase is on every step's
// critical path — so columns are only skipped by their zero u_j.)
template <int NT>
__global__ void __launch_bounds__(NT) kklll_smem_kernel(const int32_t* __restrict__ mats, int n, int64_t count,
                                                                const int32_t* __restrict__ ids, int trials,
                                                                uint64_t seed, double* __restrict__ xout, int band) {
  extern __shared__ double2 ksm2[];  // b[n][ns] (row stride ns = n | 1: column scans conflict-free) | lv[n]
  const int ns = n | 1;
  double2* b = ksm2;
  double2* lv = ksm2 + n * ns;
  __shared__ double s_d;
  __shared__ int s_p, s_last;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const double S32 = 0.8660254037844386;
  const int64_t items = count * (int64_t)trials;
  for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
    const int64_t job = item / trials;
    const int trial = (int)(item % trials);
    const int32_t* a = mats + job * (int64_t)n * n;
    const uint64_t key = trial_key(seed, (uint64_t)(ids ? ids[job] : job), (uint64_t)trial);
    __syncthreads();  // the previous trial is done with b
    for (int e = t; e < n * n; e += NT) {
      const int i = e / n, j = e - (e / n) * n;
      double r = 0.0, s = 0.0;
      if (a[e] != 0) {
        const int ri = root_index(key, (uint64_t)i, (uint64_t)j);
        r = ri == 0 ? 1.0 : -0.5;
        s = ri == 0 ? 0.0 : (ri == 1 ? S32 : -S32);
      }
      b[i * ns + j] = make_double2(r, s);
    }
    __syncthreads();
    double x = 1.0;
    if (w == 0) pivot_scan(b, ns, n, 0, lane, s_d, s_p, s_last);  // later pivots come out of the update
    __syncthreads();
    for (int k = 0; k < n; ++k) {
      const double d = s_d;
      const int p = s_p;
      const int rmax = band ? s_last : n - 1;
      if (d == 0.0) { x = 0.0; break; }  // CTA-uniform
      x = __dmul_rn(x, d);
      if (k + 1 == n) break;
      // one phase, one barrier: the row exchange of columns > k (column k is never read again
      // for X) and the multipliers of rows k+1..rmax, which read column k only — with the
      // exchange applied on the fly: the pivot value is row p's, and row i = p (after the
      // exchange: old row k) reads row k's
      if (p != k)
        for (int j = k + 1 + t; j < n; j += NT) {
          const double2 u = b[k * ns + j];
          b[k * ns + j] = b[p * ns + j];
          b[p * ns + j] = u;
        }
      {
        const double2 pk = b[p * ns + k];
        const double y = __drcp_rn(d);
        const bool d_ok = div_range_ok(d);
        for (int i = k + 1 + t; i <= rmax; i += NT) {
          const double2 v = b[(i == p ? k : i) * ns + k];
          lv[i] = make_double2(div_by(__dadd_rn(__dmul_rn(v.x, pk.x), __dmul_rn(v.y, pk.y)), d, y, d_ok),
                               div_by(__dsub_rn(__dmul_rn(v.y, pk.x), __dmul_rn(v.x, pk.y)), d, y, d_ok));
        }
      }
      __syncthreads();
      if (w == 0) {
        // warp 0: column k+1 (the next pivot column) in rows k+1..rmax, then the next pivot search
        // over the whole column while the update of columns > k+1 is still running — s_d/s_p/s_last
        // were last read before the barrier
        const int j = k + 1;
        const double2 u = b[k * ns + j];
        const bool nz = u.x != 0.0 || u.y != 0.0;
        double bm = -1.0;
        int bi = n, last = -1;
        for (int i = j + lane; i < n; i += 32) {
          double2 v = b[i * ns + j];
          if (nz && i <= rmax) {
            const double2 l = lv[i];
            v.x = __dsub_rn(v.x, __dsub_rn(__dmul_rn(l.x, u.x), __dmul_rn(l.y, u.y)));
            v.y = __dsub_rn(v.y, __dadd_rn(__dmul_rn(l.x, u.y), __dmul_rn(l.y, u.x)));
            b[i * ns + j] = v;
          }
          const double mg = __dadd_rn(__dmul_rn(v.x, v.x), __dmul_rn(v.y, v.y));
          if (mg > bm) { bm = mg; bi = i; }
          if (v.x != 0.0 || v.y != 0.0) last = i;
        }
        pivot_reduce(bm, bi, last, lane, s_d, s_p, s_last);
      } else if (rmax > k) {
        // columns k+2..n-1, rows k+1..rmax: thread t' = t - 32 -> column j = k+2 + t' % m, rows
        // k+1 + t' / m + G * r; when the m columns outnumber the NT - 32 threads, whole columns
        // j = k+2 + t' + (NT-32) * c
        const int m = n - k - 2;
        const int tt = t - 32;
        auto column = [&](int j, int g, int G) {
          const double2 u = b[k * ns + j];
          if (u.x != 0.0 || u.y != 0.0) {
#pragma unroll 4
            for (int i = k + 1 + g; i <= rmax; i += G) {
              const double2 l = lv[i];
              double2 v = b[i * ns + j];
              v.x = __dsub_rn(v.x, __dsub_rn(__dmul_rn(l.x, u.x), __dmul_rn(l.y, u.y)));
              v.y = __dsub_rn(v.y, __dadd_rn(__dmul_rn(l.x, u.y), __dmul_rn(l.y, u.x)));
              b[i * ns + j] = v;
            }
          }
        };
        static_assert(kKNmax - 2 < 256 - 32, "256 threads cover every trailing column");
        if (NT < 256 && m >= NT - 32) {
          for (int jj = tt; jj < m; jj += NT - 32) column(k + 2 + jj, 0, 1);
        } else if (m > 0) {
          const int G = (NT - 32) / m;
          const int g = tt / m;
          if (g < G) column(k + 2 + (tt - g * m), g, G);
        }
      }
      __syncthreads();
    }
    if (t == 0) xout[item] = x;
  }
}

// ---------------------------------------------------------------------------- warp kernel
// One WARP per trial for orders n <= 32, B row-major in shared memory (row stride 33 double2: a
// lane-per-column row access and a lane-per-row column access are both bank-conflict-free).
// Lane j owns column j in the row operations (exchange, update) and row j in the column
// operations (pivot search, multipliers), so a step needs no CTA barrier, only __syncwarp:
//   pivot: lane i reads b_ik, |b_ik|^2, two REDUX maxima over the bit pattern (non-negative
//          doubles order like their bits) and a ballot give the first maximal row p;
//   exchange rows k, p in columns >= k (physically, as the oracle does);
//   multipliers l_i of the rows with a nonzero b_ik (correctly rounded quotients, div_by) go to
//   shared memory; the rows are then visited in turn (warp-uniform bit loop over their ballot),
//   each lane updating its column if its pivot-row entry u_j is nonzero.
// Rows with b_ik = 0 and columns with u_j = 0 are skipped (b - l u = b up to the sign of a zero,
// see above), every other operation is the oracle's on the same entry in the same order: X is
// bit-identical.  Each warp takes a contiguous range of (job, trial) items, so the job's column
// supports (a 32-bit row mask per lane) are rebuilt only when the job changes; a trial's B is
// zero-filled and its nonzeros drawn by iterating the lane's mask.
constexpr int kWarpNS = 33;
__global__ void __launch_bounds__(32) kklll_warp_kernel(const int32_t* __restrict__ mats, int n, int64_t count,
                                                        const int32_t* __restrict__ ids, int trials, uint64_t seed,
                                                        double* __restrict__ xout) {
  extern __shared__ double2 wsm2[];  // b[n][33] | lv[32]
  double2* b = wsm2;
  double2* lv = wsm2 + n * kWarpNS;
  const int lane = threadIdx.x;
  const unsigned FULL = 0xffffffffu;
  const double S32 = 0.8660254037844386;
  const int64_t items = count * (int64_t)trials;
  const int64_t per = (items + gridDim.x - 1) / gridDim.x;
  int64_t item = (int64_t)blockIdx.x * per;
  const int64_t end = item + per < items ? item + per : items;
  if (item >= end) return;
  int64_t job = item / trials;
  int trial = (int)(item - job * trials);
  int64_t cur_job = -1;
  uint32_t colmask = 0;  // rows with a nonzero in column `lane` of the job's pattern
  uint64_t jid = 0;
  for (; item < end; ++item) {
    if (job != cur_job) {
      const int32_t* a = mats + job * (int64_t)n * n;
      colmask = 0;
      for (int i = 0; i < n; ++i)
        if (lane < n && a[i * n + lane] != 0) colmask |= 1u << i;
      jid = (uint64_t)(ids ? ids[job] : job);
      cur_job = job;
    }
    const uint64_t key = trial_key(seed, jid, (uint64_t)trial);
    __syncwarp();  // the previous trial is done with b
    for (int i = 0; i < n; ++i) b[i * kWarpNS + lane] = make_double2(0.0, 0.0);
    for (uint32_t mk = colmask; mk; mk &= mk - 1) {
      const int i = __ffs(mk) - 1;
      const int ri = root_index(key, (uint64_t)i, (uint64_t)lane);
      b[i * kWarpNS + lane] = make_double2(ri == 0 ? 1.0 : -0.5, ri == 0 ? 0.0 : (ri == 1 ? S32 : -S32));
    }
    __syncwarp();
    double x = 1.0;
    for (int k = 0; k < n; ++k) {
      const bool inr = lane >= k && lane < n;
      double2 v = make_double2(0.0, 0.0);
      if (inr) v = b[lane * kWarpNS + k];
      const double mg = __dadd_rn(__dmul_rn(v.x, v.x), __dmul_rn(v.y, v.y));
      const unsigned long long bits = (unsigned long long)__double_as_longlong(mg);
      const unsigned hi = inr ? (unsigned)(bits >> 32) : 0u;
      const unsigned mh = __reduce_max_sync(FULL, hi);
      const bool c1 = inr && hi == mh;
      const unsigned lo = c1 ? (unsigned)bits : 0u;
      const unsigned ml = __reduce_max_sync(FULL, lo);
      const unsigned win = __ballot_sync(FULL, c1 && lo == ml);
      const int p = __ffs(win) - 1;  // first maximal row (lane k is always in range: win != 0)
      const double d = __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
      if (d == 0.0) { x = 0.0; break; }  // warp-uniform
      x = __dmul_rn(x, d);
      if (k + 1 == n) break;
      double2 u = make_double2(0.0, 0.0);  // my column's entry of the pivot row (after the exchange)
      if (p != k) {
        if (inr) {
          const double2 t0 = b[k * kWarpNS + lane];
          u = b[p * kWarpNS + lane];
          b[k * kWarpNS + lane] = u;
          b[p * kWarpNS + lane] = t0;
        }
        __syncwarp();
      } else if (inr) {
        u = b[k * kWarpNS + lane];
      }
      const double2 pk = b[k * kWarpNS + k];  // broadcast
      const double y = __drcp_rn(d);
      const bool d_ok = div_range_ok(d);
      const bool below = lane > k && lane < n;
      double2 vi = make_double2(0.0, 0.0);
      if (below) vi = b[lane * kWarpNS + k];
      const bool nzr = vi.x != 0.0 || vi.y != 0.0;
      const unsigned rows = __ballot_sync(FULL, nzr);
      if (nzr)
        lv[lane] = make_double2(div_by(__dadd_rn(__dmul_rn(vi.x, pk.x), __dmul_rn(vi.y, pk.y)), d, y, d_ok),
                                div_by(__dsub_rn(__dmul_rn(vi.y, pk.x), __dmul_rn(vi.x, pk.y)), d, y, d_ok));
      __syncwarp();
      const bool unz = below && (u.x != 0.0 || u.y != 0.0);
      // four rows per pass (independent load -> multiply -> subtract -> store chains in flight)
      for (unsigned r = rows; r;) {
        int ri[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          ri[q] = __ffs(r) - 1;  // -1 once the rows run out (warp-uniform)
          r &= r - 1;
        }
        if (unz) {
          double2 l[4], w[4];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (ri[q] >= 0) {
              l[q] = lv[ri[q]];
              w[q] = b[ri[q] * kWarpNS + lane];
            }
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (ri[q] >= 0) {
              w[q].x = __dsub_rn(w[q].x, __dsub_rn(__dmul_rn(l[q].x, u.x), __dmul_rn(l[q].y, u.y)));
              w[q].y = __dsub_rn(w[q].y, __dadd_rn(__dmul_rn(l[q].x, u.y), __dmul_rn(l[q].y, u.x)));
              b[ri[q] * kWarpNS + lane] = w[q];
            }
        }
      }
      __syncwarp();
    }
    if (lane == 0) xout[item] = x;
    if (++trial == trials) { trial = 0; ++job; }
  }
}

// ---------------------------------------------------------------------------- frontal kernel
// One WARP per trial for the sparse job matrices (round 2).  Partial pivoting keeps the fill of a
// sparse matrix near the diagonal, so at step k only a FRONT of rows (not yet eliminated, first
// original nonzero column <= k: every other row is still zero in columns <= k) and a WINDOW of
// columns k..E (E = the largest last-nonzero column of a pivot row so far: every column right
// of it is untouched) can change.  The front (<= kFrR rows, one lane each) is kept in shared
// memory over a circular window of kFrC columns; a row entering the front, and a column entering
// the window, is initialised from the job matrix and the trial's roots (counter-based, so any
// entry can be regenerated).  Every update is the oracle's operation on the same entry in the same
// order (a skipped entry b - l u has l = 0 or u = 0: b up to the sign of a zero, see above), the
// multipliers the same correctly rounded quotients, and the pivot the first maximal |b_ik|^2 by
// POSITION — each row's position under the oracle's physical row swaps is tracked (rowAt/posOf)
// — so X is bit-identical to the oracle's.  A job whose front or window overflows (or whose rows
// have more than kNzRow nonzeros) is flagged and re-run by the CTA kernel above.
constexpr int kFrR = 24;    // front rows (lanes 0..23)
constexpr int kFrC = 64;    // window columns (circular, power of two)
#ifndef SPERM_KKLLL_FRONT_STRIDE  // row stride of the front in double2: 65 spreads the rows of one
#define SPERM_KKLLL_FRONT_STRIDE 65  // column over the banks (at 64 every row of a column shares them)
#endif
constexpr int kFrS = SPERM_KKLLL_FRONT_STRIDE;
constexpr int kNzRow = 12;  // original nonzeros per row in the row table
constexpr int kRowTab = 2 + kNzRow;

// per job and row: first nonzero column, nonzero count, the nonzero columns ascending (int8);
// over[job] = 1 if a row has more than kNzRow nonzeros.  One warp per job.
__global__ void kklll_rowtab_kernel(const int32_t* __restrict__ mats, int n, int64_t count, int8_t* __restrict__ tab,
                                    int* __restrict__ over) {
  const int lane = threadIdx.x & 31;
  const int64_t job = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (job >= count) return;
  const int32_t* a = mats + job * (int64_t)n * n;
  int8_t* t = tab + job * (int64_t)n * kRowTab;
  bool bad = false;
  for (int i = lane; i < n; i += 32) {
    int c = 0, first = n;
    for (int j = 0; j < n; ++j)
      if (a[i * n + j] != 0) {
        if (c < kNzRow) t[i * kRowTab + 2 + c] = (int8_t)j;
        first = min(first, j);
        ++c;
      }
    if (c > kNzRow) bad = true;
    t[i * kRowTab] = (int8_t)first;
    t[i * kRowTab + 1] = (int8_t)min(c, kNzRow);
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) over[job] = 1;
}

__global__ void __launch_bounds__(32) kklll_front_kernel(int n, int64_t count, const int32_t* __restrict__ ids,
                                                           int trials, uint64_t seed, const int8_t* __restrict__ tab,
                                                           double* __restrict__ xout, int* __restrict__ over) {
  // F[kFrR][kFrS] | rowAt[128] posOf[128] | the current job's row table [n][kRowTab] (int8)
  extern __shared__ double2 fsm[];
  double2* F = fsm;
  int8_t* rowAt = reinterpret_cast<int8_t*>(fsm + kFrR * kFrS);
  int8_t* posOf = rowAt + 128;
  int8_t* rts = posOf + 128;
  const int lane = threadIdx.x;
  const double S32 = 0.8660254037844386;
  const int64_t items = count * (int64_t)trials;
  int64_t cached = -1;
  int fz[4];  // first nonzero column of rows lane, lane + 32, lane + 64, lane + 96
  for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
    const int64_t job = item / trials;
    const int trial = (int)(item % trials);
    if (over[job]) continue;  // the CTA kernel recomputes the job
    const uint64_t key = trial_key(seed, (uint64_t)(ids ? ids[job] : job), (uint64_t)trial);
    __syncwarp();
    if (job != cached) {  // the job's row table into shared memory (trials of a job follow each other)
      const int8_t* rt = tab + job * (int64_t)n * kRowTab;
      for (int e = lane; e < n * kRowTab; e += 32) rts[e] = rt[e];
      cached = job;
      __syncwarp();
#pragma unroll
      for (int t = 0; t < 4; ++t) fz[t] = lane + 32 * t < n ? rts[(lane + 32 * t) * kRowTab] : 127;
    }
    for (int i = lane; i < n; i += 32) {
      rowAt[i] = (int8_t)i;
      posOf[i] = (int8_t)i;
    }
    __syncwarp();
    // the lane's front row: original index (-1: free slot) and current position
    int myrow = -1, mypos = 0;
    unsigned freem = (1u << kFrR) - 1u;  // free slots (warp-uniform)
    double2* my = F + min(lane, kFrR - 1) * kFrS;  // lanes >= kFrR never own a row (reads only)
    int E = -1;         // window right edge
    bool fail = false;  // front or window overflow
    // the lane's row over window columns lo..hi: zeros, then its original nonzeros (Step 1 of KKLLL:
    // the trial's cube roots, regenerated from the counter-based generator)
    auto init_cols = [&](int lo, int hi) {
      if (myrow < 0 || lo > hi) return;
      for (int j = lo; j <= hi; ++j) my[j & (kFrC - 1)] = make_double2(0.0, 0.0);
      const int8_t* r = rts + myrow * kRowTab;
      const int c = r[1];
      for (int t = 0; t < c; ++t) {
        const int j = r[2 + t];
        if (j >= lo && j <= hi) {
          const int ri = root_index(key, (uint64_t)myrow, (uint64_t)j);
          my[j & (kFrC - 1)] = make_double2(ri == 0 ? 1.0 : -0.5, ri == 0 ? 0.0 : (ri == 1 ? S32 : -S32));
        }
      }
    };
    double x = 1.0;
    for (int k = 0; k < n; ++k) {
      // window covers column k (columns E+1..k enter: original values of the front rows)
      if (E < k) {
        init_cols(E + 1, k);
        E = k;
      }
      // rows whose first nonzero is column k enter the front
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        if (32 * t >= n) break;
        unsigned ent = __ballot_sync(0xffffffffu, fz[t] == k);
        while (ent) {
          const int row = 32 * t + __ffs(ent) - 1;
          ent &= ent - 1;
          if (!freem) {
            fail = true;
            break;
          }
          const int slot = __ffs(freem) - 1;
          freem &= freem - 1;
          if (lane == slot) {
            myrow = row;
            mypos = posOf[row];
            init_cols(k, E);
          }
        }
      }
      if (fail) break;
      __syncwarp();
      // pivot: first maximal |b_ik|^2 by position over the front (a nonnegative double orders
      // like its bit pattern: two 32-bit REDUX, then the minimal position)
      const double2 bk = myrow >= 0 ? my[k & (kFrC - 1)] : make_double2(0.0, 0.0);
      const double mag = myrow >= 0 ? __dadd_rn(__dmul_rn(bk.x, bk.x), __dmul_rn(bk.y, bk.y)) : 0.0;
      const unsigned mh = myrow >= 0 ? (unsigned)__double2hiint(mag) : 0u;
      const unsigned ml = myrow >= 0 ? (unsigned)__double2loint(mag) : 0u;
      const unsigned bh = __reduce_max_sync(0xffffffffu, mh);
      const bool c1 = myrow >= 0 && mh == bh;
      const unsigned bl_ = __reduce_max_sync(0xffffffffu, c1 ? ml : 0u);
      const bool c2 = c1 && ml == bl_;
      const int bp = (int)__reduce_min_sync(0xffffffffu, c2 ? (unsigned)mypos : 0xffffffffu);
      const int ps = __ffs(__ballot_sync(0xffffffffu, c2 && mypos == bp)) - 1;  // pivot lane
      const double d = __hiloint2double((int)bh, (int)bl_);
      if (d == 0.0 || ps < 0) {
        x = 0.0;
        break;
      }
      x = __dmul_rn(x, d);
      if (k + 1 == n) break;
      const int prow = __shfl_sync(0xffffffffu, myrow, ps);
      const double2* pr = F + ps * kFrS;
      // the pivot row's last nonzero: an original nonzero right of the window extends it
      {
        const int8_t* r = rts + prow * kRowTab;
        const int c = r[1];
        const int cl = c > 0 ? r[2 + c - 1] : -1;
        if (cl > E) {
          if (cl - k + 1 > kFrC) {
            fail = true;
            break;
          }
          init_cols(E + 1, cl);
          E = cl;
          __syncwarp();
        }
      }
      // the pivot row's nonzero columns k+1..E as a bit mask of offsets j - k - 1 (< 63)
      unsigned long long um = 0;
      for (int j0 = k + 1; j0 <= E; j0 += 32) {
        const int j = j0 + lane;
        bool nz = false;
        if (j <= E) {
          const double2 u = pr[j & (kFrC - 1)];
          nz = u.x != 0.0 || u.y != 0.0;
        }
        um |= (unsigned long long)__ballot_sync(0xffffffffu, nz) << (j0 - k - 1);
      }
      // multipliers l_i = b_ik conj(b_kk) / |b_kk|^2 (one reciprocal + Markstein, as above), then
      // the update of the pivot row's nonzero columns, four independent columns per step
      const double2 pk = pr[k & (kFrC - 1)];
      double2 l = make_double2(0.0, 0.0);
      const bool act = myrow >= 0 && lane != ps && (bk.x != 0.0 || bk.y != 0.0);
      if (act) {
        const double y = __drcp_rn(d);
        const bool d_ok = div_range_ok(d);
        l = make_double2(div_by(__dadd_rn(__dmul_rn(bk.x, pk.x), __dmul_rn(bk.y, pk.y)), d, y, d_ok),
                         div_by(__dsub_rn(__dmul_rn(bk.y, pk.x), __dmul_rn(bk.x, pk.y)), d, y, d_ok));
      }
      while (um) {
        int jj[4];
        bool ok[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          ok[t] = um != 0;
          jj[t] = ok[t] ? (k + 1 + __ffsll((long long)um) - 1) & (kFrC - 1) : 0;
          um &= um - 1;
        }
        double2 u[4], v[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          u[t] = pr[jj[t]];
          v[t] = my[jj[t]];
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          if (act && ok[t]) {
            v[t].x = __dsub_rn(v[t].x, __dsub_rn(__dmul_rn(l.x, u[t].x), __dmul_rn(l.y, u[t].y)));
            v[t].y = __dsub_rn(v[t].y, __dadd_rn(__dmul_rn(l.x, u[t].y), __dmul_rn(l.y, u[t].x)));
            my[jj[t]] = v[t];
          }
        }
      }
      // the oracle's row exchange: the row at position k moves to the pivot's position
      const int pp = __shfl_sync(0xffffffffu, mypos, ps);
      const int rk = rowAt[k];
      __syncwarp();
      if (lane == 0) {
        rowAt[pp] = (int8_t)rk;
        posOf[rk] = (int8_t)pp;
        rowAt[k] = (int8_t)prow;
        posOf[prow] = (int8_t)k;
      }
      if (myrow == rk) mypos = pp;
      // the pivot row leaves the front
      if (lane == ps) myrow = -1;
      freem |= 1u << ps;
      __syncwarp();
    }
    if (fail) {
      if (lane == 0) over[job] = 1;
    } else if (lane == 0) {
      xout[item] = x;
    }
  }
}

__global__ void kklll_mean_kernel(const double* __restrict__ xs, int64_t count, int trials,
                                  double* __restrict__ est) {
  const int64_t job = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (job >= count) return;
  const double* x = xs + job * (int64_t)trials;
  double s = 0.0;
  for (int t = 0; t < trials; ++t) s = __dadd_rn(s, x[t]);
  est[job] = __ddiv_rn(s, (double)trials);
}

}  // namespace
}  // namespace sperm

using namespace sperm;

static std::mutex g_front_mu;
static double g_front_jobs = 0.0, g_front_redo = 0.0;

// jobs estimated through the frontal kernel path and jobs it handed to the CTA kernel (overflow)
extern "C" int sperm_estimate_stats(double* h_jobs, double* h_redo, int reset) {
  std::lock_guard<std::mutex> lk(g_front_mu);
  if (h_jobs) *h_jobs = g_front_jobs;
  if (h_redo) *h_redo = g_front_redo;
  if (reset) g_front_jobs = g_front_redo = 0.0;
  return SPERM_OK;
}

extern "C" int sperm_estimate(const int32_t* d_mats, int n, int64_t count, const int32_t* d_ids, int trials,
                              uint64_t seed, double* d_est, double* d_trials_out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  keep_pool_memory();
  if (n < 1 || n > kKNmax) return set_error(SPERM_ERR_ARG, "sperm_estimate: n out of range [1, 112]");
  if (count < 0) return set_error(SPERM_ERR_ARG, "sperm_estimate: count < 0");
  if (trials <= 0) trials = n * n;
  if (count == 0) return SPERM_OK;
  if (!d_mats || !d_est) return set_error(SPERM_ERR_ARG, "sperm_estimate: NULL pointer");
  double* xs = d_trials_out;
  if (!xs) SPERM_CUDA(cudaMallocAsync((void**)&xs, sizeof(double) * count * trials, st));
  const int64_t items = count * (int64_t)trials;
  // orders warp_min..32 take the warp-per-trial kernel, the rest the CTA / frontal kernels (A-B knob
  // SPERM_KKLLL_WARP_MIN, read per call; measured: C60 jobs of order 32 16.9 ms vs 32.1 ms for the
  // 64-thread CTA kernel; 2000 3-regular matrices x n^2 trials at n = 12 / 16 / 20 / 24 / 27: 0.89 /
  // 2.2 / 4.8 / 8.9 / 14.7 ms vs 1.6 / 3.3 / 11.1 / 16.9 / 58.2 ms for the register-resident kernel
  // of earlier versions, which it replaced)
  const int warp_min = [] {
    const char* e = getenv("SPERM_KKLLL_WARP_MIN");
    return e ? atoi(e) : 1;
  }();
  if (n <= 32 && n >= warp_min) {
    const size_t wsmem = sizeof(double2) * ((size_t)n * kWarpNS + 32);
    static std::atomic<unsigned> wattr{0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(wattr.load() & (1u << (dev & 31)))) {
      SPERM_CUDA(cudaFuncSetAttribute(kklll_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)(sizeof(double2) * (32 * kWarpNS + 32))));
      wattr.fetch_or(1u << (dev & 31));
    }
    int per_sm = 0;
    SPERM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kklll_warp_kernel, 32, wsmem));
    int64_t grid = (int64_t)sm_count() * std::max(per_sm, 1);
    grid = std::max<int64_t>(1, std::min(grid, items));
    TimingScope ts("kklll", st);
    count_launch();
    kklll_warp_kernel<<<(unsigned)grid, 32, wsmem, st>>>(d_mats, n, count, d_ids, trials, seed, xs);
    SPERM_LAUNCH_CHECK("kklll_warp_kernel");
  } else {
    // shared-memory-resident LU, one CTA per trial (smem_kernel on jobs [j0, j0 + cnt) of the
    // given matrices / ids, trials written to out)
    auto run_smem = [&](const int32_t* mats, int64_t cnt, const int32_t* idsp, double* out) -> int {
      // (measured on the fullerene-96 jobs: 128 threads 1.37 s, 256 1.31 s, 512 1.97 s)
      // (128-thread CTAs below order SPERM_KKLLL_T128_MAX: more trials per SM, cheaper barriers)
      // (measured, 128 vs 256 threads: C60 jobs, order 32: 44.5 vs 75.1 ms; fullerene-96, order 67:
      // 1287 vs 1080 ms; C100, order 72: 2595 vs 1919 ms — bit-identical trials either way)
      static const int t128_max = [] {
        const char* e = getenv("SPERM_KKLLL_T128_MAX");
        return e ? atoi(e) : 48;
      }();
      static const int t64_max = [] {  // 64-thread CTAs below this order (C60 jobs: 39.8 vs 44.5 ms)
        const char* e = getenv("SPERM_KKLLL_T64_MAX");
        return e ? atoi(e) : 40;
      }();
      const int nt = n < t64_max ? 64 : n < t128_max ? 128 : 256;
      auto kern = nt == 64 ? kklll_smem_kernel<64> : nt == 128 ? kklll_smem_kernel<128> : kklll_smem_kernel<256>;
      const size_t smem = sizeof(double2) * ((size_t)n * (n | 1) + n);
      SPERM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      int per_sm = 0;
      SPERM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nt, smem));
      const int64_t it = cnt * (int64_t)trials;
      int64_t grid = (int64_t)sm_count() * std::max(per_sm, 1);
      grid = std::max<int64_t>(1, std::min(grid, it));
      static const int band = [] {  // A-B knob: SPERM_KKLLL_BAND=0 updates the whole trailing block
        const char* e = getenv("SPERM_KKLLL_BAND");
        return e ? atoi(e) : 1;
      }();
      count_launch();
      kern<<<(unsigned)grid, nt, smem, st>>>(mats, n, cnt, idsp, trials, seed, out, band);
      SPERM_LAUNCH_CHECK("kklll_smem_kernel");
      return SPERM_OK;
    };
    static const int front_min = [] {  // A-B knob: smallest order for the frontal kernel
      const char* e = getenv("SPERM_KKLLL_FRONT_MIN");  // (measured: C60 jobs, order 32: 68 ms frontal
      return e ? atoi(e) : 48;  // vs 32 ms CTA; C100 order 79: 254 vs 377 ms; fullerene-96 order 67: 764 vs 904)
    }();
    TimingScope ts("kklll", st);
    if (n < front_min) {
      const int rc = run_smem(d_mats, count, d_ids, xs);
      if (rc != SPERM_OK) return rc;
    } else {
      // frontal warp-per-trial kernel; jobs it flags (front / window / row-table overflow) are
      // re-run by the CTA kernel
      int8_t* tab = nullptr;
      int* over = nullptr;
      SPERM_CUDA(cudaMallocAsync((void**)&tab, (size_t)count * n * kRowTab, st));
      SPERM_CUDA(cudaMallocAsync((void**)&over, sizeof(int) * count, st));
      SPERM_CUDA(cudaMemsetAsync(over, 0, sizeof(int) * count, st));
      count_launch();
      kklll_rowtab_kernel<<<(unsigned)((count * 32 + 127) / 128), 128, 0, st>>>(d_mats, n, count, tab, over);
      SPERM_LAUNCH_CHECK("kklll_rowtab_kernel");
      const size_t fsmem = sizeof(double2) * kFrR * kFrS + 256 + (size_t)kKNmax * kRowTab;
      static std::atomic<unsigned> attr_done{0};
      int dev = 0;
      cudaGetDevice(&dev);
      if (!(attr_done.load() & (1u << (dev & 31)))) {
        SPERM_CUDA(cudaFuncSetAttribute(kklll_front_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsmem));
        attr_done.fetch_or(1u << (dev & 31));
      }
      int per_sm = 0;
      SPERM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kklll_front_kernel, 32, fsmem));
      int64_t grid = (int64_t)sm_count() * std::max(per_sm, 1);
      grid = std::max<int64_t>(1, std::min(grid, items));
      count_launch();
      kklll_front_kernel<<<(unsigned)grid, 32, fsmem, st>>>(n, count, d_ids, trials, seed, tab, xs, over);
      SPERM_LAUNCH_CHECK("kklll_front_kernel");
      std::vector<int> h_over((size_t)count);
      SPERM_CUDA(cudaMemcpyAsync(h_over.data(), over, sizeof(int) * count, cudaMemcpyDeviceToHost, st));
      cudaFreeAsync(tab, st);
      cudaFreeAsync(over, st);
      SPERM_CUDA(cudaStreamSynchronize(st));
      std::vector<int64_t> redo;
      for (int64_t j = 0; j < count; ++j)
        if (h_over[j]) redo.push_back(j);
      {
        std::lock_guard<std::mutex> lk(g_front_mu);
        g_front_jobs += (double)count;
        g_front_redo += (double)redo.size();
      }
      if (!redo.empty()) {
        // the flagged jobs, gathered, through the CTA kernel, scattered back
        const int64_t r = (int64_t)redo.size();
        int32_t* gm = nullptr;
        int32_t* gi = nullptr;
        double* gx = nullptr;
        SPERM_CUDA(cudaMallocAsync((void**)&gm, sizeof(int32_t) * r * n * n, st));
        SPERM_CUDA(cudaMallocAsync((void**)&gi, sizeof(int32_t) * r, st));
        SPERM_CUDA(cudaMallocAsync((void**)&gx, sizeof(double) * r * trials, st));
        std::vector<int32_t> h_ids((size_t)r);
        for (int64_t t = 0; t < r; ++t) {
          SPERM_CUDA(cudaMemcpyAsync(gm + t * n * n, d_mats + redo[t] * n * n, sizeof(int32_t) * n * n,
                                     cudaMemcpyDeviceToDevice, st));
          if (d_ids)
            SPERM_CUDA(cudaMemcpyAsync(gi + t, d_ids + redo[t], sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
          else
            h_ids[t] = (int32_t)redo[t];
        }
        if (!d_ids) SPERM_CUDA(cudaMemcpyAsync(gi, h_ids.data(), sizeof(int32_t) * r, cudaMemcpyHostToDevice, st));
        const int rc = run_smem(gm, r, gi, gx);
        if (rc != SPERM_OK) return rc;
        for (int64_t t = 0; t < r; ++t)
          SPERM_CUDA(cudaMemcpyAsync(xs + redo[t] * trials, gx + t * trials, sizeof(double) * trials,
                                     cudaMemcpyDeviceToDevice, st));
        SPERM_CUDA(cudaStreamSynchronize(st));  // h_ids is read by the copy above
        cudaFreeAsync(gm, st);
        cudaFreeAsync(gi, st);
        cudaFreeAsync(gx, st);
      }
    }
  }
  cudaError_t le = cudaGetLastError();
  if (le == cudaSuccess) {
    count_launch();
    kklll_mean_kernel<<<(unsigned)((count + 127) / 128), 128, 0, st>>>(xs, count, trials, d_est);
    le = cudaGetLastError();
  }
  if (!d_trials_out) cudaFreeAsync(xs, st);
  if (le != cudaSuccess) return cuda_check(le, "kklll kernels");
  return SPERM_OK;
}
