// rnw.cu — batched R-NW (Ryser / Nijenhuis-Wilf, Gray-code order)
// leaf permanents in exact multi-prime modular arithmetic, sm_100a.
//
//   per(A) = (-1)^(n-1) 2^(1-n) sum_{t=0}^{2^(n-1)-1} (-1)^t prod_i w_i(g(t))
//   w_i(S) = 2 a_{i,nw} - sum_j a_ij + 2 sum_{j in S} a_ij        (doubled NW row sums)
//   g(t)   = t ^ (t >> 1); going from t-1 to t flips Gray bit ctz(t); (-1)^{|g(t)|} = (-1)^t.
//
// Work decomposition.  A work item is (leaf, chunk): 32 lanes x 2^m
// consecutive terms; lane l owns t in [t0, t0 + 2^m), t0 = (chunk*32 + l) 2^m.  Every lane
// range is aligned to 2^m, so the Gray bit flipped at each step is the same in all 32 lanes
// (a warp-uniform shared-memory broadcast of the column).  Persistent CTAs pull work items
// from one atomic counter in the caller's leaf order (improved Step 3).
// Terms are summed exactly (int64 per lane), reduced mod p per chunk and added to the leaf's
// uint64 accumulator (exact and order-independent, so results are bit-reproducible).
//
// Two kernels evaluate the same sum; a per-leaf prep pass picks one (the "plan"):
//
//  * generic (plan 0): the row-sum vector w[NP] lives in registers; each Gray step adds the
//    flipped column densely (4 rows per 128-bit broadcast load); the n-fold product is formed
//    as NP/G exact int32 group products chained by signed Montgomery products mod each prime.
//
//  * tree (plans 1-12): rows and columns are renumbered (per(A) is invariant) so that the B
//    lowest Gray bits belong to columns with pairwise disjoint supports of <= 3 rows ("slot"
//    rows).  The 2^B terms of an aligned block share every row sum except the slot rows of
//    their low columns, and a slot row of low column c depends on bit c alone (clear or set).
//    With the sign (-1)^{|g(t)|} = (-1)^{|g_high|} (-1)^{|u|}, the block's sum factorises:
//        sum_u (-1)^{|u|} prod_i w_i = (-1)^{|g_high|} P_F prod_{c<B} (Q_c^0 - Q_c^1),
//    with Q_c^0 / Q_c^1 the products of column c's slot rows (bit clear / set) and P_F the
//    product of the other ("fixed") rows — distributivity, since each slot row belongs to one
//    low column.  A block of 2^B Gray-code terms therefore costs one row-sum update (the high
//    Gray bit flip, touching all rows), B exact slot products and ~B/2 + NFIX/GF Montgomery
//    products per prime, instead of 2^B n-fold products.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cub/device/device_radix_sort.cuh>
#include <atomic>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>
#include <type_traits>
#include <vector>

#include "common.cuh"

namespace sperm {
namespace {

#ifndef SPERM_RNW_THREADS  // threads per R-NW CTA (A-B builds: 128)
#define SPERM_RNW_THREADS 256
#endif
#ifndef SPERM_RNW_WARPS2  // resident warps per SM the register-heavy ("2-CTA") tree plans are
#define SPERM_RNW_WARPS2 16  // bounded for (16: 2 x 256 threads, <= 128 registers)
#endif
constexpr int kRnwThreads = SPERM_RNW_THREADS;  // 8 warps per CTA
constexpr int kMaxLaneBits = 14;  // terms per lane <= 2^14
constexpr int KS = 3;             // slot rows per low column (tree plans)
constexpr int kNumNFix = 7;
constexpr int kPermRows = 64;     // per-leaf permutation record: 64 row bytes + 64 column bytes
constexpr int kPermW = 128;
constexpr int kPermGend = kPermW - 1;  // byte 127 (column bytes >= 48 are unused): E mode
constexpr int kNumKeys = 104;     // plan * 8 + nfix index
static_assert(kNumKeys <= 128, "rnw_group_small_kernel scans 4 keys per lane");

__host__ __device__ constexpr int nfix_of(int i) {
  return i == 0 ? 4 : i == 1 ? 8 : i == 2 ? 12 : i == 3 ? 16 : i == 4 ? 24 : i == 5 ? 32 : 40;
}
// tree plans: (B, GF) — B low columns summed in closed form per block, GF fixed rows per exact
// group.  Plan 0 = generic kernel.  Plans in order of preference (more low columns = fewer
// blocks first); the first whose bounds hold is used.
//   plan:  1  2  3  4  5  6  7  8 |  9 10 11 12
//   B:     8  7  6  5  4  3  2  1 |  8  6  4  2
//   GF:    4  4  4  4  4  4  4  4 |  2  2  2  2
__host__ __device__ constexpr int plan_b(int p) {
  return p >= 1 && p <= 8 ? 9 - p : p == 9 ? 8 : p == 10 ? 6 : p == 11 ? 4 : p == 12 ? 2 : 0;
}
__host__ __device__ constexpr int plan_gf(int p) { return p <= 8 ? 4 : 2; }
constexpr int kNumPlans = 13;
// resident 256-thread CTAs per SM a tree kernel is compiled for: 3 (<= 85 registers, 24 warps to
// hide the fixed-latency multiply chains of short blocks) where ptxas fits it without spilling
// (-Xptxas -v over all plans and NFIX), else 2
__host__ __device__ constexpr int tree_warps(int B, int nfix, int gf) {
  return gf == 4 ? ((B <= 4 && 3 * B + nfix <= 24) || (B == 5 && nfix <= 4) || (B <= 3 && nfix <= 16) ? 24
                                                                                                   : SPERM_RNW_WARPS2)
                 : (3 * B + nfix <= 20 ? 24 : SPERM_RNW_WARPS2);
}
__host__ __device__ constexpr int tree_min_blocks(int B, int nfix, int gf) {
  return tree_warps(B, nfix, gf) / (kRnwThreads / 32);
}
constexpr int kMaxLow = 8;  // low columns picked per leaf
// Tree-kernel block loop variants (A-B builds, tools/build_variant.py): a flip of a high column
// touches few rows of a sparse leaf; kSparseW adds its column only to the touched row-sum groups,
// kSparseE recomputes only the touched low columns' E_c and fixed-row groups (warp-uniform masks).
// Measured on configs[1]: sparse W 0.164 vs 0.160 ms (predicated, no fewer issue slots), sparse E
// 0.159 (neutral); both off by default.
#ifndef SPERM_RNW_SPARSE_W
#define SPERM_RNW_SPARSE_W 0
#endif
#ifndef SPERM_RNW_SPARSE_E
#define SPERM_RNW_SPARSE_E 0
#endif
#ifndef SPERM_RNW_BLOCK_UNROLL  // measured (configs[1] kernel ms/step): 1: 0.160, 2: 0.151, 3: 0.150,
#define SPERM_RNW_BLOCK_UNROLL 4  // 4: 0.146, 8: 0.151 (more independent chains in flight per warp)
#endif
#ifndef SPERM_RNW_EMODE_NRT  // 3-CTA tree plans with at most this many register rows also get
#define SPERM_RNW_EMODE_NRT 16  // block loops specialised per E mode (B = 4, NFIX = 4: C100's leaves)
#endif
#ifndef SPERM_RNW_EFORM  // E_c = Q_c^0 - Q_c^1 evaluation: 0 products of sums, 1 / 2 multiply-add form
#define SPERM_RNW_EFORM 2  // (configs[1] kernel 0.147 / 0.147 / 0.144 ms)
#endif
// Grouped block loop: the lane's blocks are run in groups of SPERM_RNW_GROUP consecutive blocks
// (a power of two; 0 = the plain loop, unrolled kBlockUnroll times where registers allow).  Inside
// a group the flipped high column, the sign bit and (mostly) the flip direction are compile-time
// constants.  Measured (B200): configs[1] kernel 0.1336 -> 0.123 ms/step, C100 order-15 leaves 19.5
// -> 17.0 ms per 4M (with the per-leaf setup loops rolled; see there), order-16 17.0 -> 14.4 ms, C60
// order-32 leaves 76 -> 66 ms.  Groups of 8 spill in the 3-CTA variants (order-15: 17.5 ms), of 2
// save less (18.0 ms).  SPERM_RNW_GROUP_FENCE: a compiler fence between the blocks of a group keeps
// ptxas from hoisting the next blocks' loads (without it: spills, configs[1] 0.133 ms; = 2, a
// fence between pairs of blocks only: no measurable difference).
#ifndef SPERM_RNW_GROUP
#define SPERM_RNW_GROUP 4
#endif
#ifndef SPERM_RNW_GROUP_FENCE
#define SPERM_RNW_GROUP_FENCE 1
#endif
constexpr int kEForm = SPERM_RNW_EFORM;
static_assert(SPERM_RNW_EFORM == 0 || KS == 3, "multiply-add E form is written for 3 slot rows");
constexpr bool kSparseW = SPERM_RNW_SPARSE_W != 0;
constexpr bool kSparseE = SPERM_RNW_SPARSE_E != 0;
constexpr int kBlockUnroll = SPERM_RNW_BLOCK_UNROLL;

// the CRT primes (kPrimes, common.cuh) and p^-1 mod 2^32
__constant__ int32_t c_p[SPERM_KMAX] = {2147483647, 2147483629, 2147483587, 2147483579,
                                        2147483563, 2147483549, 2147483543, 2147483497};
__constant__ int32_t c_pinv[SPERM_KMAX] = {2147483647, 1469330917, -1091344149, -591336077,
                                           -2096954621, -1062895947, -1493012441, -1066630951};
// The same values as compile-time functions: in the fully unrolled per-prime loops of the R-NW
// kernels q is a constant, so p and p^-1 become instruction immediates (no constant-bank loads).
__host__ __device__ constexpr int32_t prime_p(int q) {
  return q == 0 ? 2147483647 : q == 1 ? 2147483629 : q == 2 ? 2147483587 : q == 3 ? 2147483579
       : q == 4 ? 2147483563 : q == 5 ? 2147483549 : q == 6 ? 2147483543 : 2147483497;
}
__host__ __device__ constexpr int32_t prime_pinv(int q) {
  return q == 0 ? 2147483647 : q == 1 ? 1469330917 : q == 2 ? -1091344149 : q == 3 ? -591336077
       : q == 4 ? -2096954621 : q == 5 ? -1062895947 : q == 6 ? -1493012441 : -1066630951;
}
static_assert(prime_p(7) == (int32_t)kPrimes[7] && prime_p(0) == (int32_t)kPrimes[0], "prime table");
static_assert((int32_t)((uint32_t)prime_p(3) * (uint32_t)prime_pinv(3)) == 1, "p * p^-1 = 1 mod 2^32");

// Signed Montgomery product a*b*2^-32 mod p for |a|,|b| < p < 2^31; result in (-p, p).
__device__ __forceinline__ int32_t smont(int32_t a, int32_t b, int32_t p, int32_t pinv) {
  const int64_t t = (int64_t)a * b;
  const int32_t m = (int32_t)t * pinv;
  return (int32_t)(t >> 32) - __mulhi(m, p);
}
// per-leaf metadata: x = k | err << 4 | plan << 8 | nfix_idx << 16 | G << 24, y = Montgomery
// exponent; err (prep): bit 0 a row abs sum >= 2^30, bit 1 the bound needs more than max_primes
__device__ __forceinline__ int meta_k(int2 m) { return m.x & 0xf; }
__device__ __forceinline__ int meta_err(int2 m) { return (m.x >> 4) & 0x3; }
__device__ __forceinline__ int meta_plan(int2 m) { return (m.x >> 8) & 0xff; }
__device__ __forceinline__ int meta_G(int2 m) { return (m.x >> 24) & 0xff; }

// log2(r!)/r for r = 1..SPERM_NMAX (Bregman-Minc), computed once per process on first use
__device__ double d_breg[SPERM_NMAX + 1];
__device__ __forceinline__ double breg_term(int r) { return d_breg[r]; }
__global__ void breg_init_kernel() {
  const int r = threadIdx.x;
  if (r <= SPERM_NMAX) d_breg[r] = r > 0 ? lgamma((double)r + 1.0) / ((double)r * 0.6931471805599453) : 0.0;
}

// ============================================================================ prep
// One warp per leaf.  Row / column abs sums -> number of primes k, generic group size G;
// then the tree plan: 32 lanes run the greedy disjoint-support column pick from 32
// rotations of the start column, the best (lowest lane on ties) wins; the first plan whose
// exact-arithmetic bounds hold is taken.
// row/column masks of a leaf: 32-bit words for n <= 32, 64-bit for n <= 48
__device__ __forceinline__ int mpop(uint32_t x) { return __popc(x); }
__device__ __forceinline__ int mpop(unsigned long long x) { return __popcll(x); }
__device__ __forceinline__ int mffs(uint32_t x) { return __ffs((int)x); }
__device__ __forceinline__ int mffs(unsigned long long x) { return __ffsll((long long)x); }
template <typename M>
__device__ __forceinline__ M mask_below(int n) {  // bits 0..n-1
  return n >= (int)(8 * sizeof(M)) ? ~M(0) : (M(1) << n) - 1;
}

// segment collectives of the prep kernel: a W-lane segment (W = 32 or 16) of the warp
template <int W>
__device__ __forceinline__ unsigned seg_mask() { return W == 32 ? 0xffffffffu : 0xffffu << (threadIdx.x & 16); }
template <int W>
__device__ __forceinline__ unsigned seg_ballot(bool p) {
  const unsigned b = __ballot_sync(seg_mask<W>(), p);
  return W == 32 ? b : (b >> (threadIdx.x & 16)) & 0xffffu;
}
template <int W>
__device__ __forceinline__ constexpr unsigned seg_full() { return W == 32 ? 0xffffffffu : 0xffffu; }

template <typename M, int U, int W>
__global__ void rnw_prep_kernel(const int32_t* __restrict__ mats, int n, int NPg, int64_t count,
                                const int64_t* __restrict__ coef, int min_primes, int max_primes, int lift, int allow_tree,
                                int2* __restrict__ meta, int8_t* __restrict__ perm, int* __restrict__ err,
                                unsigned long long* __restrict__ leaf_acc) {
  // one W-lane segment per leaf (W = 32, or 16 for n <= 16: two leaves per warp, no idle lanes);
  // `lane` is the lane within the segment, collectives stay inside it (seg_* helpers)
  const int lane = threadIdx.x & (W - 1);
  const unsigned SM = seg_mask<W>();  // the segment's lanes: segments branch independently
  const int wib = threadIdx.x / W;
  cudaTriggerProgrammaticLaunchCompletion();  // the grouping kernel may be scheduled already
  const int64_t seg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / W;
  if (seg - (threadIdx.x & 31) / W >= count) return;  // the whole warp is past the end
  // a segment past the end (W = 16, odd count) repeats the last leaf, writing the same values,
  // so both segments of the warp stay in every collective
  const int64_t leaf = seg < count ? seg : count - 1;
  if (lane < SPERM_KMAX) leaf_acc[leaf * SPERM_KMAX + lane] = 0;  // the R-NW accumulators
  // stage the leaf in shared memory with coalesced loads; the per-lane row/column scans
  // below then read shared memory (one segment per leaf, 256 / W segments per CTA)
  extern __shared__ int32_t prep_sm[];
  // odd row stride: the lane-per-row scans a[i*ns + j] hit distinct banks (n + 1 is even for odd n:
  // at n = 15 the 16 lanes of a segment shared two banks; C100 order-15 prep 5.36 -> see DESIGN)
  const int ns = n | 1;
  int32_t* sa = prep_sm + wib * (n * ns);
  {
    // every load of a batch is issued before its stores (U = the smallest of 4, 8, 12, 16 words
    // per lane that covers the leaf, else batches of 16), so the leaf arrives in one memory round
    // trip instead of n*n/32 dependent ones, with few predicated-off slots
    const int32_t* g = mats + leaf * (int64_t)n * n;
    const int nn = n * n;
    const uint32_t magic = (uint32_t)(0xffffffffull / (uint32_t)n) + 1u;  // e / n for e < 2^16
    for (int base = 0; base < nn; base += W * U) {
      int32_t r[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = base + u * W + lane;
        r[u] = e < nn ? g[e] : 0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = base + u * W + lane;
        const int i = (int)__umulhi((uint32_t)e, magic);
        if (e < nn) sa[i * ns + (e - i * n)] = r[u];
      }
    }
    __syncwarp(SM);
  }
  const int32_t* a = sa;
  constexpr int NSEG = 256 / W;
  __shared__ int64_t sR[NSEG][SPERM_NMAX];
  __shared__ M sSupp[NSEG][SPERM_NMAX];
  __shared__ int sCnt[NSEG][SPERM_NMAX];
  __shared__ int sBl[NSEG][SPERM_NMAX];  // bit length of each row bound: R_i < 2^bl_i
  int64_t* R = sR[wib];
  M* supp = sSupp[wib];
  int* cnt = sCnt[wib];
  // log2 of the row / column sum bounds and their Bregman-Minc forms, summed in fp32 with the
  // hardware log2 (MUFU.LG2): every term is within 4e-6 of the exact log2 and the <= 2 x 48 fp32
  // additions of a sum below 2^11 lose < 48 x 2^-13 = 6e-3 bits in total; `need` below adds 0.02
  // bits, so the bound only ever errs upwards (a leaf within 0.02 bits of a prime boundary, about
  // 1 in 1500, takes one prime more than necessary).  fp64 log2 calls and fp64 segment reductions
  // were ~11 % of this kernel's instructions.
  float lr = 0.f, lc = 0.f, br = 0.f, bc = 0.f;
  bool zero = false, range_bad = false, binary = true;
  for (int i = lane; i < n; i += W) {
    int64_t r = 0, c = 0;
    M sm = 0;
    int nz = 0;
    for (int j = 0; j < n; ++j) {
      const int32_t u = a[i * ns + j];
      r += llabs((long long)u);
      if (u != 0 && u != 1) binary = false;
      const int32_t v = a[j * ns + i];
      c += llabs((long long)v);
      if (v != 0) { sm |= M(1) << j; ++nz; }
    }
    R[i] = r;
    sBl[wib][i] = r ? 64 - __clzll(r) : 0;
    supp[i] = sm;  // support of column i (rows j with a_ji != 0)
    cnt[i] = nz;
    if (r == 0 || c == 0) zero = true;
    if (r >= (1ll << 30)) range_bad = true;
    if (r > 0) {
      lr += __log2f((float)r);
      // Bregman term log2(r!)/r; only used when the leaf is 0/1, where r = count <= n <= 48
      if (r <= SPERM_NMAX) br += (float)breg_term((int)r);
    }
    if (c > 0) {
      lc += __log2f((float)c);
      if (c <= SPERM_NMAX) bc += (float)breg_term((int)c);
    }
  }
  for (int o = W / 2; o; o >>= 1) {
    lr += __shfl_xor_sync(SM, lr, o, W);
    lc += __shfl_xor_sync(SM, lc, o, W);
    br += __shfl_xor_sync(SM, br, o, W);
    bc += __shfl_xor_sync(SM, bc, o, W);
  }
  zero = seg_ballot<W>(zero) != 0;
  range_bad = seg_ballot<W>(range_bad) != 0;
  binary = seg_ballot<W>(binary) == seg_full<W>();
  // Bregman-Minc: per(A) <= prod_i (r_i!)^(1/r_i) for a 0/1 matrix (and by columns)
  if (binary) {
    lr = fminf(lr, br);
    lc = fminf(lc, bc);
  }
  __syncwarp(SM);

  // ---- tree plan: greedy pick of up to kMaxLow low columns with disjoint supports of <= 3
  // rows, lane l starting from column l mod n; picks packed one byte each (no local memory)
  unsigned long long packed = 0;
  int np = 0;
  if (allow_tree && n >= 8 && !range_bad) {
    M used = 0;
    const int l0 = lane % n;
    const M nmask = mask_below<M>(n);
    for (int lvl = 1; lvl <= KS; ++lvl) {
      // columns with exactly lvl nonzeros, visited in the lane's rotated order l0, l0+1, ...
      M m = 0;
      for (int c0 = 0; c0 < n; c0 += W) {
        const int j = c0 + lane;
        m |= (M)seg_ballot<W>(j < n && cnt[j] == lvl) << c0;
      }
      M rot = l0 ? ((m >> l0) | (m << (n - l0))) & nmask : m;
      while (rot) {
        int j = mffs(rot) - 1 + l0;
        rot &= rot - 1;
        j -= j >= n ? n : 0;
        if (!(supp[j] & used) && np < kMaxLow && np < n - 2) {
          packed |= (unsigned long long)j << (8 * np);
          ++np;
          used |= supp[j];
        }
      }
    }
  }
  // best lane: most picks, lowest lane on ties
  int key = (np << 8) | (W - 1 - lane);
  for (int o = W / 2; o; o >>= 1) key = max(key, __shfl_xor_sync(SM, key, o, W));
  const int best = W - 1 - (key & 0xff);
  np = key >> 8;
  packed = __shfl_sync(SM, packed, best, W);
  // lane c < np: support of low column c and the product of its slot rows' bounds
  auto sat_mul = [](int64_t x, int64_t y) -> int64_t {
    // saturating product of non-negative bounds (no 64-bit division): saturate at 2^40 when the
    // operands' bit lengths could reach 2^62; every threshold tested below is < 2^31
    if (x == 0 || y == 0) return 0;
    if ((64 - __clzll(x)) + (64 - __clzll(y)) > 62) return (int64_t)1 << 40;
    const int64_t p = x * y;
    return p > ((int64_t)1 << 40) ? ((int64_t)1 << 40) : p;
  };
  M my_supp = 0;
  int64_t my_q = 1;
  if (lane < np) {
    my_supp = supp[(packed >> (8 * lane)) & 0xff];
    for (M b = my_supp; b; b &= b - 1) my_q = sat_mul(my_q, R[mffs(b) - 1]);
  }

  // ---- number of primes (lane 0).  k = the leaf's own need; a leaf whose exact value fits the
  // symmetric range of one or two primes (2 |coef| bound < p_0 [p_1]) is evaluated mod those alone
  // when `lift` is set, and the finalize lifts its exact value to the residues of min_primes primes
  int k = lift ? 1 : min_primes;
  int ebits = 0;  // meta_err; also OR-ed into *err when err != NULL (small batches: the grouping kernel)
  if (lane == 0) {
    if (range_bad) ebits |= 1;
    float lb = zero ? -1.f : fminf(lr, lc);
    const int64_t cf = coef ? coef[leaf] : 1;
    if (cf == 0) lb = -1.f;
    else if (lb >= 0.f) lb += __log2f(fabsf((float)cf));
    // need prod p_q > 2 * bound; each p_q > 2^30.99999; margin for the fp32 sums (see above)
    const float need = lb + 1.f + 0.02f + 1e-5f * fabsf(lb);
    const int kcap = max_primes > 0 ? max_primes : SPERM_KMAX;
    while (k <= SPERM_KMAX && 30.9999f * (float)k <= need) ++k;
    if (k > kcap) {
      if (max_primes <= 0) ebits |= 2;
      k = kcap;
    }
    if (k > 2) k = max(k, min_primes);  // one- and two-prime leaves are lifted
    if (ebits && err) atomicOr(err, ebits);
    k |= ebits << 4;
  }
  k = __shfl_sync(SM, k, 0, W);  // k | err << 4: meta.x's low byte
  // ---- tree plans: lane l tests plan l+1 (exact-arithmetic bounds); the first feasible wins
  const int pl = lane + 1;
  bool feasible = false;
  int fi = 0, pmexp = 0;
  int emode = 0;  // exact E groups: 0 singles, 1 pairs, 2 quads
  M slot_rows = 0;
  {
    const bool test = pl >= allow_tree && allow_tree >= 1 && pl < kNumPlans && np > 0;
    const int B = plan_b(pl), GF = plan_gf(pl);
    // every slot product |Q_c| <= q_c < 2^30 keeps E_c = Q_c^0 - Q_c^1 in int32 (|E_c| <= 2 q_c);
    // the E_c are then multiplied exactly in fixed groups — quads (c = 4j..4j+3) if every quad's
    // bound product is < 2^31, else pairs if every pair's is, else singly (the leaf's E mode) —
    // and each group costs one Montgomery product per prime
    bool qok = true, pair_ok = true, quad_ok = true;
    int64_t pp = 1, qp = 1;
#pragma unroll
    for (int c = 0; c < kMaxLow; ++c) {  // warp-uniform shuffles, per-lane plan bounds
      if (c >= np) break;                  // warp-uniform: no plan uses more than np columns
      const int64_t q = __shfl_sync(SM, my_q, c, W);
      const M sc = __shfl_sync(SM, my_supp, c, W);
      if (c < B) {
        slot_rows |= sc;
        if (q >= ((int64_t)1 << 30)) qok = false;
        const int64_t e = 2 * q;
        pp = (c & 1) ? sat_mul(pp, e) : e;
        qp = (c & 3) ? sat_mul(qp, e) : e;
        if (pp >= ((int64_t)1 << 31)) pair_ok = false;
        if (qp >= ((int64_t)1 << 31)) quad_ok = false;
      }
    }
    emode = quad_ok ? 2 : pair_ok ? 1 : 0;
    const int ngroups = emode == 2 ? (B + 3) / 4 : emode == 1 ? (B + 1) / 2 : B;
    if (test && np >= B && n - 6 >= B) {
      bool ok = qok;
      const int nf = n - mpop(slot_rows);
      while (fi < kNumNFix && nfix_of(fi) < nf) ++fi;
      if (fi == kNumNFix) ok = false;
      // every exact group of GF consecutive fixed rows: prod R_i < 2^(sum bl_i) <= 2^30
      // (bit-length sums: a conservative, division- and multiply-free test)
      const int* bl = sBl[wib];
      int pos = 0, bits = 0;
      for (int i = 0; i < n; ++i) {
        if ((slot_rows >> i) & 1) continue;
        bits += bl[i];
        if ((++pos & (GF - 1)) == 0) {
          if (bits > 30) ok = false;
          bits = 0;
        }
      }
      if (bits > 30) ok = false;
      feasible = ok;
      // Montgomery factors per block value: NGF-1 (P_F chain) + one per exact E group
      if (ok) pmexp = nfix_of(fi) / GF - 1 + ngroups;
    }
  }
  const unsigned fmask = seg_ballot<W>(feasible);
  if (fmask) {
    const int win = __ffs(fmask) - 1;  // lowest plan index = preferred
    const int wpl = win + 1, B = plan_b(wpl);
    const int wfi = __shfl_sync(SM, fi, win, W);
    const int NF = nfix_of(wfi);
    slot_rows = __shfl_sync(SM, slot_rows, win, W);
    // permutation record, written by all lanes in parallel: rows [slot rows of low column c
    // (ascending, -1 padded to KS)..., fixed rows ascending, -1 to NS + NF]; columns [low
    // columns, high columns ascending, nw]
    int8_t* pr = perm + leaf * kPermW;
    int8_t* pc = pr + kPermRows;
    const M nmask = mask_below<M>(n);
    const M fixed = ~slot_rows & nmask;
    M low = 0;
    for (int c = 0; c < B; ++c) low |= M(1) << ((packed >> (8 * c)) & 0xff);
    // nw column: the non-low column with most nonzeros (highest index on ties)
    int nwkey = -1;
    for (int j = lane; j < n; j += W)
      if (!((low >> j) & 1)) nwkey = max(nwkey, (cnt[j] << 8) | j);
    for (int o = W / 2; o; o >>= 1) nwkey = max(nwkey, __shfl_xor_sync(SM, nwkey, o, W));
    const int nw = nwkey & 0xff;
    const M high = nmask & ~low & ~(M(1) << nw);
    for (int i = lane; i < n; i += W) {
      const M below = (M(1) << i) - 1;
      if ((fixed >> i) & 1) {
        pr[B * KS + mpop(fixed & below)] = (int8_t)i;
      } else {
        for (int c = 0; c < B; ++c) {
          const M sc = supp[(packed >> (8 * c)) & 0xff];
          if ((sc >> i) & 1) pr[c * KS + mpop(sc & below)] = (int8_t)i;
        }
      }
      if ((high >> i) & 1) pc[B + mpop(high & below)] = (int8_t)i;
    }
    if (lane < B) {
      const int j = (packed >> (8 * lane)) & 0xff;
      pc[lane] = (int8_t)j;
      for (int s = mpop(supp[j]); s < KS; ++s) pr[lane * KS + s] = -1;
    }
    for (int f = n - mpop(slot_rows) + lane; f < NF; f += W) pr[B * KS + f] = -1;
    if (lane == 0) pc[n - 1] = (int8_t)nw;
    if (lane == win) {
      pr[kPermGend] = (int8_t)emode;  // this lane tested the winning plan
      meta[leaf] = make_int2(k | (wpl << 8) | (wfi << 16), pmexp);
    }
  } else if (lane == 0) {
    // generic plan: largest group size G in {8,4,2,1} with every group product of row bounds
    // < 2^30 (row bounds are < 2^30, so a product of two fits int64 before the test)
    int G = 1;
    for (int gs = 8; gs >= 2 && !range_bad; gs >>= 1) {
      bool ok = true;
      for (int s = 0; s < NPg && ok; s += gs) {
        int64_t prod = 1;
        for (int r = s; r < s + gs && ok; ++r) {
          prod *= r < n ? R[r] : 1;
          if (prod >= (1ll << 30)) ok = false;
        }
      }
      if (ok) { G = gs; break; }
    }
    meta[leaf] = make_int2(k | (G << 24), NPg / G - 1);
  }
}

// ============================================================================ generic kernel
template <int NP, int G>
__device__ __forceinline__ void term_product(const int32_t (&w)[NP], int k, int32_t (&out)[SPERM_KMAX]) {
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
      for (int g = 1; g < NG; ++g) pr = smont(pr, gp[g], prime_p(q), prime_pinv(q));
      out[q] = pr;
    }
  }
}

template <int NP>
struct GLayout {
  static constexpr int kPos = 0;                                // dpos[col][NP]
  static constexpr int kNeg = ((NP * NP + 31) / 32) * 32 + 16;  // dneg[col][NP], bank-shifted
  static constexpr int kW0 = kNeg + NP * NP;                    // w0[NP]
  static constexpr int kWords = ((kW0 + NP + 3) / 4) * 4;       // per warp, 16-byte aligned
};

// One lane's 2^m terms starting at t0 (t0 a multiple of 2^m, m >= 1).
template <int NP, int G>
__device__ __forceinline__ void lane_range(int32_t (&w)[NP], const int32_t* __restrict__ sm, int m, uint64_t t0,
                                           int k, int64_t (&acc)[SPERM_KMAX]) {
  using L = GLayout<NP>;
  int32_t d0[NP];
#pragma unroll
  for (int v = 0; v < NP / 4; ++v) {
    const int4 d = reinterpret_cast<const int4*>(sm + L::kPos)[v];
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
        const int4 d = col[v];
        w[4 * v] += d.x; w[4 * v + 1] += d.y; w[4 * v + 2] += d.z; w[4 * v + 3] += d.w;
      }
    }
    term_product<NP, G>(w, k, pe);
    // odd step t0+u+1 flips column 0: added iff bit 1 of t0+u+1 is 0
    if (!(((t0 + u + 1) >> 1) & 1ull)) {
#pragma unroll
      for (int i = 0; i < NP; ++i) w[i] += d0[i];
    } else {
#pragma unroll
      for (int i = 0; i < NP; ++i) w[i] -= d0[i];
    }
    term_product<NP, G>(w, k, po);
#pragma unroll
    for (int q = 0; q < SPERM_KMAX; ++q)
      if (q < k) acc[q] += (int64_t)pe[q] - (int64_t)po[q];
  }
}

template <int NP>
__global__ void __launch_bounds__(kRnwThreads) rnw_generic_kernel(
    const int32_t* __restrict__ mats, int n, int m, int cbits, const int32_t* __restrict__ leaves,
    const int2* __restrict__ meta, unsigned long long* __restrict__ queue, uint64_t total_items,
    unsigned long long* __restrict__ leaf_acc, unsigned long long* __restrict__ leaf_cycles,
    const int* __restrict__ go) {
  cudaGridDependencySynchronize();  // a PDL launch: the grouping kernel's writes are visible
  if (go && *go == 0) return;  // a speculative launch whose plan histogram did not match
  using L = GLayout<NP>;
  extern __shared__ int4 smem4[];
  const int lane = threadIdx.x & 31;
  int32_t* sm = reinterpret_cast<int32_t*>(smem4) + (threadIdx.x >> 5) * L::kWords;
  const uint64_t T = 1ull << (n - 1);
  int64_t cur_leaf = -1;
  int64_t prev_leaf = -1;
  long long t_item = 0;
  while (true) {
    unsigned long long item = 0;
    if (lane == 0) item = atomicAdd(queue, 1ull);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (leaf_cycles && lane == 0) {  // SM cycles of the previous work item, charged to its leaf
      const long long now = clock64();
      if (prev_leaf >= 0) atomicAdd(leaf_cycles + prev_leaf, (unsigned long long)(now - t_item));
      t_item = now;
    }
    if (item >= total_items) break;
    const int64_t leaf = leaves[(int64_t)(item >> cbits)];
    prev_leaf = leaf;
    const uint64_t chunk = item & ((1ull << cbits) - 1);
    const int2 mt = meta[leaf];
    const int k = meta_k(mt), G = meta_G(mt);
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
          case 8: term_product<NP, 8>(w, k, pr); break;
          case 4: term_product<NP, 4>(w, k, pr); break;
          case 2: term_product<NP, 2>(w, k, pr); break;
          default: term_product<NP, 1>(w, k, pr); break;
        }
        const bool neg = t0 & 1ull;
#pragma unroll
        for (int q = 0; q < SPERM_KMAX; ++q)
          if (q < k) acc[q] = neg ? -(int64_t)pr[q] : (int64_t)pr[q];
      } else {
        switch (G) {
          case 8: lane_range<NP, 8>(w, sm, m, t0, k, acc); break;
          case 4: lane_range<NP, 4>(w, sm, m, t0, k, acc); break;
          case 2: lane_range<NP, 2>(w, sm, m, t0, k, acc); break;
          default: lane_range<NP, 1>(w, sm, m, t0, k, acc); break;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < SPERM_KMAX; ++q) {
      if (q < k) {
        int64_t v = acc[q];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) {
          int64_t r = v % c_p[q];
          if (r < 0) r += c_p[q];
          atomicAdd(leaf_acc + leaf * SPERM_KMAX + q, (unsigned long long)r);
        }
      }
    }
  }
}

// ============================================================================ tree kernel
// shared memory per warp (words): colpos[nh][S4] | colneg[nh][S4] (bank-shifted) | w0[S4] |
// delta[NS] | mask[nh]
struct TreeSmem {
  int S4, nh, pos, neg, w0, delta, mask, words;
};
__host__ __device__ inline TreeSmem tree_smem(int NRT, int NS, int n, int B) {
  TreeSmem t;
  t.S4 = (NRT + 3) / 4 * 4;
  t.nh = n - 1 - B;
  t.pos = 0;
  t.neg = ((t.nh * t.S4 + 31) / 32) * 32 + 16;
  t.w0 = ((t.neg + t.nh * t.S4 + 3) / 4) * 4;
  t.delta = t.w0 + t.S4;
  t.mask = t.delta + NS;
  t.words = ((t.mask + t.nh + 3) / 4) * 4;
  return t;
}

template <int NFIX, int PLAN>
__global__ void __launch_bounds__(kRnwThreads, tree_min_blocks(plan_b(PLAN), NFIX, plan_gf(PLAN))) rnw_tree_kernel(
    const int32_t* __restrict__ mats, int n, int m, int cbits, const int32_t* __restrict__ leaves,
    const int2* __restrict__ meta, const int8_t* __restrict__ perm, unsigned long long* __restrict__ queue,
    uint64_t total_items, unsigned long long* __restrict__ leaf_acc, unsigned long long* __restrict__ leaf_cycles,
    const int* __restrict__ go) {
  cudaGridDependencySynchronize();  // a PDL launch: the grouping kernel's writes are visible
  if (go && *go == 0) return;  // a speculative launch whose plan histogram did not match
  constexpr int B = plan_b(PLAN), GF = plan_gf(PLAN);
  constexpr int NS = B * KS;       // slot rows
  constexpr int NRT = NS + NFIX;   // row sums held in registers
  constexpr int S4 = (NRT + 3) / 4 * 4;
  constexpr int NGF = NFIX / GF;   // exact fixed-row groups
  // block-loop unroll: kBlockUnroll where registers allow (2-CTA builds with <= 28 register rows,
  // B <= 7; the others spill when unrolled)
  constexpr bool kUnr = tree_warps(B, NFIX, GF) < 24 && NRT <= 28 && B <= 7;
  // GRP: blocks per group of the grouped block loop (0: the plain loop, unrolled UNR times)
  constexpr int GRP = SPERM_RNW_GROUP;
  constexpr int UNR = (kUnr && GRP == 0) ? kBlockUnroll : 1;
  extern __shared__ int4 smem4[];
  const int lane = threadIdx.x & 31;
  const TreeSmem L = tree_smem(NRT, NS, n, B);
  int32_t* sm = reinterpret_cast<int32_t*>(smem4) + (threadIdx.x >> 5) * L.words;
  int64_t cur_leaf = -1;
  int64_t prev_leaf = -1;
  long long t_item = 0;
  int emode = 0;
  while (true) {
    unsigned long long item = 0;
    if (lane == 0) item = atomicAdd(queue, 1ull);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (leaf_cycles && lane == 0) {  // SM cycles of the previous work item, charged to its leaf
      const long long now = clock64();
      if (prev_leaf >= 0) atomicAdd(leaf_cycles + prev_leaf, (unsigned long long)(now - t_item));
      t_item = now;
    }
    if (item >= total_items) break;
    const int64_t leaf = leaves[(int64_t)(item >> cbits)];
    prev_leaf = leaf;
    const uint64_t chunk = item & ((1ull << cbits) - 1);
    const int k = meta_k(meta[leaf]);
    if (leaf != cur_leaf) {
      __syncwarp();
      const int32_t* a = mats + leaf * (int64_t)n * n;
      const int8_t* pr = perm + leaf * kPermW;
      const int8_t* pc = pr + kPermRows;
      // (per-leaf setup loops are kept rolled: the hot code of a small-leaf launch — setup, one or
      // two block-loop instantiations, the reduction — has to fit the 32 KB L1.5 instruction cache)
#pragma unroll 1
      for (int e = lane; e < L.nh * S4; e += 32) {
        const int h = e / S4, r = e - (e / S4) * S4;
        const int row = r < NRT ? pr[r] : -1;
        const int32_t v = row >= 0 ? 2 * a[row * n + pc[B + h]] : 0;
        sm[L.pos + e] = v;
        sm[L.neg + e] = -v;
      }
      const int nw = pc[n - 1];
#pragma unroll 1
      for (int r = lane; r < S4; r += 32) {
        const int row = r < NRT ? pr[r] : -1;
        int32_t w0 = 1;
        if (row >= 0) {
          int32_t s = 0;
#pragma unroll 1
          for (int j = 0; j < n; ++j) s += a[row * n + j];
          w0 = 2 * a[row * n + nw] - s;
        }
        sm[L.w0 + r] = w0;
      }
#pragma unroll 1
      for (int s = lane; s < NS; s += 32) {
        const int row = pr[s];
        sm[L.delta + s] = row >= 0 ? 2 * a[row * n + pc[s / KS]] : 0;
      }
      __syncwarp();
      // what a flip of high column h touches (sparse leaves: a column has few rows): bit v < 16 =
      // row-sum group W[4v..4v+3], bit 16 + c = low column c's slot rows, bit 24 = a fixed row
      for (int h = lane; h < ((kSparseW || kSparseE) ? L.nh : 0); h += 32) {
        uint32_t mk = 0;
        for (int r = 0; r < NRT; ++r)
          if (sm[L.pos + h * S4 + r] != 0) mk |= (1u << (r >> 2)) | (r < NS ? 1u << (16 + r / KS) : 1u << 24);
        sm[L.mask + h] = (int32_t)mk;
      }
      emode = pr[kPermGend];
      __syncwarp();
      cur_leaf = leaf;
    }
    const uint64_t t0 = ((chunk << 5) + (uint64_t)lane) << m;
    // base row sums (low bits clear) of the lane's first block
    int32_t W[S4];
#pragma unroll
    for (int r = 0; r < S4; ++r) W[r] = sm[L.w0 + r];
    {
      const uint64_t g0 = t0 ^ (t0 >> 1);
#pragma unroll 1
      for (int h = max(m - 1 - B, 0); h < L.nh; ++h)
        if ((g0 >> (B + h)) & 1ull) {
          const int4* col = reinterpret_cast<const int4*>(sm + L.pos + h * S4);
#pragma unroll
          for (int v = 0; v < S4 / 4; ++v) {
            const int4 d = col[v];
            W[4 * v] += d.x; W[4 * v + 1] += d.y; W[4 * v + 2] += d.z; W[4 * v + 3] += d.w;
          }
        }
    }
    int32_t D[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) D[s] = sm[L.delta + s];
    int32_t C12[kEForm == 2 ? B : 1];  // D1 * D2 per low column (E form 2)
#pragma unroll
    for (int c = 0; c < (kEForm == 2 ? B : 0); ++c) C12[c] = D[c * KS + 1] * D[c * KS + 2];
    int64_t acc[SPERM_KMAX];
#pragma unroll
    for (int q = 0; q < SPERM_KMAX; ++q) acc[q] = 0;
    // The lane's blocks are O0 + ob, O0 = t0 >> B = (chunk * 32 + lane) << (m - B), ob < 2^(m-B):
    // O0 + ob = O0 | ob, so the Gray bits a block needs (bit 0: the sign; bit hh + 1 <= m - B:
    // the flip direction) are those of the 32-bit ob | ext, ext = bit 0 of (chunk * 32 + lane)
    // moved to position m - B — no 64-bit arithmetic in the block loop.
    const uint32_t ext = (uint32_t)(((chunk << 5) + (uint64_t)lane) & 1ull) << (m - B);
    const uint32_t nblk = 1u << (m - B);
    // the block loop, instantiated for the leaf's prime count K = 1, 2, 3 (straight-line prime
    // loops) and for K = SPERM_KMAX with a runtime bound; the E mode is tested once per block.
    // (measured: configs[1] kernel 0.235 -> 0.186 ms/step, order-15 leaves 34 -> 26 ms / 4M)
    // E_c and the fixed-row group products persist across blocks: a block recomputes only what
    // the flipped high column touches (its warp-uniform mask; the first block computes all)
    constexpr int NP2 = (B + 1) / 2, NP4 = (B + 3) / 4;
    int32_t E[B], FG[NGF];
    // instantiated per prime count K and per E mode EM (the leaf's exact E grouping: 2 quads,
    // 1 pairs, 0 singles; warp-uniform per leaf), so the loop body has no mode branches
    auto blocks = [&](auto kc, auto emc) {
      constexpr int K = decltype(kc)::value;
      constexpr int EM = decltype(emc)::value;
      // flip high Gray bit B + hh (warp-uniform column): add or subtract its doubled column
      auto flip = [&](int hh, bool add, uint32_t mk) {
        const int4* col = reinterpret_cast<const int4*>(sm + (add ? L.pos : L.neg) + hh * S4);
#pragma unroll
        for (int v = 0; v < S4 / 4; ++v) {
          if (!(kSparseW) || (mk & (1u << v))) {
            const int4 d = col[v];
            W[4 * v] += d.x; W[4 * v + 1] += d.y; W[4 * v + 2] += d.z; W[4 * v + 3] += d.w;
          }
        }
      };
      // the block's sum over its 2^B low-bit patterns: prod_c (Q_c^0 - Q_c^1); exact products
      // of pairs and quads of the E_c (used when the leaf's E mode says they fit int32;
      // wrapped otherwise and then unused); `odd` = bit 0 of the block's high Gray index
      auto eval = [&](bool odd, uint32_t mk) {
        int32_t P2[NP2], P4[NP4];
#pragma unroll
        for (int c = 0; c < B; ++c) {
          if (!(kSparseE) || (mk & (1u << (16 + c)))) {
            if constexpr (kEForm == 0) {
              int32_t x0 = W[c * KS], x1 = W[c * KS] + D[c * KS];
#pragma unroll
              for (int s = 1; s < KS; ++s) {
                x0 *= W[c * KS + s];
                x1 *= W[c * KS + s] + D[c * KS + s];
              }
              E[c] = x0 - x1;
            } else {
              // -E_c = W0 t + D0 v with t = D1 W2 + D2 (W1 + D1), v = W1 W2 + t = (W1+D1)(W2+D2):
              // multiply-adds on the FMA pipe instead of adds on the ALU pipe (exact mod 2^32;
              // the sign (-1)^B of the negated factors rides on f0)
              const int32_t w0 = W[c * KS], w1 = W[c * KS + 1], w2 = W[c * KS + 2];
              const int32_t d0 = D[c * KS], d1 = D[c * KS + 1], d2 = D[c * KS + 2];
              int32_t t;
              if constexpr (kEForm == 2) t = d2 * w1 + C12[c];
              else t = d2 * (w1 + d1);
              t = d1 * w2 + t;
              const int32_t v = w1 * w2 + t;
              E[c] = w0 * t + d0 * v;
            }
          }
        }
#pragma unroll
        for (int j = 0; j < (EM != 0 ? NP2 : 0); ++j)
          P2[j] = 2 * j + 1 < B ? (int32_t)((uint32_t)E[2 * j] * (uint32_t)E[2 * j + 1]) : E[2 * j];
#pragma unroll
        for (int j = 0; j < (EM == 2 || EM < 0 ? NP4 : 0); ++j)
          P4[j] = 2 * j + 1 < NP2 ? (int32_t)((uint32_t)P2[2 * j] * (uint32_t)P2[2 * j + 1]) : P2[2 * j];
        if (!(kSparseE) || (mk & (1u << 24))) {
#pragma unroll
          for (int g = 0; g < NGF; ++g) {
            int32_t x = W[NS + g * GF];
#pragma unroll
            for (int r = 1; r < GF; ++r) x *= W[NS + g * GF + r];
            FG[g] = x;
          }
        }
        // the sign (-1)^{|high Gray bits|} rides on the first factor (prime-independent): the
        // Montgomery chain then yields a residue of the signed block value, congruent mod p
        const int32_t f0 = (odd ^ (kEForm != 0 && (B & 1))) ? -FG[0] : FG[0];
        // per prime: P_F's chain, then the exact E groups of the leaf's mode
        auto chain = [&](auto gsz, const int32_t* grp) {
          constexpr int NGR = decltype(gsz)::value;
#pragma unroll
          for (int q = 0; q < K; ++q) {
            if (K == SPERM_KMAX && q >= k) break;
            const int32_t p = prime_p(q), pinv = prime_pinv(q);
            int32_t v = f0;
#pragma unroll
            for (int g = 1; g < NGF; ++g) v = smont(v, FG[g], p, pinv);
#pragma unroll
            for (int j = 0; j < NGR; ++j) v = smont(v, grp[j], p, pinv);
            acc[q] += (int64_t)v;
          }
        };
        if constexpr (EM == 2) chain(std::integral_constant<int, NP4>{}, P4);
        else if constexpr (EM == 1) chain(std::integral_constant<int, NP2>{}, P2);
        else if constexpr (EM == 0) chain(std::integral_constant<int, B>{}, E);
        else if (emode == 2) chain(std::integral_constant<int, NP4>{}, P4);  // EM < 0: per block
        else if (emode == 1) chain(std::integral_constant<int, NP2>{}, P2);
        else chain(std::integral_constant<int, B>{}, E);
      };
      if (GRP > 1 && nblk >= (uint32_t)GRP) {
        // groups of GRP consecutive blocks ob = o + i, i < GRP (GRP a power of two, o a multiple
        // of it): for i > 0 the flipped column hh = ctz(i) and the block's sign bit i & 1 are
        // compile-time constants (shared-memory loads with immediate offsets, no select on the
        // sign), and so is the flip direction, bit hh + 1 of ob | ext, except for i = GRP / 2
        // (and i = 0), where it is a bit of o | ext.  nblk >= GRP >= 2 puts ext at bit >= 1.
        constexpr int LG = GRP >= 8 ? 3 : GRP >= 4 ? 2 : 1;
        for (uint32_t o = 0; o < nblk; o += GRP) {
          const uint32_t go_ = o | ext;
          if (o) {
            const int hh = __ffs(o) - 1;
            flip(hh, !((go_ >> (hh + 1)) & 1u), 0xffffffffu);
          }
          eval(false, 0xffffffffu);
#pragma unroll
          for (int i = 1; i < (GRP > 1 ? GRP : 1); ++i) {
            const int hh = (i & 1) ? 0 : (i & 2) ? 1 : (i & 4) ? 2 : 3;  // ctz(i), i < 16
            const bool add = (hh + 1 < LG) ? !((i >> (hh + 1)) & 1) : !((go_ >> LG) & 1u);
            // keep the blocks in order (FENCE = 2: only between pairs of blocks)
            if (SPERM_RNW_GROUP_FENCE == 1 || (SPERM_RNW_GROUP_FENCE == 2 && !(i & 1))) asm volatile("" ::: "memory");
            flip(hh, add, 0xffffffffu);
            eval((i & 1) != 0, 0xffffffffu);
          }
        }
      } else {
#pragma unroll UNR
        for (uint32_t ob = 0; ob < nblk; ++ob) {
          uint32_t mk = 0xffffffffu;
          const uint32_t gb = ob | ext;  // the block's low Gray-relevant bits (see ext)
          if (ob) {  // only the touched row groups (sparse variants)
            const int hh = __ffs(ob) - 1;
            if (kSparseW || kSparseE) mk = (uint32_t)sm[L.mask + hh];
            flip(hh, !((gb >> (hh + 1)) & 1u), mk);
          }
          eval((gb & 1u) != 0, mk);
        }
      }
    };
    // (the mode-specialised loops triple the code; only the unrolled 2-CTA variants (<= 28 register
    // rows) get them — specialised, several 3-CTA and wide variants spilled)
    auto by_mode = [&](auto kc) {
      if constexpr (kUnr || NRT <= SPERM_RNW_EMODE_NRT) {  // unrolled 2-CTA variants, small plans
        if (emode == 2) blocks(kc, std::integral_constant<int, 2>{});  // warp-uniform per leaf
        else if (emode == 1) blocks(kc, std::integral_constant<int, 1>{});
        else blocks(kc, std::integral_constant<int, 0>{});
      } else {
        blocks(kc, std::integral_constant<int, -1>{});
      }
    };
    if constexpr (NRT <= 40) {
      switch (k) {
        case 1: by_mode(std::integral_constant<int, 1>{}); break;
        case 2: by_mode(std::integral_constant<int, 2>{}); break;
        case 3: by_mode(std::integral_constant<int, 3>{}); break;
        default: by_mode(std::integral_constant<int, SPERM_KMAX>{}); break;
      }
    } else {  // many register-resident rows: one copy of the loop per mode (no spills)
      by_mode(std::integral_constant<int, SPERM_KMAX>{});
    }
#pragma unroll
    for (int q = 0; q < SPERM_KMAX; ++q) {
      if (q < k) {
        int64_t v = acc[q];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) {
          // v mod p without a 64-bit division: |v| < 32 lanes x 2^14 blocks x 2^31 = 2^50 is exact
          // in fp64, the rounded quotient is off by at most one
          const int32_t p = prime_p(q);
          int64_t r = v - (int64_t)p * __double2ll_rn((double)v * (1.0 / (double)p));
          if (r < 0) r += p;
          if (r < 0) r += p;
          if (r >= p) r -= p;
          atomicAdd(leaf_acc + leaf * SPERM_KMAX + q, (unsigned long long)r);
        }
      }
    }
  }
}

// ============================================================================ finalize
// Largest Montgomery exponent a plan can record in meta.y (generic: NP/G - 1 <= 47; tree:
// NFIX/GF - 1 + B <= 27).
constexpr int kMaxMexp = 48;
constexpr int kFinThreads = 256;  // 32 leaves x 8 primes per block iteration

// p_0^-1 mod p_1 (Garner's step for the lifted two-prime leaves)
__host__ __device__ constexpr uint64_t modpow_c(uint64_t b, uint64_t e, uint64_t m) {
  uint64_t r = 1;
  b %= m;
  while (e) {
    if (e & 1) r = r * b % m;
    b = b * b % m;
    e >>= 1;
  }
  return r;
}
constexpr uint64_t kInvP0ModP1 = modpow_c(2147483647ull, 2147483629ull - 2, 2147483629ull);
static_assert(2147483647ull % 2147483629ull * kInvP0ModP1 % 2147483629ull == 1, "p0^-1 mod p1");

// Per-call scale factors f[q][mexp] = (-1)^(n-1) 2^(1-n) R^mexp mod p_q (R = 2^32: the kernels'
// Montgomery factors), computed on the host (fin_table) and passed by value.
struct FinTable {
  uint32_t f[SPERM_KMAX][kMaxMexp];
};

// v mod p for any 64-bit v and an odd p < 2^31: the quotient is estimated in fp64 (v and 1/p
// each rounded to 53 bits, the product truncated: within 3 * 2^-19 of v / p, so off by at most
// one) and the remainder corrected exactly in 64-bit wrap-around arithmetic (it lies in (-p, 2p))
// — instead of a 64-bit integer division per residue.
__device__ __forceinline__ uint32_t mod_u64(uint64_t v, uint32_t p, double ip) {
  const uint64_t qe = (uint64_t)__dmul_rz(__ull2double_rn(v), ip);
  int64_t r = (int64_t)(v - qe * (uint64_t)p);
  if (r < 0) r += p;
  else if (r >= (int64_t)p) r -= p;
  return (uint32_t)r;
}

// Residue q of a leaf (Step 4): coef * f[q][mexp] * S_q mod p_q for q < k (S_q = the
// leaf's accumulated sum mod p_q), and for k <= q < keff the lifted value — a leaf whose exact value
// fits the symmetric range of p_0 (k = 1) or p_0 p_1 (k = 2) is reconstructed (symmetric residue, or
// Garner's step) and reduced mod p_q.  `f` = the call's table f[SPERM_KMAX][kMaxMexp]; acc(qq) = S_qq.
template <typename AccFn>
__device__ __forceinline__ uint32_t fin_residue(int n, int q, int k, int mexp, int64_t cf, const uint32_t* f,
                                                AccFn acc) {
  auto smod = [](int64_t v, uint32_t p, double ip) -> uint32_t {  // signed v mod p in [0, p)
    const uint32_t r = mod_u64(v < 0 ? 0ull - (uint64_t)v : (uint64_t)v, p, ip);
    return (v < 0 && r) ? p - r : r;
  };
  auto res = [&](int qq, uint32_t pp, double ip) -> uint32_t {
    const uint32_t v = n == 0 ? 1u : mod_u64((uint64_t)mod_u64(acc(qq), pp, ip) * f[qq * kMaxMexp + mexp], pp, ip);
    return mod_u64((uint64_t)v * smod(cf, pp, ip), pp, ip);
  };
  const uint32_t pq = (uint32_t)c_p[q];
  const double iq = 1.0 / (double)pq;
  if (q < k) return res(q, pq, iq);
  const uint32_t p0 = (uint32_t)c_p[0], p1 = (uint32_t)c_p[1];
  const double i0 = 1.0 / (double)p0, i1 = 1.0 / (double)p1;
  const uint32_t r0 = res(0, p0, i0);
  int64_t V;
  if (k == 1) {
    V = r0 > p0 / 2 ? (int64_t)r0 - (int64_t)p0 : (int64_t)r0;
  } else {
    const uint32_t r1 = res(1, p1, i1);
    const uint32_t t = mod_u64((uint64_t)mod_u64((uint64_t)r1 + p1 - mod_u64(r0, p1, i1), p1, i1) * kInvP0ModP1, p1, i1);
    const uint64_t u = r0 + (uint64_t)p0 * t, m01 = (uint64_t)p0 * p1;  // < p0 p1 < 2^62
    V = u > m01 / 2 ? (int64_t)u - (int64_t)m01 : (int64_t)u;
  }
  return smod(V, pq, iq);
}

// Leaf residues per = f[q][mexp] S mod p_q, times the leaf coefficient; accumulated into the job
// rows and the total row.  A grid-stride kernel: 32 leaves per block iteration, each (job, q)
// run of equal jobs added with one atomic.
__global__ void __launch_bounds__(kFinThreads) rnw_finalize_kernel(
    int n, int64_t count, const int2* __restrict__ meta, const unsigned long long* __restrict__ leaf_acc,
    const int64_t* __restrict__ coef, const int32_t* __restrict__ job, uint32_t* __restrict__ leaf_res,
    int32_t* __restrict__ leaf_k, unsigned long long* __restrict__ job_acc, int64_t num_jobs, const FinTable tab,
    int min_primes) {
  __shared__ uint32_t s_f[SPERM_KMAX][kMaxMexp];
  for (int t = threadIdx.x; t < SPERM_KMAX * kMaxMexp; t += blockDim.x) s_f[t / kMaxMexp][t % kMaxMexp] = tab.f[t / kMaxMexp][t % kMaxMexp];
  __shared__ unsigned long long s_val[kFinThreads];
  __shared__ int32_t s_job[kFinThreads / SPERM_KMAX];
  __syncthreads();
  const int q = threadIdx.x % SPERM_KMAX, li = threadIdx.x / SPERM_KMAX;
  for (int64_t base = (int64_t)blockIdx.x * kFinThreads; base < count * SPERM_KMAX;
       base += (int64_t)gridDim.x * kFinThreads) {
    const int64_t idx = base + threadIdx.x;
    const int64_t leaf = idx / SPERM_KMAX;
    uint64_t val = 0;
    int32_t jb = -1;
    if (leaf < count) {
      const int2 mt = meta[leaf];
      const int k = meta_k(mt);
      const int keff = max(k, min_primes);
      if (q == 0 && leaf_k) leaf_k[leaf] = keff;
      jb = job ? job[leaf] : 0;
      if (q < keff)
        val = fin_residue(n, q, k, mt.y, coef ? coef[leaf] : 1, &s_f[0][0],
                          [&](int qq) { return (uint64_t)leaf_acc[leaf * SPERM_KMAX + qq]; });
      if (leaf_res) leaf_res[idx] = (uint32_t)val;
    }
    if (job_acc) {
      s_val[threadIdx.x] = val;
      if (q == 0) s_job[li] = jb;
      __syncthreads();
      // thread (li, q) heads a run of leaves with equal jobs: sums the run, one atomic per run
      if (jb >= 0 && (li == 0 || s_job[li - 1] != jb)) {
        unsigned long long sum = 0;
        for (int r = li; r < kFinThreads / SPERM_KMAX && s_job[r] == jb; ++r) sum += s_val[r * SPERM_KMAX + q];
        if (sum) atomicAdd(job_acc + (int64_t)jb * SPERM_KMAX + q, sum);
      }
      if (job && li == 0) {  // the total row: one atomic per prime per block iteration
        unsigned long long sum = 0;
        for (int r = 0; r < kFinThreads / SPERM_KMAX; ++r) sum += s_val[r * SPERM_KMAX + q];
        if (sum) atomicAdd(job_acc + num_jobs * SPERM_KMAX + q, sum);
      }
      __syncthreads();
    }
  }
}

__global__ void reduce_mod_kernel(const unsigned long long* __restrict__ acc, int64_t rows,
                                  uint32_t* __restrict__ out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= rows * SPERM_KMAX) return;
  out[idx] = (uint32_t)(acc[idx] % (unsigned long long)c_p[idx % SPERM_KMAX]);
}

__global__ void fold_mod_kernel(unsigned long long* __restrict__ acc, int64_t rows) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= rows * SPERM_KMAX) return;
  acc[idx] %= (unsigned long long)c_p[idx % SPERM_KMAX];
}

// evaluation-order leaf ids, their plan keys, and per key: leaves, sum of k (primes) and sum
// of k * mexp (Montgomery products per block value, summed over primes: the op model's input)
// The sort key is the plan key with a 4-bit sub-key below it (SPERM_RNW_SUBKEY): the leaf's prime
// class (k = 1, 2, 3, more) and its exact-E mode, i.e. the block-loop instantiation it runs, so
// that the warps of a persistent grid, which take leaves in sorted order, sit in the same loop
// copy at the same time (instruction-cache footprint); the caller's order holds within a sub-key.
__global__ void rnw_keys_kernel(int64_t count, const int32_t* __restrict__ order, const int2* __restrict__ meta,
                                const int8_t* __restrict__ perm, int subkey,
                                uint16_t* __restrict__ keys, int32_t* __restrict__ ids, int* __restrict__ hist,
                                int* __restrict__ hist_k, unsigned long long* __restrict__ hist_kx) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int key = 0;
  int2 mt = make_int2(0, 0);
  if (i < count) {
    const int32_t leaf = order ? order[i] : (int32_t)i;
    mt = meta[leaf];
    const int plan = meta_plan(mt);
    key = plan == 0 ? 0 : plan * 8 + ((mt.x >> 16) & 0xff);
    int sub = 0;
    if (subkey && plan != 0)
      sub = ((min(meta_k(mt), 4) - 1) << 2) | (perm[(int64_t)leaf * kPermW + kPermGend] & 3);
    keys[i] = (uint16_t)((key << 4) | sub);
    ids[i] = leaf;
  }
  // block histogram in shared memory (32-bit: <= 256 leaves x 8 x 47 per bin), warp-aggregated
  // per key (leaves mostly share a few keys), then one global atomic per nonzero bin
  __shared__ int s_h[kNumKeys], s_hk[kNumKeys], s_hx[kNumKeys];
  for (int t = threadIdx.x; t < kNumKeys; t += blockDim.x) s_h[t] = s_hk[t] = s_hx[t] = 0;
  __syncthreads();
  {
    const bool live = i < count;
    const unsigned same = __match_any_sync(0xffffffffu, live ? key : -1);
    const int kk = live ? meta_k(mt) : 0;
    const int c1 = __popc(same), ck = __reduce_add_sync(same, (unsigned)kk),
              cx = __reduce_add_sync(same, (unsigned)(kk * mt.y));
    if (live && (threadIdx.x & 31) == __ffs(same) - 1) {
      atomicAdd(&s_h[key], c1);
      atomicAdd(&s_hk[key], ck);
      atomicAdd(&s_hx[key], cx);
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < kNumKeys; t += blockDim.x)
    if (s_h[t]) {
      atomicAdd(hist + t, s_h[t]);
      atomicAdd(hist_k + t, s_hk[t]);
      atomicAdd(hist_kx + t, (unsigned long long)s_hx[t]);
    }
}

// Speculative plan-group launch: the host launches the previous call's groups (same device, order,
// count and prime bounds) before it has read this call's histogram back; this kernel sets the go
// flag they test iff the histogram (hence every group's leaf range and launch shape) is the one
// they were launched for and prep raised no error.  The host compares the same two histograms.
struct KeyHist {
  int h[kNumKeys];
};
__global__ void rnw_spec_check_kernel(const int* __restrict__ hist, const int* __restrict__ err, KeyHist pred,
                                      int* __restrict__ go) {
  __shared__ int bad;
  if (threadIdx.x == 0) bad = *err;
  __syncthreads();
  for (int t = threadIdx.x; t < kNumKeys; t += blockDim.x)
    if (hist[t] != pred.h[t]) atomicOr(&bad, 1);
  __syncthreads();
  if (threadIdx.x == 0) *go = bad == 0;
}

// Small batches (count <= kSmallGroup): the keys kernel, the radix sort and the speculation check
// in one single-CTA kernel — key histogram, exclusive scan, a stable scatter of the leaf ids into
// their groups (so each group's work queue hands its leaves out in the caller's d_order, like the
// stable radix sort of larger batches), histogram store and the go flag.  Stable scatter per
// chunk of blockDim leaves: every warp's count per key (match_any), an exclusive scan of those
// counts over the warps per key, then each leaf's slot = group cursor + warps before + lanes
// before it with the same key.
constexpr int kSmallGroup = 4096;
constexpr int kSmallGroupThreads = 1024;
__global__ void __launch_bounds__(kSmallGroupThreads) rnw_group_small_kernel(
    int count, const int32_t* __restrict__ order, const int2* __restrict__ meta, int32_t* __restrict__ sorted,
    int* __restrict__ hist, int* __restrict__ hist_k, unsigned long long* __restrict__ hist_kx,
    int* __restrict__ err, unsigned long long* __restrict__ queue, KeyHist pred, int spec, int* __restrict__ go) {
  __shared__ int s_h[kNumKeys], s_hk[kNumKeys], s_cur[kNumKeys];
  __shared__ unsigned long long s_hx[kNumKeys];
  __shared__ int s_wc[kSmallGroupThreads / 32][kNumKeys];  // per-warp key counts, then prefixes
  __shared__ int s_bad, s_err;
  cudaTriggerProgrammaticLaunchCompletion();  // the first plan group may be scheduled already
  cudaGridDependencySynchronize();             // a PDL launch: prep's meta is complete and visible
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  // small batches skip the workspace memset: this kernel writes every word the plan groups and
  // the host read (histograms, the groups' work counters, err from the leaves' meta_err, go)
  for (int t = threadIdx.x; t < kNumKeys; t += blockDim.x) {
    s_h[t] = s_hk[t] = 0;
    s_hx[t] = 0;
    queue[t] = 0;
  }
  if (threadIdx.x == 0) s_err = 0;
  __syncthreads();
  int eb = 0;
  for (int base = 0; base < count; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const bool live = i < count;
    int key = -1, kk = 0, y = 0;
    if (live) {
      const int2 mt = meta[order ? order[i] : i];
      const int plan = meta_plan(mt);
      key = plan == 0 ? 0 : plan * 8 + ((mt.x >> 16) & 0xff);
      kk = meta_k(mt);
      y = mt.y;
      eb |= meta_err(mt);
    }
    const unsigned same = __match_any_sync(0xffffffffu, key);
    const int c1 = __popc(same), ck = __reduce_add_sync(same, (unsigned)kk),
              cx = __reduce_add_sync(same, (unsigned)(kk * y));
    if (live && lane == __ffs(same) - 1) {
      atomicAdd(&s_h[key], c1);
      atomicAdd(&s_hk[key], ck);
      atomicAdd(&s_hx[key], (unsigned long long)(unsigned)cx);
    }
  }
  eb = __reduce_or_sync(0xffffffffu, eb);
  if (lane == 0 && eb) atomicOr(&s_err, eb);
  __syncthreads();
  if (threadIdx.x < 32) {  // exclusive scan of the key counts: 4 keys per lane, then a warp scan
    int c[4], tot = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = lane * 4 + u;
      c[u] = k < kNumKeys ? s_h[k] : 0;
      tot += c[u];
    }
    int inc = tot;
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += v;
    }
    int off = inc - tot;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = lane * 4 + u;
      if (k < kNumKeys) s_cur[k] = off;
      off += c[u];
    }
    if (lane == 0) {
      s_bad = s_err;
      *err = s_err;
    }
  }
  for (int base = 0; base < count; base += blockDim.x) {
    for (int t = threadIdx.x; t < nwarps * kNumKeys; t += blockDim.x) s_wc[t / kNumKeys][t % kNumKeys] = 0;
    __syncthreads();
    const int i = base + threadIdx.x;
    const bool live = i < count;
    int key = -1, leaf = 0;
    if (live) {
      leaf = order ? order[i] : i;
      const int2 mt = meta[leaf];
      const int plan = meta_plan(mt);
      key = plan == 0 ? 0 : plan * 8 + ((mt.x >> 16) & 0xff);
    }
    const unsigned same = __match_any_sync(0xffffffffu, key);
    if (live && lane == __ffs(same) - 1) s_wc[warp][key] = __popc(same);
    __syncthreads();
    for (int k = threadIdx.x; k < kNumKeys; k += blockDim.x) {  // per key: exclusive prefix over the warps
      int run = s_cur[k];
      for (int w = 0; w < nwarps; ++w) {
        const int c = s_wc[w][k];
        s_wc[w][k] = run;
        run += c;
      }
      s_cur[k] = run;
    }
    __syncthreads();
    if (live) sorted[s_wc[warp][key] + __popc(same & ((1u << lane) - 1u))] = leaf;
    __syncthreads();
  }
  for (int t = threadIdx.x; t < kNumKeys; t += blockDim.x) {
    hist[t] = s_h[t];
    hist_k[t] = s_hk[t];
    hist_kx[t] = s_hx[t];
    if (spec && s_h[t] != pred.h[t]) atomicOr(&s_bad, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) *go = spec && s_bad == 0;
}

// ============================================================================ launch helpers
struct Launch {
  const int32_t* mats;
  int n, m, cbits;
  const int32_t* leaves;
  int64_t nleaves;
  const int2* meta;
  const int8_t* perm;
  unsigned long long* queue;
  unsigned long long* leaf_acc;
  cudaStream_t st;
  unsigned long long* leaf_cycles;  // optional per-leaf SM-cycle counters
  const int* go;                    // speculative launch: run only if *go != 0 (else NULL)
  bool pdl = false;                 // programmatic dependent launch after the previous kernel on st
};

// cudaLaunchKernelEx with programmatic stream serialization: the kernel's CTAs may start while the
// previous kernel on the stream finishes; it calls cudaGridDependencySynchronize() before reading
// what that kernel wrote (a no-op when launched without the attribute).
template <typename Kern, typename... Args>
cudaError_t launch_pdl(Kern kernel, dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// Non-blocking streams and reusable events for the plan groups, one pool per device (streams
// and events belong to the device that was current when they were created).  Events are leased
// per call (EventLease) and only returned once the call has enqueued every wait on them, so an
// event is never re-recorded before a cudaStreamWaitEvent on its previous record was issued,
// however many groups a call has or how many threads call concurrently.
struct StreamPool {
  std::mutex mu;
  std::vector<cudaStream_t> streams;
  std::vector<cudaEvent_t> free_events;
  cudaStream_t stream(int g) {
    std::lock_guard<std::mutex> lk(mu);
    while ((int)streams.size() <= g % 8) {
      cudaStream_t s;
      cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
      streams.push_back(s);
    }
    return streams[g % 8];
  }
  cudaEvent_t acquire() {
    std::lock_guard<std::mutex> lk(mu);
    if (free_events.empty()) {
      cudaEvent_t e;
      cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      return e;
    }
    cudaEvent_t e = free_events.back();
    free_events.pop_back();
    return e;
  }
  void release(std::vector<cudaEvent_t>& evs) {
    std::lock_guard<std::mutex> lk(mu);
    free_events.insert(free_events.end(), evs.begin(), evs.end());
    evs.clear();
  }
};
struct EventLease {
  StreamPool& pool;
  std::vector<cudaEvent_t> evs;
  explicit EventLease(StreamPool& p) : pool(p) {}
  cudaEvent_t get() {
    evs.push_back(pool.acquire());
    return evs.back();
  }
  ~EventLease() { pool.release(evs); }
};
StreamPool& stream_pool() {
  static std::mutex m;
  static std::map<int, std::unique_ptr<StreamPool>> pools;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(m);
  std::unique_ptr<StreamPool>& p = pools[dev];
  if (!p) p.reset(new StreamPool);
  return *p;
}

// Terms per lane 2^m: small enough that a group has 1-2x per_warp work items per resident warp
// of the GPU (16 per SM; items of equal size, pulled dynamically), at least mmin (the tree block
// size), at most 2^14 and such that a leaf holds at least one 32-lane chunk.
int choose_m(int n, int64_t nleaves, int mmin) {
  const int tb = n - 1;
  static const double per_warp = [] {  // A-B knob: SPERM_RNW_ITEMS_PER_WARP (default 1: with the
    const char* e = getenv("SPERM_RNW_ITEMS_PER_WARP");  // closed-form blocks measured best of
    const double v = e ? atof(e) : 0.0;                  // 0.75/1/1.5/2/4 on configs[1], 0.169 vs
    return v > 0.0 ? v : 1.0;                            // 0.190 ms at 2; fullerene96 R-NW -8 %)
  }();
  const double target_items = (double)sm_count() * 16.0 * per_warp;
  const double per_lane = std::ldexp((double)nleaves, tb) / (32.0 * target_items);
  int m = per_lane >= 1.0 ? (int)std::floor(std::log2(per_lane)) : 0;
  m = std::min(m, kMaxLaneBits);
  m = std::min(m, std::max(0, tb - 5));
  return std::max(m, mmin);
}

template <typename K>
int launch_persistent(K kernel, size_t smem, const Launch& L, uint64_t total, bool tree) {
  // attribute + occupancy query cached per (kernel, shared-memory size, device): host time per call
  // (the dynamic shared-memory attribute only ever grows: the largest size requested so far)
  static std::mutex mu;
  static std::map<std::tuple<const void*, size_t, int>, int> cache;
  static std::map<std::pair<const void*, int>, size_t> attr_max;
  int dev = 0;
  cudaGetDevice(&dev);
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    size_t& amax = attr_max[std::make_pair((const void*)kernel, dev)];
    if (smem > amax) {
      SPERM_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      amax = smem;
    }
    const auto key = std::make_tuple((const void*)kernel, smem, dev);
    auto it = cache.find(key);
    if (it == cache.end()) {
      SPERM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kRnwThreads, smem));
      cache[key] = per_sm;
    } else {
      per_sm = it->second;
    }
  }
  if (per_sm < 1) return set_error(SPERM_ERR_ARG, "sperm_permanent: kernel does not fit on an SM");
  uint64_t grid = (uint64_t)sm_count() * per_sm;
  const uint64_t blocks_needed = (total + kRnwThreads / 32 - 1) / (kRnwThreads / 32);
  grid = std::max<uint64_t>(1, std::min(grid, blocks_needed));
  (void)tree;
  count_launch();
  SPERM_CUDA(launch_pdl(kernel, dim3((unsigned)grid), dim3(kRnwThreads), smem, L.st, L.pdl, L.mats, L.n, L.m,
                        L.cbits, L.leaves, L.meta, L.perm, L.queue, total, L.leaf_acc, L.leaf_cycles, L.go));
  SPERM_LAUNCH_CHECK("rnw kernel");
  return SPERM_OK;
}

template <int NP>
int launch_generic(const Launch& L) {
  const int tb = L.n - 1;
  const int m = choose_m(L.n, L.nleaves, tb >= 6 ? 1 : 0);
  const int cbits = std::max(0, tb - 5 - m);
  const uint64_t total = (uint64_t)L.nleaves << cbits;
  const size_t smem = (size_t)GLayout<NP>::kWords * 4 * (kRnwThreads / 32);
  auto kern = rnw_generic_kernel<NP>;
  SPERM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  SPERM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRnwThreads, smem));
  uint64_t grid = (uint64_t)sm_count() * std::max(per_sm, 1);
  const uint64_t blocks_needed = (total + kRnwThreads / 32 - 1) / (kRnwThreads / 32);
  grid = std::max<uint64_t>(1, std::min(grid, blocks_needed));
  count_launch();
  kern<<<(unsigned)grid, kRnwThreads, smem, L.st>>>(L.mats, L.n, m, cbits, L.leaves, L.meta, L.queue, total,
                                                    L.leaf_acc, L.leaf_cycles, L.go);
  SPERM_LAUNCH_CHECK("rnw_generic_kernel");
  return SPERM_OK;
}

template <int NFIX, int PLAN>
int launch_tree(const Launch& L) {
  constexpr int B = plan_b(PLAN);
  constexpr int NS = B * KS, NRT = NS + NFIX;
  const int tb = L.n - 1;
  static const int min_block_bits = [] {  // A-B knob: SPERM_RNW_MIN_BLOCK_BITS (log2 blocks per lane per item)
    const char* e = getenv("SPERM_RNW_MIN_BLOCK_BITS");
    return e ? std::max(0, std::min(8, atoi(e))) : 4;  // 2 3 4 5 6: configs[1] 0.220 0.215 0.210 0.213 0.220 ms
  }();
  const int m = choose_m(L.n, L.nleaves, std::min(B + min_block_bits, L.n - 6));
  if (m > tb - 5) return set_error(SPERM_ERR_ARG, "sperm_permanent: leaf too small for the tree plan");
  const int cbits = tb - 5 - m;
  const uint64_t total = (uint64_t)L.nleaves << cbits;
  const TreeSmem ts = tree_smem(NRT, NS, L.n, B);
  const size_t smem = (size_t)ts.words * 4 * (kRnwThreads / 32);
  Launch l2 = L;
  l2.m = m;
  l2.cbits = cbits;
  return launch_persistent(rnw_tree_kernel<NFIX, PLAN>, smem, l2, total, true);
}

template <int PLAN>
int launch_tree_nfix(int fi, const Launch& L) {
  switch (fi) {
    case 0: return launch_tree<nfix_of(0), PLAN>(L);
    case 1: return launch_tree<nfix_of(1), PLAN>(L);
    case 2: return launch_tree<nfix_of(2), PLAN>(L);
    case 3: return launch_tree<nfix_of(3), PLAN>(L);
    case 4: return launch_tree<nfix_of(4), PLAN>(L);
    case 5: return launch_tree<nfix_of(5), PLAN>(L);
    default: return launch_tree<nfix_of(6), PLAN>(L);
  }
}

}  // namespace

// Build parts.  The 84 tree-kernel variants (each with its block loops per prime count and E mode)
// dominate the compile time of this file, so the build compiles it several times in parallel with
// -DSPERM_RNW_PART=p: part 0 holds the C ABI, the host code and every other kernel, parts 1..3 only
// instantiate the tree variants of the plans they own and export one launcher each
// (rnw_tree_part<p>); without the macro (tools/build_variant.py, single object) everything is
// instantiated here.  The launch record crosses the parts as an opaque pointer: every part compiles
// the same `Launch` definition.
#ifndef SPERM_RNW_PART
#define SPERM_RNW_PART -1
#endif
constexpr int kRnwPart = SPERM_RNW_PART;
__host__ __device__ constexpr int plan_part(int plan) {  // owner of a plan's variants
  return plan == 1 || plan == 2 || plan == 9 ? 1 : plan == 3 || plan == 4 || plan == 10 ? 2
       : plan >= 5 && plan <= 8 ? 3 : 0;
}
int rnw_tree_part1(int plan, int fi, const void* launch);
int rnw_tree_part2(int plan, int fi, const void* launch);
int rnw_tree_part3(int plan, int fi, const void* launch);

namespace {

template <int PLAN>
int tree_dispatch(int fi, const Launch& L) {
  constexpr int owner = plan_part(PLAN);
  if constexpr (kRnwPart < 0 || kRnwPart == owner) return launch_tree_nfix<PLAN>(fi, L);
  else if constexpr (owner == 1) return rnw_tree_part1(PLAN, fi, &L);
  else if constexpr (owner == 2) return rnw_tree_part2(PLAN, fi, &L);
  else if constexpr (owner == 3) return rnw_tree_part3(PLAN, fi, &L);
  else return set_error(SPERM_ERR_ARG, "sperm_permanent: plan owned by build part 0");
}

int launch_tree_plan(int plan, int fi, const Launch& L) {
  switch (plan) {
    case 1: return tree_dispatch<1>(fi, L);
    case 2: return tree_dispatch<2>(fi, L);
    case 3: return tree_dispatch<3>(fi, L);
    case 4: return tree_dispatch<4>(fi, L);
    case 5: return tree_dispatch<5>(fi, L);
    case 6: return tree_dispatch<6>(fi, L);
    case 7: return tree_dispatch<7>(fi, L);
    case 8: return tree_dispatch<8>(fi, L);
    case 9: return tree_dispatch<9>(fi, L);
    case 10: return tree_dispatch<10>(fi, L);
    case 11: return tree_dispatch<11>(fi, L);
    case 12: return tree_dispatch<12>(fi, L);
    default: return set_error(SPERM_ERR_ARG, "sperm_permanent: bad plan key");
  }
}

}  // namespace

#if SPERM_RNW_PART == 1
int rnw_tree_part1(int plan, int fi, const void* launch) {
  return launch_tree_plan(plan, fi, *static_cast<const Launch*>(launch));
}
#elif SPERM_RNW_PART == 2
int rnw_tree_part2(int plan, int fi, const void* launch) {
  return launch_tree_plan(plan, fi, *static_cast<const Launch*>(launch));
}
#elif SPERM_RNW_PART == 3
int rnw_tree_part3(int plan, int fi, const void* launch) {
  return launch_tree_plan(plan, fi, *static_cast<const Launch*>(launch));
}
#endif

#if SPERM_RNW_PART <= 0  // the rest of the file: part 0 (or the single-object build) only
namespace {

int launch_key(int key, int NPg, const Launch& L) {
  if (key == 0) {
    switch (NPg) {
      case 8: return launch_generic<8>(L);
      case 16: return launch_generic<16>(L);
      case 24: return launch_generic<24>(L);
      case 32: return launch_generic<32>(L);
      case 40: return launch_generic<40>(L);
      case 48: return launch_generic<48>(L);
      default: return set_error(SPERM_ERR_ARG, "sperm_permanent: unsupported order");
    }
  }
  return launch_tree_plan(key / 8, key % 8, L);
}

// First tree plan the prep pass may choose (0 = generic kernel only).  Testing / A-B
// measurements only: SPERM_RNW_PLAN_MIN=<p> restricts the plans to p..12.
int first_plan() {
  const char* e = getenv("SPERM_RNW_PLAN_MIN");
  if (!e || !e[0]) return 1;
  const int p = atoi(e);
  return (p >= 0 && p < kNumPlans) ? p : 1;
}

// Leaves lifted in the finalize (prep's `lift`): a leaf whose exact value fits the symmetric range
// of p_0 (or p_0 p_1) is evaluated mod p_0 (and p_1) only, whatever min_primes asks (the R-NW
// block loop then runs one or two Montgomery chains instead of min_primes).  A-B knob:
// SPERM_LIFT=0 turns it off.
// Programmatic dependent launch of the grouping kernel after prep and of the first speculative plan
// group after the grouping (small batches): their CTAs are scheduled while the previous kernel
// finishes.  A-B knob: SPERM_PDL=0.
bool pdl_enabled() {
  const char* e = getenv("SPERM_PDL");
  return !(e && e[0] == '0');
}

bool lift_enabled() {
  const char* e = getenv("SPERM_LIFT");
  return !(e && e[0] == '0');
}

bool subkey_enabled() {  // A-B knob SPERM_RNW_SUBKEY=1, read per call (measured: order-15 leaves 17.04 ->
  const char* e = getenv("SPERM_RNW_SUBKEY");  // 16.95 ms per 4M, within noise of the extra sort
  return e && e[0] == '1';                     // pass; off by default; tested)
}

// f[q][y] = (-1)^(n-1) 2^(1-n) (2^32)^y mod p_q (exact uint64 arithmetic on the host)
FinTable fin_table(int n) {
  FinTable t;
  for (int q = 0; q < SPERM_KMAX; ++q) {
    const uint64_t p = kPrimes[q];
    uint64_t base = 1;  // 2^(1-n) = ((p+1)/2)^(n-1)
    for (int i = 1; i < n; ++i) base = base * ((p + 1) / 2) % p;
    if (n > 0 && ((n - 1) & 1)) base = (p - base) % p;
    const uint64_t R = ((uint64_t)1 << 32) % p;
    uint64_t f = base;
    for (int y = 0; y < kMaxMexp; ++y) {
      t.f[q][y] = (uint32_t)f;
      f = f * R % p;
    }
  }
  return t;
}

// ---------------------------------------------------------------------------- op model
// Algorithmic 32-bit integer lane-operations of one evaluation, per the kernels' own
// formulation.  IMAD.WIDE and IMAD.HI occupy the multiply (FMA) pipe twice
// as long as IMAD (tools/microbench), so they count 2 "fma units"; IADD/LOP/shift count on
// the ALU pipe.  Used for the roofline in bench.py; cross-checked against ncu pipe counters.
struct RnwStats {
  double terms = 0, fma = 0, alu = 0;
};
std::mutex g_stats_mu;
RnwStats g_stats;

void record_stats(int key, int NPg, int n, int64_t leaves, int64_t sum_k, double sum_kx) {
  // sum_kx = sum over the key's leaves of k * mexp: Montgomery products per term (generic) or
  // per block value (tree), summed over the primes
  const double T = std::ldexp(1.0, n - 1);
  double fma_terms = 0, alu_terms = 0;  // totals over the key's leaves, per term-count unit
  if (key == 0) {
    // generic, per term: NP adds, NP - NP/G products (G per leaf, modelled as 4) and per prime
    // (NP/G - 1) smont (5 units: WIDE 2, IMAD, HI 2; + one IADD on the alu) and a 2-op accumulate
    const int NG = NPg / 4;
    fma_terms = T * ((NPg - NG) * (double)leaves + 5.0 * sum_kx);
    alu_terms = T * (NPg * (double)leaves + sum_kx + 2.0 * sum_k);
  } else {
    const int plan = key / 8, fi = key % 8;
    const int B = plan_b(plan), GF = plan_gf(plan);
    const int NS = B * KS, NFIX = nfix_of(fi), S4 = (NS + NFIX + 3) / 4 * 4, NGF = NFIX / GF;
    const double blocks = std::ldexp(T, -B);  // per leaf
    // per block, prime-independent: W update (S4 adds), slot products 2 (KS - 1) muls + KS adds
    // + 1 subtract per low column, <= B - 1 group joins, NGF (GF - 1) fixed-row products, ~8 ops
    // of loop / Gray bookkeeping, the sign on the first factor (2 ops); per prime: the block's
    // smont chain (sum_kx) + a 64-bit accumulate (2 ops)
    const double f_sh = B * 2.0 * (KS - 1) + (B - 1) + NGF * (GF - 1.0);
    const double a_sh = S4 + B * (KS + 1.0) + 8;
    // ptxas issues about half of the 32-bit adds as IMAD.IADD on the multiply pipe (SASS mix of
    // the tree kernels): split them evenly
    fma_terms = blocks * ((f_sh + 0.5 * a_sh + 1.0) * (double)leaves + 5.5 * sum_kx + 1.0 * sum_k);
    alu_terms = blocks * ((0.5 * a_sh + 1.0) * (double)leaves + 0.5 * sum_kx + 1.0 * sum_k);
  }
  std::lock_guard<std::mutex> lk(g_stats_mu);
  g_stats.terms += T * leaves;
  g_stats.fma += fma_terms;
  g_stats.alu += alu_terms;
}

}  // namespace
}  // namespace sperm

using namespace sperm;

extern "C" int sperm_rnw_stats(double* h_terms, double* h_fma_units, double* h_alu_ops, int reset) {
  std::lock_guard<std::mutex> lk(g_stats_mu);
  if (h_terms) *h_terms = g_stats.terms;
  if (h_fma_units) *h_fma_units = g_stats.fma;
  if (h_alu_ops) *h_alu_ops = g_stats.alu;
  if (reset) g_stats = RnwStats();
  return SPERM_OK;
}

extern "C" double sperm_rnw_terms(int n, int64_t count) {
  if (n <= 0) return (double)count;
  return (double)count * std::ldexp(1.0, n - 1);
}

namespace sperm {
namespace {
// Garner inverses inv[j][i] = p_j^-1 mod p_i (j < i), computed on the host once, passed by value
struct CrtInv {
  uint32_t inv[SPERM_KMAX][SPERM_KMAX];
};
const CrtInv& crt_inv() {
  static const CrtInv t = [] {
    CrtInv c{};
    for (int i = 0; i < SPERM_KMAX; ++i)
      for (int j = 0; j < SPERM_KMAX; ++j) {
        const uint64_t p = kPrimes[i];
        uint64_t r = 1, b = kPrimes[j] % p, e = p - 2;
        while (e) {
          if (e & 1) r = r * b % p;
          b = b * b % p;
          e >>= 1;
        }
        c.inv[j][i] = (uint32_t)r;
      }
    return c;
  }();
  return t;
}

// one row per thread: Garner digits, Horner in 32-bit limbs, symmetric range (as sperm_crt)
__global__ void crt_kernel(const uint32_t* __restrict__ res, int64_t count, int stride, const int32_t* __restrict__ kk,
                           int k_all, uint32_t* __restrict__ out, int limbs, const CrtInv tab) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= count) return;
  const int k = kk ? kk[r] : k_all;
  uint32_t* o = out + r * (limbs + 1);
  if (k < 1 || k > SPERM_KMAX) {
    for (int t = 0; t <= limbs; ++t) o[t] = 0u;
    return;
  }
  uint64_t v[SPERM_KMAX];
#pragma unroll
  for (int i = 0; i < SPERM_KMAX; ++i) {
    if (i < k) {
      const uint64_t p = (uint32_t)prime_p(i);
      uint64_t x = res[r * stride + i] % p;
#pragma unroll
      for (int j = 0; j < SPERM_KMAX; ++j)
        if (j < i) x = (x + p - v[j] % p) % p * tab.inv[j][i] % p;
      v[i] = x;
    }
  }
  constexpr int LW = SPERM_KMAX + 2;
  uint32_t X[LW], M[LW];
#pragma unroll
  for (int t = 0; t < LW; ++t) X[t] = M[t] = 0u;
  X[0] = (uint32_t)v[k - 1];
  M[0] = 1u;
  for (int i = k - 2; i >= 0; --i) {  // X = X * p_i + v_i
    uint64_t carry = v[i];
#pragma unroll
    for (int t = 0; t < LW; ++t) {
      const uint64_t cur = (uint64_t)X[t] * (uint32_t)prime_p(i) + carry;
      X[t] = (uint32_t)cur;
      carry = cur >> 32;
    }
  }
  for (int i = 0; i < k; ++i) {
    uint64_t carry = 0;
#pragma unroll
    for (int t = 0; t < LW; ++t) {
      const uint64_t cur = (uint64_t)M[t] * (uint32_t)prime_p(i) + carry;
      M[t] = (uint32_t)cur;
      carry = cur >> 32;
    }
  }
  int cmp = 0;  // compare 2X with M, most significant limb first
  {
    uint32_t hi_carry = 0;
    uint32_t X2[LW];
#pragma unroll
    for (int t = 0; t < LW; ++t) {
      X2[t] = (X[t] << 1) | hi_carry;
      hi_carry = X[t] >> 31;
    }
#pragma unroll
    for (int t = LW - 1; t >= 0; --t)
      if (cmp == 0 && X2[t] != M[t]) cmp = X2[t] > M[t] ? 1 : -1;
  }
  int sign = 1;
  if (cmp > 0) {  // x - M < 0: magnitude M - X
    int64_t borrow = 0;
#pragma unroll
    for (int t = 0; t < LW; ++t) {
      const int64_t d = (int64_t)M[t] - X[t] - borrow;
      borrow = d < 0;
      X[t] = (uint32_t)(d + (borrow ? (int64_t)1 << 32 : 0));
    }
    sign = -1;
  }
  bool zero = true;
  for (int t = 0; t < limbs; ++t) {
    const uint32_t x = t < LW ? X[t] : 0u;
    o[t] = x;
    zero = zero && x == 0u;
  }
  o[limbs] = (uint32_t)(zero ? 0 : sign);
}
}  // namespace
}  // namespace sperm

extern "C" int sperm_crt_device(const uint32_t* d_residues, int64_t count, int stride, const int32_t* d_k, int k_all,
                                uint32_t* d_out, int limbs, void* stream) {
  if (count < 0 || stride < 1 || limbs > SPERM_KMAX + 2 || limbs < 2 ||
      (count > 0 && (!d_residues || !d_out)) || (!d_k && (k_all < 1 || k_all > SPERM_KMAX || limbs < k_all + 1)))
    return set_error(SPERM_ERR_ARG, "sperm_crt_device: bad arguments");
  if (count == 0) return SPERM_OK;
  count_launch();
  crt_kernel<<<(unsigned)((count + 127) / 128), 128, 0, (cudaStream_t)stream>>>(d_residues, count, stride, d_k, k_all,
                                                                                 d_out, limbs, crt_inv());
  SPERM_LAUNCH_CHECK("crt_kernel");
  return SPERM_OK;
}

extern "C" int sperm_reduce_mod(const uint64_t* d_acc, int64_t rows, uint32_t* d_out, void* stream) {
  if (rows < 0 || (rows > 0 && (!d_acc || !d_out))) return set_error(SPERM_ERR_ARG, "sperm_reduce_mod: bad args");
  if (rows == 0) return SPERM_OK;
  const int64_t tot = rows * SPERM_KMAX;
  count_launch();
  reduce_mod_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      (const unsigned long long*)d_acc, rows, d_out);
  SPERM_LAUNCH_CHECK("reduce_mod_kernel");
  return SPERM_OK;
}

extern "C" int sperm_fold_mod(uint64_t* d_acc, int64_t rows, void* stream) {
  if (rows < 0 || (rows > 0 && !d_acc)) return set_error(SPERM_ERR_ARG, "sperm_fold_mod: bad args");
  if (rows == 0) return SPERM_OK;
  const int64_t tot = rows * SPERM_KMAX;
  count_launch();
  fold_mod_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, (cudaStream_t)stream>>>((unsigned long long*)d_acc, rows);
  SPERM_LAUNCH_CHECK("fold_mod_kernel");
  return SPERM_OK;
}

extern "C" int sperm_permanent(const int32_t* d_mats, int n, int64_t count, const int64_t* d_coef,
                               const int32_t* d_order, const int32_t* d_job, int64_t num_jobs,
                               int min_primes, int max_primes, uint32_t* d_leaf_res, int32_t* d_leaf_k,
                               uint64_t* d_job_acc, uint64_t* d_leaf_cycles, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  keep_pool_memory();
  if (n < 0 || n > SPERM_NMAX) return set_error(SPERM_ERR_ARG, "sperm_permanent: n out of range [0, 48]");
  if (count < 0) return set_error(SPERM_ERR_ARG, "sperm_permanent: count < 0");
  if (min_primes < 1 || min_primes > SPERM_KMAX)
    return set_error(SPERM_ERR_ARG, "sperm_permanent: min_primes out of range");
  if (max_primes != 0 && (max_primes < min_primes || max_primes > SPERM_KMAX))
    return set_error(SPERM_ERR_ARG, "sperm_permanent: max_primes must be 0 or in [min_primes, 8]");
  if (count == 0) return SPERM_OK;
  {  // the Bregman table of the prep kernel, once per device
    static std::atomic<unsigned> breg_done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned bit = 1u << (dev & 31);
    if (!(breg_done.load() & bit)) {
      count_launch();
      breg_init_kernel<<<1, 64, 0, st>>>();
      SPERM_LAUNCH_CHECK("breg_init_kernel");
      breg_done.fetch_or(bit);
    }
  }
  if (n > 0 && !d_mats) return set_error(SPERM_ERR_ARG, "sperm_permanent: d_mats is NULL");
  if (d_job_acc && d_job && num_jobs <= 0) return set_error(SPERM_ERR_ARG, "sperm_permanent: num_jobs");
  const int NPg = n <= 8 ? 8 : ((n + 7) / 8) * 8;

  // workspace (stream-ordered): meta | leaf_acc | perm | keys, ids, sorted keys/ids | queue, err, hist
  int2* meta = nullptr;
  unsigned long long* leaf_acc = nullptr;
  int8_t* perm = nullptr;
  uint16_t* keys = nullptr;
  int32_t* ids = nullptr;
  int* small = nullptr;  // [2] err, [4..) hist, hist_k, then u64 queue[keys], hist_kx[keys]
  void* sort_tmp = nullptr;
  auto cleanup = [&]() {
    cudaFreeAsync(meta, st);
    cudaFreeAsync(leaf_acc, st);
    cudaFreeAsync(perm, st);
    cudaFreeAsync(keys, st);
    cudaFreeAsync(ids, st);
    cudaFreeAsync(small, st);
    if (sort_tmp) cudaFreeAsync(sort_tmp, st);
  };
#define SPERM_TRY(call)                                 \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) { cleanup(); return cuda_check(e_, #call); } \
  } while (0)
  SPERM_TRY(cudaMallocAsync((void**)&meta, sizeof(int2) * count, st));
  SPERM_TRY(cudaMallocAsync((void**)&leaf_acc, sizeof(unsigned long long) * count * SPERM_KMAX, st));
  SPERM_TRY(cudaMallocAsync((void**)&perm, (size_t)kPermW * count, st));
  SPERM_TRY(cudaMallocAsync((void**)&keys, 2 * sizeof(uint16_t) * (size_t)count, st));
  SPERM_TRY(cudaMallocAsync((void**)&ids, sizeof(int32_t) * 2 * count, st));
  const size_t small_bytes = sizeof(int) * (4 + 2 * kNumKeys) + sizeof(unsigned long long) * 2 * kNumKeys;
  SPERM_TRY(cudaMallocAsync((void**)&small, small_bytes, st));
  const bool small_group = count <= kSmallGroup;
  if (!small_group) SPERM_TRY(cudaMemsetAsync(small, 0, small_bytes, st));  // (small: the grouping kernel)
  // per-group work counters after the histograms (8-byte aligned: 4 + 2*48 ints = 400 bytes)
  unsigned long long* queue = reinterpret_cast<unsigned long long*>(small + 4 + 2 * kNumKeys);
  unsigned long long* hist_kx = queue + kNumKeys;
  int* err = small + 2;
  int* hist = small + 4;
  // the previous call's groups, launched before the read-back completes when this call has the same
  // shape (repeated batches): the host's synchronization then overlaps the R-NW kernels
  struct Spec {
    int dev = -1, n = -1, NPg = 0, minp = 0, maxp = 0, plan0 = -1;
    int64_t count = -1;
    KeyHist hist;
    std::vector<int> order;
  };
  thread_local Spec spec;
  const bool spec_on = [] {  // A-B knob: SPERM_SPECULATE=0 disables (read per call: the bench
    const char* e = getenv("SPERM_SPECULATE");  // times both settings in one process; configs[1]
    return !(e && e[0] == '0');  // 0.170 vs 0.212 ms/step with NVML clock sampling running)
  }();
  int dev = 0;
  SPERM_TRY(cudaGetDevice(&dev));
  const bool speculate = spec_on && n > 0 && spec.dev == dev && spec.n == n && spec.count == count &&
                         spec.NPg == NPg && spec.minp == min_primes && spec.maxp == max_primes &&
                         spec.plan0 == first_plan();
  int* go = small;  // small[0]: zeroed above / written by the grouping kernel
  {
    TimingScope ts("rnw_prep", st);
    // one 16-lane segment per leaf for n <= 16 (two leaves per warp), else one warp
    static const int prep16 = [] {  // A-B knob: SPERM_PREP16=0 keeps one warp per leaf
      const char* e = getenv("SPERM_PREP16");
      return e ? atoi(e) : 1;
    }();
    const int W = (n <= 16 && prep16) ? 16 : 32;
    const int64_t threads = count * W;
    count_launch();
    // CTA width: 256 threads, narrowed (down to one warp) while the grid would cover fewer than two
    // CTAs per SM — a small batch (configs[1]: 256 leaves = 32 CTAs of 256) otherwise runs on a
    // fifth of the SMs, its warps sharing their SMs' issue slots (ncu: 10 of 11.7 us)
    int prep_threads = 256;
    while (prep_threads > 32 && (threads + prep_threads - 1) / prep_threads < 2 * (int64_t)sm_count()) prep_threads >>= 1;
    const size_t prep_smem = (size_t)(prep_threads / W) * n * (n | 1) * sizeof(int32_t);  // odd row stride per segment
    const int per_lane = (n * n + W - 1) / W;
    auto prep = n > 32 ? rnw_prep_kernel<unsigned long long, 16, 32>
              : W == 16 ? (per_lane <= 8 ? rnw_prep_kernel<uint32_t, 8, 16> : rnw_prep_kernel<uint32_t, 16, 16>)
              : per_lane <= 4 ? rnw_prep_kernel<uint32_t, 4, 32> : per_lane <= 8 ? rnw_prep_kernel<uint32_t, 8, 32>
              : per_lane <= 12 ? rnw_prep_kernel<uint32_t, 12, 32> : rnw_prep_kernel<uint32_t, 16, 32>;
    {  // the attribute once per device, for the largest order (host time per call)
      static std::atomic<unsigned> prep_attr{0};
      int dev = 0;
      cudaGetDevice(&dev);
      const unsigned bit = 1u << (dev & 31);
      if (!(prep_attr.load() & bit)) {
        const int max_smem = 8 * SPERM_NMAX * (SPERM_NMAX + 1) * (int)sizeof(int32_t);
        for (auto kf : {rnw_prep_kernel<uint32_t, 4, 32>, rnw_prep_kernel<uint32_t, 8, 32>,
                        rnw_prep_kernel<uint32_t, 12, 32>, rnw_prep_kernel<uint32_t, 16, 32>,
                        rnw_prep_kernel<uint32_t, 8, 16>, rnw_prep_kernel<uint32_t, 16, 16>})
          SPERM_TRY(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem));
        SPERM_TRY(cudaFuncSetAttribute(rnw_prep_kernel<unsigned long long, 16, 32>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem));
        prep_attr.fetch_or(bit);
      }
    }
    prep<<<(unsigned)((threads + prep_threads - 1) / prep_threads), prep_threads, prep_smem, st>>>(d_mats, n, NPg, count, d_coef, min_primes, max_primes,
                                                                       lift_enabled() ? 1 : 0, first_plan(), meta,
                                                                       perm, small_group ? nullptr : err, leaf_acc);
    SPERM_TRY(cudaGetLastError());
    count_launch();
    if (small_group)
      SPERM_TRY(launch_pdl(rnw_group_small_kernel, dim3(1),
                           dim3((unsigned)std::min<int64_t>(kSmallGroupThreads, (count + 31) / 32 * 32)), 0, st,
                           pdl_enabled(), (int)count, d_order, (const int2*)meta, (int32_t*)(ids + count), hist,
                           hist + kNumKeys, hist_kx, err, queue, spec.hist, speculate ? 1 : 0, go));
    else
      rnw_keys_kernel<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(count, d_order, meta, perm, subkey_enabled() ? 1 : 0,
                                                                       keys, ids, hist, hist + kNumKeys, hist_kx);
    SPERM_TRY(cudaGetLastError());
  }
  // leaves grouped by plan key (and loop-instantiation sub-key), evaluation order kept inside each
  // group (stable radix sort on the 11-bit keys), queued before the histogram read-back so that the host's only work after
  // the synchronization is launching the plan groups
  const int32_t* sorted = ids + count;
  if (!small_group) {
    size_t tmp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys + count, ids, ids + count, (int)count, 0, 11, st);
    SPERM_TRY(cudaMallocAsync(&sort_tmp, tmp_bytes, st));
    SPERM_TRY(cub::DeviceRadixSort::SortPairs(sort_tmp, tmp_bytes, keys, keys + count, ids, ids + count,
                                              (int)count, 0, 11, st));
  }
  // one read-back of the whole small block (err, histograms, queues, kx) into a per-thread
  // pinned buffer (a pageable copy is staged and slower), marked by a per-thread event
  thread_local void* h_small_pinned = nullptr;
  thread_local std::map<int, cudaEvent_t> rb_events;
  if (!h_small_pinned) SPERM_TRY(cudaMallocHost(&h_small_pinned, small_bytes));
  cudaEvent_t& rb = rb_events[dev];
  if (!rb) SPERM_TRY(cudaEventCreateWithFlags(&rb, cudaEventDisableTiming));
  // One persistent launch per plan group, each on its own stream of a small pool forked from `st`
  // (a later group's CTAs fill the SMs freed by an earlier group's tail), joined back into `st`.
  // Each group has its own work counter; groups are launched largest work first.
  int rc = SPERM_OK;
  // The largest group runs on `st` itself, the others on pool streams 1..7 (stream 0 carries the
  // speculative path's read-back); joins: their completion events, waited on by `st` afterwards.
  std::vector<cudaEvent_t> joins;
  StreamPool& pool = stream_pool();
  EventLease lease(pool);  // returned at exit, after every wait on them has been enqueued
  auto launch_groups = [&](const int* hh, const std::vector<int>& order_keys, const int* go) -> int {
    cudaEvent_t fork = nullptr;
    if (order_keys.size() > 1) {
      fork = lease.get();
      SPERM_CUDA(cudaEventRecord(fork, st));
    }
    int64_t offs[kNumKeys];
    int64_t off = 0;
    for (int key = 0; key < kNumKeys; ++key) {
      offs[key] = off;
      off += hh[key];
    }
    int g = 0;
    for (int key : order_keys) {
      cudaStream_t gs = g == 0 ? st : pool.stream(1 + (g - 1) % 7);
      if (gs != st) SPERM_CUDA(cudaStreamWaitEvent(gs, fork, 0));
      Launch L{d_mats, n, 0, 0, sorted + offs[key], hh[key], meta, perm, queue + key, leaf_acc, gs,
               (unsigned long long*)d_leaf_cycles, go};
      L.pdl = gs == st && go != nullptr && small_group && pdl_enabled();  // right after the grouping kernel
      const int r = launch_key(key, NPg, L);
      if (gs != st) {
        cudaEvent_t join = lease.get();
        SPERM_CUDA(cudaEventRecord(join, gs));
        joins.push_back(join);
      }
      if (r != SPERM_OK) return r;
      ++g;
    }
    return SPERM_OK;
  };
  std::unique_ptr<TimingScope> ts_rnw;
  if (speculate) {
    if (!small_group) {
      count_launch();
      rnw_spec_check_kernel<<<1, 128, 0, st>>>(hist, err, spec.hist, go);
      SPERM_TRY(cudaGetLastError());
    }
    ts_rnw.reset(new TimingScope("rnw", st));
    // the read-back on pool stream 0, forked before the groups (`st` waits for it with the joins)
    cudaEvent_t cf = lease.get();
    cudaStream_t cs = pool.stream(0);
    SPERM_TRY(cudaEventRecord(cf, st));
    SPERM_TRY(cudaStreamWaitEvent(cs, cf, 0));
    SPERM_TRY(cudaMemcpyAsync(h_small_pinned, small, small_bytes, cudaMemcpyDeviceToHost, cs));
    SPERM_TRY(cudaEventRecord(rb, cs));
    joins.push_back(rb);
    rc = launch_groups(spec.hist.h, spec.order, go);
  }
  auto join_groups = [&]() -> int {
    for (cudaEvent_t j : joins) SPERM_CUDA(cudaStreamWaitEvent(st, j, 0));
    joins.clear();
    return SPERM_OK;
  };
  if (!speculate) {  // the read-back on `st` after the grouping
    SPERM_TRY(cudaMemcpyAsync(h_small_pinned, small, small_bytes, cudaMemcpyDeviceToHost, st));
    SPERM_TRY(cudaEventRecord(rb, st));
  }
  {
    const int rj = join_groups();
    if (rc == SPERM_OK) rc = rj;
  }
  if (rc != SPERM_OK) { ts_rnw.reset(); cleanup(); return rc; }
  SPERM_TRY(cudaEventSynchronize(rb));
  int hsmall[4 + 2 * kNumKeys];
  unsigned long long h_kx[kNumKeys];
  memcpy(hsmall, h_small_pinned, sizeof(hsmall));
  memcpy(h_kx, static_cast<const char*>(h_small_pinned) + sizeof(int) * (4 + 2 * kNumKeys) +
                   sizeof(unsigned long long) * kNumKeys,
         sizeof(h_kx));
  if (hsmall[2] & 1) { ts_rnw.reset(); cleanup(); return set_error(SPERM_ERR_RANGE, "sperm_permanent: a row abs sum is >= 2^30"); }
  if (hsmall[2] & 2) { ts_rnw.reset(); cleanup(); return set_error(SPERM_ERR_PRIMES, "sperm_permanent: bound needs > 8 primes"); }
  const int* h_hist = hsmall + 4;
  static const bool debug = getenv("SPERM_DEBUG") != nullptr;
  if (debug) {  // plan histogram of this call (diagnostics)
    fprintf(stderr, "[sperm] permanent n=%d count=%lld:", n, (long long)count);
    for (int key = 0; key < kNumKeys; ++key)
      if (h_hist[key])
        fprintf(stderr, " key%d(plan%d,nfix%d)=%d sum_k=%d", key, key / 8, key ? nfix_of(key % 8) : 0, h_hist[key],
                hsmall[4 + kNumKeys + key]);
    fprintf(stderr, "%s\n", speculate ? " (speculative launch)" : "");
  }
  if (n > 0) {
    for (int key = 0; key < kNumKeys; ++key)
      if (h_hist[key]) record_stats(key, NPg, n, h_hist[key], hsmall[4 + kNumKeys + key], (double)h_kx[key]);
  }
  if (n > 0) {
    std::vector<int> order_keys;
    for (int key = 0; key < kNumKeys; ++key)
      if (h_hist[key]) order_keys.push_back(key);
    const int* h_sumk = hsmall + 4 + kNumKeys;
    std::stable_sort(order_keys.begin(), order_keys.end(), [&](int a, int b) { return h_sumk[a] > h_sumk[b]; });
    const bool matched = speculate && memcmp(spec.hist.h, h_hist, sizeof(spec.hist.h)) == 0;
    spec.dev = dev;
    spec.n = n;
    spec.count = count;
    spec.NPg = NPg;
    spec.minp = min_primes;
    spec.maxp = max_primes;
    spec.plan0 = first_plan();
    memcpy(spec.hist.h, h_hist, sizeof(spec.hist.h));
    spec.order = order_keys;
    if (!matched) {  // the speculative kernels (if any) found go == 0 and exited
      if (!ts_rnw) ts_rnw.reset(new TimingScope("rnw", st));
      rc = launch_groups(h_hist, order_keys, nullptr);
      const int rj = join_groups();
      if (rc == SPERM_OK) rc = rj;
    }
  }
  ts_rnw.reset();
  if (rc != SPERM_OK) { cleanup(); return rc; }
  {
    TimingScope ts("rnw_finalize", st);
    const int64_t tot = count * SPERM_KMAX;
    count_launch();
    const int64_t fblocks = std::min<int64_t>((tot + kFinThreads - 1) / kFinThreads, (int64_t)sm_count() * 8);
    rnw_finalize_kernel<<<(unsigned)fblocks, kFinThreads, 0, st>>>(
        n, count, meta, leaf_acc, d_coef, d_job, d_leaf_res, d_leaf_k, (unsigned long long*)d_job_acc, num_jobs,
        fin_table(n), min_primes);
  }
  cudaError_t le = cudaGetLastError();
  cleanup();
#undef SPERM_TRY
  if (le != cudaSuccess) return cuda_check(le, "rnw_finalize_kernel");
  return SPERM_OK;
}

// Host-buffer entry point: H2D of the matrices, sperm_permanent, device CRT, D2H of the exact
// values — the whole batched R-NW as one synchronous call on host memory.
extern "C" int sperm_permanent_host(const int32_t* h_mats, int n, int64_t count, int min_primes, uint32_t* h_out,
                                    int limbs, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 0 || n > SPERM_NMAX || count < 0 || limbs < min_primes + 1 || limbs > SPERM_KMAX + 2 ||
      (count > 0 && ((n > 0 && !h_mats) || !h_out)))
    return set_error(SPERM_ERR_ARG, "sperm_permanent_host: bad arguments");
  if (count == 0) return SPERM_OK;
  const size_t mat_bytes = sizeof(int32_t) * (size_t)n * n * count;
  int32_t* d_mats = nullptr;
  uint32_t* d_res = nullptr;
  int32_t* d_k = nullptr;
  uint32_t* d_out = nullptr;
  auto release = [&]() {
    cudaFreeAsync(d_mats, st);
    cudaFreeAsync(d_res, st);
    cudaFreeAsync(d_k, st);
    cudaFreeAsync(d_out, st);
  };
  int rc = SPERM_OK;
  cudaError_t e = cudaMallocAsync((void**)&d_mats, mat_bytes > 0 ? mat_bytes : 4, st);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&d_res, sizeof(uint32_t) * SPERM_KMAX * count, st);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&d_k, sizeof(int32_t) * count, st);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&d_out, sizeof(uint32_t) * (limbs + 1) * count, st);
  if (e == cudaSuccess && mat_bytes) e = cudaMemcpyAsync(d_mats, h_mats, mat_bytes, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) {
    release();
    return cuda_check(e, "sperm_permanent_host: allocation / H2D");
  }
  rc = sperm_permanent(d_mats, n, count, nullptr, nullptr, nullptr, 0, min_primes, 0, d_res, d_k, nullptr, nullptr,
                       stream);
  if (rc == SPERM_OK) rc = sperm_crt_device(d_res, count, SPERM_KMAX, d_k, 0, d_out, limbs, stream);
  if (rc == SPERM_OK) {
    e = cudaMemcpyAsync(h_out, d_out, sizeof(uint32_t) * (limbs + 1) * count, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) rc = cuda_check(e, "sperm_permanent_host: D2H");
  }
  release();
  e = cudaStreamSynchronize(st);
  if (rc == SPERM_OK && e != cudaSuccess) rc = cuda_check(e, "sperm_permanent_host: synchronize");
  return rc;
}

#else  // parts 1..3 end here
}  // namespace sperm
#endif  // SPERM_RNW_PART <= 0
