// subtree.cu — Algorithm H_per's recursion (Step 1's pivot line, Eq. (2)'s
// split) below the job level, DEPTH FIRST and entirely on chip.
//
// Below the job level a job's value is the sum over its leaves, so the order in which its leaves
// appear does not matter (the job list itself, PH Step 2, keeps the ordered level kernel of
// expand.cu).  The level-by-level expansion writes every intermediate node to HBM and reads it
// back one level later; here one warp takes a root node (order n0 <= 32) and walks its whole
// subtree down to the leaves of order L in shared memory:
//
//   * the current node lives in a shared-memory buffer (row stride n0 | 1: lane-per-row and
//     lane-per-column reads are both bank-conflict free); lane i keeps the nonzero counts of row
//     i and column i in registers, and a child's counts are derived from the parent's in O(n)
//     (the lines a split touches), so no node is ever rescanned;
//   * the pivot (reading R2: fewest nonzeros, rows before columns, lowest index) is two warp
//     min-reductions over the lanes' packed (count, index) keys; the pivot line's nonzeros come
//     from one ballot;
//   * a split with two surviving children (s = 3, 4) pushes the second child to the warp's stack
//     — one slot per order, since the pending siblings of a depth-first walk have distinct
//     orders — and continues with the first; s = 1, 2 continue in place (double buffer);
//   * a node of order <= L is a leaf: written densely to HBM (one atomic slot per leaf); a node
//     with s >= 5 (reading R5: not split) is written to the early outputs padded to order n0 by
//     an identity block (per(diag(X, I)) = per(X)), so every early node has the same order.
//
// The same children as expand.cu's kernel (same Eq. (2) scalars, the same zero-line test of
// reading R4, the same overflow checks): the leaves form the same multiset as the level-by-level
// recursion's, in an unspecified order.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "common.cuh"

namespace sperm {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kSubWarps = 4;  // warps per CTA (shared-memory bound: one stack per warp)

// words of the stack slots of orders L .. m-1 (slot(m) = coef (2 words) | m packed line counts |
// m x m entries, stride m): sum_{k=L}^{m-1} (k(k+1) + 2), every slot an even number of words
__host__ __device__ __forceinline__ int slot_prefix(int L, int m) {
  auto F = [](int x) { return x * (x + 1) * (x + 2) / 3; };  // sum_{k=1}^{x} k(k+1)
  return (F(m - 1) - F(L - 1)) + 2 * (m - L);
}
__host__ __device__ __forceinline__ int sub_warp_words(int n0, int L) {
  const int S = n0 | 1;
  return ((2 * n0 * S + slot_prefix(L, n0)) + 3) / 4 * 4;
}

// dst[ii * dstride + jj] = child entry (ii, jj) of the node in src (stride S), for a child that
// deletes row dr and column dc and merges (merge 1: column keep := al*col(dc) + be*col(keep);
// merge 2: row keep := al*row(dr) + be*row(keep); 0: none).  m = child order.  Merged entries
// are computed mod 2^32 (exact: the split already rejected overflowing ones).
__device__ __forceinline__ void build_child(const int32_t* __restrict__ src, int S, int m, int dr, int dc, int merge,
                                            int keep, int32_t al, int32_t be, int32_t* __restrict__ dst,
                                            int dstride, int lane) {
  const int mm = m * m;
  const uint32_t magic = (uint32_t)(0xffffffffull / (uint32_t)m) + 1u;  // e / m exactly for e < 2^16
  constexpr int UB = 4;
  for (int base = 0; base < mm; base += 32 * UB) {
    int32_t r[UB];
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const int e = base + u * 32 + lane;
      int32_t v = 0;
      if (e < mm) {
        const int ii = (int)__umulhi((uint32_t)e, magic), jj = e - ii * m;
        const int i = ii + (ii >= dr), j = jj + (jj >= dc);
        v = src[i * S + j];
        if (merge == 1 && j == keep)
          v = (int32_t)((uint32_t)al * (uint32_t)src[i * S + dc] + (uint32_t)be * (uint32_t)v);
        else if (merge == 2 && i == keep)
          v = (int32_t)((uint32_t)al * (uint32_t)src[dr * S + j] + (uint32_t)be * (uint32_t)v);
      }
      r[u] = v;
    }
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const int e = base + u * 32 + lane;
      if (e < mm) {
        const int ii = (int)__umulhi((uint32_t)e, magic);
        dst[ii * dstride + (e - ii * m)] = r[u];
      }
    }
  }
}

// A candidate child in the pivot's frame (the frame is A for a row pivot, A^T for a column
// pivot: frame row r = the pivot line).  Minor: delete frame row r and frame column p, coef *= v.
// Merge: delete frame row r and frame column kb, frame column ka := al*col(kb) + be*col(ka).
struct FKid {
  int minor;  // 1 minor, 0 merge
  int ka, kb;  // merge columns (minor: kb = p)
  int32_t al, be;
};

// GSTACK: the stack slots live in a per-warp global scratch area (L2-resident) instead of shared
// memory, so shared memory holds only the two working buffers and more warps fit per SM.
// NOATOMIC (timing experiment only, wrong output): leaves go to a per-warp slot, no atomic.
template <bool GSTACK, bool NOATOMIC>
__global__ void __launch_bounds__(32 * kSubWarps) subtree_kernel(
    const int32_t* __restrict__ mats, const int64_t* __restrict__ coef, const int32_t* __restrict__ job, int n0,
    int64_t count, int L, int warp_words, int32_t* __restrict__ out_mats, int64_t* __restrict__ out_coef,
    int32_t* __restrict__ out_job, int64_t cap_out, int32_t* __restrict__ early_mats,
    int64_t* __restrict__ early_coef, int32_t* __restrict__ early_job, int64_t cap_early,
    unsigned long long* __restrict__ ws, int* __restrict__ err, int32_t* __restrict__ gstack, int stack_words) {
  extern __shared__ int32_t ssm[];
  const int lane = threadIdx.x & 31;
  int32_t* base = ssm + (threadIdx.x >> 5) * warp_words;
  const int S = n0 | 1;
  int32_t* const Wb0 = base;
  int32_t* const Wb1 = base + n0 * S;
  int32_t* const stk = GSTACK ? gstack + ((int64_t)blockIdx.x * kSubWarps + (threadIdx.x >> 5)) * stack_words
                              : base + 2 * n0 * S;
  const int64_t L2 = (int64_t)L * L;
  const uint32_t magic0 = (uint32_t)(0xffffffffull / (uint32_t)n0) + 1u;
  while (true) {
    unsigned long long root = 0;
    if (lane == 0) root = (*(volatile int*)err & 2) ? ~0ull : atomicAdd(ws, 1ull);  // stop on a full output
    root = __shfl_sync(kFull, root, 0);
    if (root >= (unsigned long long)count) break;
    // ---- the root: staged (all of a batch's loads before its stores) and its line counts
    int cur = 0;
    int32_t* W = Wb0;
    {
      const int32_t* g = mats + (int64_t)root * n0 * n0;
      const int nn = n0 * n0;
      constexpr int UR = 8;
      for (int b = 0; b < nn; b += 32 * UR) {
        int32_t r[UR];
#pragma unroll
        for (int u = 0; u < UR; ++u) {
          const int e = b + u * 32 + lane;
          r[u] = e < nn ? g[e] : 0;
        }
#pragma unroll
        for (int u = 0; u < UR; ++u) {
          const int e = b + u * 32 + lane;
          const int i = (int)__umulhi((uint32_t)e, magic0);
          if (e < nn) W[i * S + (e - i * n0)] = r[u];
        }
      }
    }
    __syncwarp();
    int n = n0;
    int64_t cf = coef ? coef[root] : 1;
    const int32_t jb = job ? job[root] : (int32_t)root;
    int rc = 0, cc = 0;  // lane i: nonzeros of row i and of column i of the current node
    if (lane < n)
      for (int j = 0; j < n; ++j) {
        rc += W[lane * S + j] != 0;
        cc += W[j * S + lane] != 0;
      }
    uint32_t pending = 0;  // bit m: a node of order m waits in stack slot m
    while (true) {
      bool pop = false;
      if (n <= L) {
        // ---- leaf (order L): one output slot, dense row-major copy
        unsigned long long slot = 0;
        if (NOATOMIC) {
          slot = ((int64_t)blockIdx.x * kSubWarps + (threadIdx.x >> 5)) % (cap_out > 0 ? cap_out : 1);
          if (lane == 0) atomicAdd(ws + 1, 0ull);
        } else {
          if (lane == 0) slot = atomicAdd(ws + 1, 1ull);
          slot = __shfl_sync(kFull, slot, 0);
        }
        if ((int64_t)slot < cap_out) {
          int32_t* o = out_mats + (int64_t)slot * L2;
          const uint32_t mg = (uint32_t)(0xffffffffull / (uint32_t)n) + 1u;
          for (int e = lane; e < n * n; e += 32) {
            const int i = (int)__umulhi((uint32_t)e, mg);
            o[e] = W[i * S + (e - i * n)];
          }
          if (lane == 0) {
            out_coef[slot] = cf;
            out_job[slot] = jb;
          }
        } else if (lane == 0) {
          atomicOr(err, 2);
        }
        pop = true;
      } else {
        // ---- pivot line (reading R2): fewest nonzeros; rows first, a column only if strictly
        // fewer; lowest index on ties
        const int rkey = __reduce_min_sync(kFull, lane < n ? (rc << 8) | lane : 0x7fffffff);
        const int ckey = __reduce_min_sync(kFull, lane < n ? (cc << 8) | lane : 0x7fffffff);
        const bool colpiv = (ckey >> 8) < (rkey >> 8);
        const int s = colpiv ? ckey >> 8 : rkey >> 8;
        const int r = colpiv ? ckey & 0xff : rkey & 0xff;
        if (s == 0) {
          pop = true;  // a zero line: per = 0 (only a root can have one)
        } else if (s >= 5) {
          // ---- early node (reading R5: not split), padded to order n0 with an identity block
          unsigned long long slot = 0;
          if (lane == 0) slot = atomicAdd(ws + 2, 1ull);
          slot = __shfl_sync(kFull, slot, 0);
          if ((int64_t)slot < cap_early) {
            int32_t* o = early_mats + (int64_t)slot * n0 * n0;
            for (int e = lane; e < n0 * n0; e += 32) {
              const int i = (int)__umulhi((uint32_t)e, magic0), j = e - i * n0;
              o[e] = (i < n && j < n) ? W[i * S + j] : (i == j ? 1 : 0);
            }
            if (lane == 0) {
              early_coef[slot] = cf;
              early_job[slot] = jb;
            }
          }
          pop = true;
        } else {
          // frame accessors: frame entry (i, j) = A(i, j) for a row pivot, A(j, i) for a column
          // pivot; frame line counts likewise
          auto at = [&](int i, int j) -> int32_t { return colpiv ? W[j * S + i] : W[i * S + j]; };
          const int frc = colpiv ? cc : rc, fcc = colpiv ? rc : cc;
          // the pivot line's nonzeros p0 < p1 < ... and their values (Eq. (2)'s a, b, c, d)
          const int32_t pv = lane < n ? at(r, lane) : 0;
          unsigned pm = __ballot_sync(kFull, pv != 0);
          int p[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            p[t] = pm ? __ffs(pm) - 1 : 0;
            pm &= pm - 1;
          }
          int32_t v[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) v[t] = __shfl_sync(kFull, pv, p[t]);
          FKid kid[2];
          int nk;
          if (s == 1) {
            kid[0] = {1, -1, p[0], 0, 0};
            nk = 1;
          } else {
            kid[0] = {0, p[0], p[1], v[0], v[1]};
            nk = 1;
            if (s == 3) {
              kid[1] = {1, -1, p[2], 0, 0};
              nk = 2;
            } else if (s == 4) {
              kid[1] = {0, p[2], p[3], v[2], v[3]};
              nk = 2;
            }
          }
          // survival (no zero line, reading R4), overflow, and the child's line counts
          int alive[2] = {0, 0};
          int crc[2] = {0, 0}, ccc[2] = {0, 0};  // the child's physical counts (lane = child index)
          int64_t kcf[2] = {cf, cf};
          bool ovf = false;
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            if (c >= nk) break;
            const FKid k = kid[c];
            int nrc = 1, ncc = 1;  // frame counts of row `lane` / column `lane` in the child
            bool mnz = false;
            if (k.minor) {
              if (lane < n) {
                nrc = frc - (at(lane, k.kb) != 0);
                ncc = fcc - (pv != 0);  // pv = frame (r, lane)
              }
              const int32_t pvk = c == 0 ? v[0] : v[2];
              const __int128 prod = (__int128)cf * pvk;
              if (prod > (__int128)INT64_MAX || prod < (__int128)INT64_MIN) ovf = true;
              kcf[c] = (int64_t)prod;
            } else {
              if (lane < n && lane != r) {
                const int32_t va = at(lane, k.ka), vb = at(lane, k.kb);
                const long long mv = (long long)k.al * vb + (long long)k.be * va;
                if (mv > INT32_MAX || mv < INT32_MIN) ovf = true;
                mnz = mv != 0;
                nrc = frc - (va != 0) - (vb != 0) + (mnz ? 1 : 0);
              }
              const int mcnt = __popc(__ballot_sync(kFull, mnz));
              if (lane < n) ncc = lane == k.ka ? mcnt : fcc - (pv != 0);
            }
            const bool dead = lane < n && ((lane != r && nrc == 0) || (lane != k.kb && ncc == 0));
            alive[c] = __all_sync(kFull, !dead) ? 1 : 0;
            // child frame index ii <- parent lane ii + (ii >= r), jj <- jj + (jj >= kb)
            const int fr = __shfl_sync(kFull, nrc, lane + (lane >= r) < 32 ? lane + (lane >= r) : 31);
            const int fc = __shfl_sync(kFull, ncc, lane + (lane >= k.kb) < 32 ? lane + (lane >= k.kb) : 31);
            crc[c] = colpiv ? fc : fr;
            ccc[c] = colpiv ? fr : fc;
          }
          if (__any_sync(kFull, ovf) && lane == 0) atomicOr(err, 1);
          // physical deletion / merge of each child (row pivot: frame = A; column pivot: the
          // frame's column ops are row ops of A)
          auto phys = [&](const FKid& k, int& dr, int& dc, int& merge, int& keep) {
            dr = colpiv ? k.kb : r;
            dc = colpiv ? r : k.kb;
            merge = k.minor ? 0 : (colpiv ? 2 : 1);
            keep = k.ka;
          };
          const int m = n - 1;
          int32_t* Wn = cur ? Wb0 : Wb1;
          if (alive[0] && alive[1]) {
            // second child -> stack slot m (coef | counts | entries, stride m)
            int dr, dc, mg, kp;
            phys(kid[1], dr, dc, mg, kp);
            int32_t* sl = stk + slot_prefix(L, m);
            build_child(W, S, m, dr, dc, mg, kp, kid[1].al, kid[1].be, sl + 2 + m, m, lane);
            if (lane < m) sl[2 + lane] = crc[1] | (ccc[1] << 16);
            if (lane == 0) *reinterpret_cast<int64_t*>(sl) = kcf[1];
            pending |= 1u << m;
          }
          const int first = alive[0] ? 0 : alive[1] ? 1 : -1;
          if (first < 0) {
            pop = true;
          } else {
            // (selects, not dynamic indexing: the kid / count arrays stay in registers)
            const FKid kf = first == 0 ? kid[0] : kid[1];
            int dr, dc, mg, kp;
            phys(kf, dr, dc, mg, kp);
            build_child(W, S, m, dr, dc, mg, kp, kf.al, kf.be, Wn, S, lane);
            __syncwarp();
            W = Wn;
            cur ^= 1;
            n = m;
            rc = first == 0 ? crc[0] : crc[1];
            cc = first == 0 ? ccc[0] : ccc[1];
            cf = first == 0 ? kcf[0] : kcf[1];
          }
        }
      }
      if (pop) {
        if (!pending) break;
        const int m = __ffs(pending) - 1;  // the deepest pending sibling
        pending &= pending - 1;
        const int32_t* sl = stk + slot_prefix(L, m);
        __syncwarp();
        const uint32_t mg = (uint32_t)(0xffffffffull / (uint32_t)m) + 1u;
        for (int e = lane; e < m * m; e += 32) {
          const int i = (int)__umulhi((uint32_t)e, mg);
          W[i * S + (e - i * m)] = sl[2 + m + e];
        }
        const int pk = lane < m ? sl[2 + lane] : 0;
        rc = pk & 0xffff;
        cc = pk >> 16;
        cf = *reinterpret_cast<const int64_t*>(sl);
        n = m;
        __syncwarp();
      }
    }
  }
}

}  // namespace
}  // namespace sperm

using namespace sperm;

static std::mutex g_sub_mu;
static double g_sub_bytes = 0.0, g_sub_nodes = 0.0;

extern "C" int sperm_expand_subtree(const int32_t* d_in_mats, const int64_t* d_in_coef, const int32_t* d_in_job,
                                    int n, int64_t count, int leaf_order, int32_t* d_out_mats, int64_t* d_out_coef,
                                    int32_t* d_out_job, int64_t cap_out, int32_t* d_early_mats,
                                    int64_t* d_early_coef, int32_t* d_early_job, int64_t cap_early,
                                    int64_t* h_out_count, int64_t* h_early_count, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  keep_pool_memory();
  if (!h_out_count || !h_early_count) return set_error(SPERM_ERR_ARG, "sperm_expand_subtree: NULL count outputs");
  *h_out_count = 0;
  *h_early_count = 0;
  const int L = leaf_order;
  if (n < 2 || n > 32) return set_error(SPERM_ERR_ARG, "sperm_expand_subtree: n out of range [2, 32]");
  if (L < 1 || L >= n) return set_error(SPERM_ERR_ARG, "sperm_expand_subtree: leaf_order out of range [1, n-1]");
  if (count < 0) return set_error(SPERM_ERR_ARG, "sperm_expand_subtree: count < 0");
  if (count == 0) return SPERM_OK;
  if (!d_in_mats) return set_error(SPERM_ERR_ARG, "sperm_expand_subtree: d_in_mats is NULL");
  if (cap_out > 0 && (!d_out_mats || !d_out_coef || !d_out_job))
    return set_error(SPERM_ERR_ARG, "sperm_expand_subtree: NULL leaf output");
  if (cap_early > 0 && (!d_early_mats || !d_early_coef || !d_early_job))
    return set_error(SPERM_ERR_ARG, "sperm_expand_subtree: NULL early output");
  static const int gstack_env = [] {  // A-B knob: 0 = stack in shared memory
    const char* e = getenv("SPERM_SUBTREE_GSTACK");
    return e ? atoi(e) : 1;
  }();
  static const int noatomic_env = [] {  // timing experiment only (wrong output)
    const char* e = getenv("SPERM_SUBTREE_NOATOMIC");
    return e ? atoi(e) : 0;
  }();
  const bool gstack = gstack_env != 0;
  const int stack_words = slot_prefix(L, n);
  const int ww = gstack ? ((2 * n * (n | 1)) + 3) / 4 * 4 : sub_warp_words(n, L);
  const size_t smem = (size_t)kSubWarps * ww * 4;
  if (smem > 227 * 1024) return set_error(SPERM_ERR_ARG, "sperm_expand_subtree: stack exceeds shared memory");
  auto kern = gstack ? (noatomic_env ? subtree_kernel<true, true> : subtree_kernel<true, false>)
                     : (noatomic_env ? subtree_kernel<false, true> : subtree_kernel<false, false>);
  {
    static std::atomic<unsigned> attr_done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned bit = 1u << (dev & 31);
    if (!(attr_done.load() & bit)) {
      for (auto k : {subtree_kernel<true, true>, subtree_kernel<true, false>, subtree_kernel<false, true>,
                     subtree_kernel<false, false>})
        SPERM_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      attr_done.fetch_or(bit);
    }
  }
  int per_sm = 0;
  SPERM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * kSubWarps, smem));
  int64_t grid = (int64_t)sm_count() * std::max(per_sm, 1);
  grid = std::max<int64_t>(1, std::min<int64_t>(grid, (count + kSubWarps - 1) / kSubWarps));
  // workspace: root ticket, leaf count, early count (u64) | err (i32)
  unsigned long long* ws = nullptr;
  const size_t gwords = gstack ? (size_t)grid * kSubWarps * stack_words : 0;
  SPERM_CUDA(cudaMallocAsync((void**)&ws, sizeof(unsigned long long) * 4 + 4 * gwords, st));
  SPERM_CUDA(cudaMemsetAsync(ws, 0, sizeof(unsigned long long) * 4, st));
  int* err = reinterpret_cast<int*>(ws + 3);
  int32_t* gstk = gstack ? reinterpret_cast<int32_t*>(ws + 4) : nullptr;
  {
    TimingScope ts("expand", st);
    count_launch();
    kern<<<(unsigned)grid, 32 * kSubWarps, smem, st>>>(d_in_mats, d_in_coef, d_in_job, n, count, L, ww, d_out_mats,
                                                       d_out_coef, d_out_job, cap_out, d_early_mats, d_early_coef,
                                                       d_early_job, cap_early, ws, err, gstk, stack_words);
  }
  cudaError_t le = cudaGetLastError();
  if (le != cudaSuccess) {
    cudaFreeAsync(ws, st);
    return cuda_check(le, "subtree_kernel");
  }
  unsigned long long hw[4] = {0, 0, 0, 0};
  SPERM_CUDA(cudaMemcpyAsync(hw, ws, sizeof(hw), cudaMemcpyDeviceToHost, st));
  cudaFreeAsync(ws, st);
  le = cudaStreamSynchronize(st);
  if (le != cudaSuccess) return cuda_check(le, "sperm_expand_subtree read-back");
  const int herr = (int)(hw[3] & 0xffffffffull);
  *h_out_count = (int64_t)hw[1];
  *h_early_count = (int64_t)hw[2];
  if (herr & 1) return set_error(SPERM_ERR_RANGE, "sperm_expand_subtree: merged entry or coefficient overflow");
  if ((herr & 2) || (int64_t)hw[1] > cap_out)
    return set_error(SPERM_ERR_CAPACITY, "sperm_expand_subtree: leaf capacity too small (roots abandoned)");
  if ((int64_t)hw[2] > cap_early)
    return set_error(SPERM_ERR_CAPACITY, "sperm_expand_subtree: early capacity too small");
  {
    std::lock_guard<std::mutex> lk(g_sub_mu);
    g_sub_bytes += (double)count * (4.0 * n * n + 12.0) + (double)hw[1] * (4.0 * L * L + 12.0) +
                   (double)hw[2] * (4.0 * n * n + 12.0);
    g_sub_nodes += (double)count;
  }
  return SPERM_OK;
}

extern "C" int sperm_expand_subtree_stats(double* h_bytes, double* h_roots, int reset) {
  std::lock_guard<std::mutex> lk(g_sub_mu);
  if (h_bytes) *h_bytes = g_sub_bytes;
  if (h_roots) *h_roots = g_sub_nodes;
  if (reset) g_sub_bytes = g_sub_nodes = 0.0;
  return SPERM_OK;
}
