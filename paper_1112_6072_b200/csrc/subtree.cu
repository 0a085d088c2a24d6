// subtree.cu — Algorithm H_per's recursion (Step 1's pivot line, Eq. (2)'s
// split) below the job level, DEPTH FIRST and entirely on chip.
//
// Below the job level a job's value is the sum over its leaves, so the order in which its leaves
// appear does not matter (the job list itself, PH Step 2, keeps the ordered level kernel of
// expand.cu).  The level-by-level expansion writes every intermediate node to HBM and reads it
// back one level later, and builds every child densely (O(n^2) per child).  Here one warp takes a
// root node (order n0 <= 32) and walks its whole subtree down to the leaves of order L with O(n)
// work per node:
//
//   * the root is staged once in shared memory (M, row stride n0 | 1: lane-per-row and
//     lane-per-column accesses are both bank-conflict free) and every node of its subtree is a
//     VIEW of M: lane i holds the node's row map R[i] and column map C[i] (entry (i, j) of the
//     node = M[R[i]][C[j]]) and the nonzero counts of its row i and column i;
//   * a child deletes one row and one column (two shuffles of the maps) and, for Eq. (2)'s merge,
//     overwrites one line of M in place (line ka := al * line kb + be * line ka: one load pair
//     and store per lane); its line counts are derived from the parent's in O(n), so no node is
//     ever rescanned or copied;
//   * the pivot (reading R2: fewest nonzeros, rows before columns, lowest index) is two warp
//     min-reductions over the lanes' packed (count, index) keys; the pivot line's nonzeros come
//     from one ballot;
//   * a split with two surviving children (s = 3, 4) continues with the first and pushes a frame
//     (the parent's maps, the second child's split and counts) to the warp's stack; every in-place
//     merge made while a frame is pending logs the line it overwrites, and popping a frame replays
//     the log back to the frame's mark (M is the parent's again) before applying the second
//     child's split.  Frames and the log (<= n0 - L entries each) live in a per-warp scratch area
//     in global memory (L2-resident), so shared memory holds only M and many warps fit per SM;
//   * a node of order <= L is a leaf: gathered through its maps and written densely to HBM (one
//     atomic slot per leaf); a node with s >= 5 (reading R5: not split) is written to the early
//     outputs padded to order n0 by an identity block (per(diag(X, I)) = per(X)).
//
// The same children as expand.cu's kernel (same Eq. (2) scalars, the same zero-line test of
// reading R4, the same overflow checks): the leaves form the same multiset as the level-by-level
// recursion's, in an unspecified order.
//
// History (C100, L = 15): dense children with the stack in shared memory 5.18 s of
// expansion; stack in global scratch 3.72 s (occupancy was the limit, not the leaf atomic); ncu
// then showed the dense child copies at ~45 % of the instructions (4300 per leaf) -> this view form.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "common.cuh"

namespace sperm {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kSubWarps = 4;  // warps per CTA
// per-warp scratch (words): frames [depth + 1][kFrameW] | undo log [depth + 1][kUndoW]
constexpr int kFrameW = 112;  // header (12 words) | parent row map [32] | parent column map [32] | child counts [32]
constexpr int kUndoW = 34;    // line (1 word: column index, or row index | 0x100) | the line's 32 values | pad

// A child in the pivot's frame (the frame is A for a row pivot, A^T for a column pivot: frame row
// r = the pivot line).  Minor: delete frame row r and frame column kb, coef *= the pivot entry.
// Merge: delete frame row r and frame column kb, frame column ka := al*col(kb) + be*col(ka).
struct FKid {
  int minor;  // 1 minor, 0 merge
  int ka, kb;
  int32_t al, be;
};

// frame entry (physical row fr, physical column fc) of the view: M[fr][fc] for a row pivot,
// M[fc][fr] for a column pivot (frame rows are the node's columns) = M[fr * ra + fc * ca] with the
// frame strides ra = colpiv ? 1 : S, ca = colpiv ? S : 1 — the kernel keeps fr * ra and fc * ca
// (scaled indices) so that an access is one add

__global__ void __launch_bounds__(32 * kSubWarps) subtree_kernel(
    const int32_t* __restrict__ mats, const int64_t* __restrict__ coef, const int32_t* __restrict__ job, int n0,
    int64_t count, int L, int32_t* __restrict__ out_mats, int64_t* __restrict__ out_coef,
    int32_t* __restrict__ out_job, int64_t cap_out, int32_t* __restrict__ early_mats,
    int64_t* __restrict__ early_coef, int32_t* __restrict__ early_job, int64_t cap_early,
    unsigned long long* __restrict__ ws, int* __restrict__ err, int32_t* __restrict__ scratch, int scratch_words) {
  extern __shared__ int32_t ssm[];
  const int lane = threadIdx.x & 31;
  const int S = n0 | 1;
  int32_t* const M = ssm + (threadIdx.x >> 5) * (((n0 * S) + 3) / 4 * 4);
  int32_t* const frames = scratch + ((int64_t)blockIdx.x * kSubWarps + (threadIdx.x >> 5)) * scratch_words;
  int32_t* const ulog = frames + (n0 - L + 1) * kFrameW;
  const uint32_t magic0 = (uint32_t)(0xffffffffull / (uint32_t)n0) + 1u;
  const uint32_t magicL = (uint32_t)(0xffffffffull / (uint32_t)L) + 1u;
  while (true) {
    unsigned long long root = 0;
    if (lane == 0) root = (*(volatile int*)err & 2) ? ~0ull : atomicAdd(ws, 1ull);  // stop on a full output
    root = __shfl_sync(kFull, root, 0);
    if (root >= (unsigned long long)count) break;
    // ---- the root: staged (all of a batch's loads before its stores) and its line counts
    __syncwarp();
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
          if (e < nn) M[i * S + (e - i * n0)] = r[u];
        }
      }
    }
    __syncwarp();
    int n = n0;
    int64_t cf = coef ? coef[root] : 1;
    const int32_t jb = job ? job[root] : (int32_t)root;
    int rid = lane, cid = lane;  // the view's row / column maps (lane i: R[i], C[i])
    int rc = 0, cc = 0;           // lane i: nonzeros of row i and of column i of the view
    if (lane < n)
      for (int j = 0; j < n; ++j) {
        rc += M[lane * S + j] != 0;
        cc += M[j * S + lane] != 0;
      }
    int nfr = 0, nlog = 0;  // pending frames, undo-log entries
    // applies a child's split to the view (maps, and for a merge the line of M, logged while a
    // frame is pending); frame maps: FR = colpiv ? C : R, FC = colpiv ? R : C
    auto apply = [&](bool colpiv, int r, const FKid& k) {
      const int FR = colpiv ? cid : rid, FC = colpiv ? rid : cid;
      if (!k.minor) {
        const int ra = colpiv ? 1 : S, ca = colpiv ? S : 1;
        const int pk = __shfl_sync(kFull, FC, k.ka), pb = __shfl_sync(kFull, FC, k.kb);
        const int pkA = pk * ca, pbA = pb * ca;
        if (nfr > 0) {  // log the whole physical line pk (n0 values) before overwriting it
          int32_t* u = ulog + nlog * kUndoW;
          if (lane < n0) u[1 + lane] = M[lane * ra + pkA];
          if (lane == 0) u[0] = colpiv ? (pk | 0x100) : pk;
          ++nlog;
          __syncwarp();  // every lane has read its logged entry before the line is overwritten
        }
        if (lane < n) {
          const int frA = FR * ra;
          const int32_t x = M[frA + pkA], y = M[frA + pbA];
          M[frA + pkA] = (int32_t)((uint32_t)k.al * (uint32_t)y + (uint32_t)k.be * (uint32_t)x);
        }
      }
      // delete frame row r and frame column kb: lane ii takes the map entry ii + (ii >= r)
      const int fr2 = __shfl_sync(kFull, FR, min(lane + (lane >= r), 31));
      const int fc2 = __shfl_sync(kFull, FC, min(lane + (lane >= k.kb), 31));
      rid = colpiv ? fc2 : fr2;
      cid = colpiv ? fr2 : fc2;
      __syncwarp();
    };
    while (true) {
      bool pop = false;
      if (n <= L) {
        // ---- leaf (order L): one output slot; gathered through the maps, row-major
        unsigned long long slot = 0;
        if (lane == 0) slot = atomicAdd(ws + 1, 1ull);
        slot = __shfl_sync(kFull, slot, 0);
        if ((int64_t)slot < cap_out) {
          int32_t* o = out_mats + (int64_t)slot * L * L;
          if (L <= 16) {  // two rows per step: half-warp h writes row 2t + h, lane j of it column j
            const int h = lane >> 4, j = lane & 15;
            const int pc = __shfl_sync(kFull, cid, j);
            for (int i0 = 0; i0 < L; i0 += 2) {
              const int i = i0 + h;
              const int pr = __shfl_sync(kFull, rid, i & 31);
              if (i < L && j < L) o[i * L + j] = M[pr * S + pc];
            }
          } else {
            for (int b = 0; b < L * L; b += 32) {
              const int e = b + lane;
              const int i = (int)__umulhi((uint32_t)e, magicL), j = e - i * L;
              const int pr = __shfl_sync(kFull, rid, i & 31), pc = __shfl_sync(kFull, cid, j & 31);
              if (e < L * L) o[e] = M[pr * S + pc];
            }
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
            for (int b = 0; b < n0 * n0; b += 32) {
              const int e = b + lane;
              const int i = (int)__umulhi((uint32_t)e, magic0), j = e - i * n0;
              const int pr = __shfl_sync(kFull, rid, i & 31), pc = __shfl_sync(kFull, cid, j & 31);
              if (e < n0 * n0) o[e] = (i < n && j < n) ? M[pr * S + pc] : (i == j ? 1 : 0);
            }
            if (lane == 0) {
              early_coef[slot] = cf;
              early_job[slot] = jb;
            }
          }
          pop = true;
        } else {
          const int FR = colpiv ? cid : rid, FC = colpiv ? rid : cid;
          const int frc = colpiv ? cc : rc, fcc = colpiv ? rc : cc;  // frame line counts
          const int frA = FR * (colpiv ? 1 : S), fcA = FC * (colpiv ? S : 1);  // scaled (see above)
          const int FRrA = __shfl_sync(kFull, frA, r);                           // the pivot line
          // the pivot line's nonzeros p0 < p1 < ... and their values (Eq. (2)'s a, b, c, d)
          const int32_t pv = lane < n ? M[FRrA + fcA] : 0;
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
            kid[1] = kid[0];
            nk = 1;
          } else {
            kid[0] = {0, p[0], p[1], v[0], v[1]};
            kid[1] = kid[0];
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
            const int pkbA = __shfl_sync(kFull, fcA, k.kb);
            int nrc = 1, ncc = 1;  // frame counts of row `lane` / column `lane` in the child
            bool mnz = false;
            if (k.minor) {
              if (lane < n) {
                nrc = frc - (M[frA + pkbA] != 0);
                ncc = fcc - (pv != 0);  // pv = frame (r, lane)
              }
              const int32_t pvk = c == 0 ? v[0] : v[2];
              const __int128 prod = (__int128)cf * pvk;
              if (prod > (__int128)INT64_MAX || prod < (__int128)INT64_MIN) ovf = true;
              kcf[c] = (int64_t)prod;
            } else {
              const int pkaA = __shfl_sync(kFull, fcA, k.ka);
              if (lane < n && lane != r) {
                const int32_t va = M[frA + pkaA], vb = M[frA + pkbA];
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
            const int fr = __shfl_sync(kFull, nrc, min(lane + (lane >= r), 31));
            const int fc = __shfl_sync(kFull, ncc, min(lane + (lane >= k.kb), 31));
            crc[c] = colpiv ? fc : fr;
            ccc[c] = colpiv ? fr : fc;
          }
          if (__any_sync(kFull, ovf) && lane == 0) atomicOr(err, 1);
          if (alive[0] && alive[1]) {
            // frame: the parent's maps and order, the second child's split, coefficient and counts
            int32_t* f = frames + nfr * kFrameW;
            if (lane == 0) {
              f[0] = nlog;
              f[1] = n;
              f[2] = colpiv;
              f[3] = r;
              f[4] = kid[1].minor;
              f[5] = kid[1].ka;
              f[6] = kid[1].kb;
              f[7] = kid[1].al;
              f[8] = kid[1].be;
              *reinterpret_cast<int64_t*>(f + 10) = kcf[1];
            }
            f[12 + lane] = rid;
            f[44 + lane] = cid;
            f[76 + lane] = crc[1] | (ccc[1] << 16);
            ++nfr;
          }
          const int first = alive[0] ? 0 : alive[1] ? 1 : -1;
          if (first < 0) {
            pop = true;
          } else {
            // (selects, not dynamic indexing: the kid / count arrays stay in registers)
            apply(colpiv, r, first == 0 ? kid[0] : kid[1]);
            n -= 1;
            rc = first == 0 ? crc[0] : crc[1];
            cc = first == 0 ? ccc[0] : ccc[1];
            cf = first == 0 ? kcf[0] : kcf[1];
          }
        }
      }
      if (pop) {
        if (nfr == 0) break;
        // the newest frame: undo the merges logged since it was pushed (newest first), restore
        // the parent's view, then apply the second child's split
        --nfr;
        const int32_t* f = frames + nfr * kFrameW;
        __syncwarp();
        const int mark = f[0];
        while (nlog > mark) {
          --nlog;
          const int32_t* u = ulog + nlog * kUndoW;
          const int line = u[0];
          if (lane < n0) {
            if (line & 0x100) M[(line & 0xff) * S + lane] = u[1 + lane];
            else M[lane * S + line] = u[1 + lane];
          }
          __syncwarp();
        }
        n = f[1];
        const bool colpiv = f[2] != 0;
        const int r = f[3];
        const FKid k = {f[4], f[5], f[6], f[7], f[8]};
        cf = *reinterpret_cast<const int64_t*>(f + 10);
        rid = f[12 + lane];
        cid = f[44 + lane];
        const int pk = f[76 + lane];
        apply(colpiv, r, k);
        n -= 1;
        rc = pk & 0xffff;
        cc = pk >> 16;
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
  const size_t smem = (size_t)kSubWarps * (((n * (n | 1)) + 3) / 4 * 4) * 4;
  const int scratch_words = (n - L + 1) * (kFrameW + kUndoW);
  {
    static std::atomic<unsigned> attr_done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned bit = 1u << (dev & 31);
    if (!(attr_done.load() & bit)) {
      SPERM_CUDA(cudaFuncSetAttribute(subtree_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      attr_done.fetch_or(bit);
    }
  }
  int per_sm = 0;
  SPERM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, subtree_kernel, 32 * kSubWarps, smem));
  int64_t grid = (int64_t)sm_count() * std::max(per_sm, 1);
  grid = std::max<int64_t>(1, std::min<int64_t>(grid, (count + kSubWarps - 1) / kSubWarps));
  // workspace: root ticket, leaf count, early count (u64) | err (i32) | per-warp scratch
  unsigned long long* ws = nullptr;
  const size_t swords = (size_t)grid * kSubWarps * scratch_words;
  SPERM_CUDA(cudaMallocAsync((void**)&ws, sizeof(unsigned long long) * 4 + 4 * swords, st));
  SPERM_CUDA(cudaMemsetAsync(ws, 0, sizeof(unsigned long long) * 4, st));
  int* err = reinterpret_cast<int*>(ws + 3);
  int32_t* scratch = reinterpret_cast<int32_t*>(ws + 4);
  {
    TimingScope ts("expand", st);
    count_launch();
    subtree_kernel<<<(unsigned)grid, 32 * kSubWarps, smem, st>>>(
        d_in_mats, d_in_coef, d_in_job, n, count, L, d_out_mats, d_out_coef, d_out_job, cap_out, d_early_mats,
        d_early_coef, d_early_job, cap_early, ws, err, scratch, scratch_words);
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
