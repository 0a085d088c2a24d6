// expand.cu — one breadth-first level of Algorithm PH Step 2:
// every node is split by Eq. (2) on its pivot line (Algorithm
// H_per Step 1) into at most two children of order n-1.
//
// One warp per node, one pass (expand_level_kernel): the node is staged in shared memory, the
// pivot picked (lane-per-line counts) and each child tested for survival from the line counts
// (no zero line, reading R4); a decoupled look-back over tiles of consecutive nodes gives every
// surviving child its output slot in natural order (parents in order, A1 before A2 — stable,
// reading R6), and the children are written output-element parallel (write_dense).
//
// A child is described by the lines it deletes and the merge it performs:
//   row pivot r, merge of p_a,p_b:  delete row r, column p_b; column p_a := al*col(p_b) + be*col(p_a)
//   row pivot r, cofactor at p:     delete row r, column p;   coef *= a_rp
//   column pivot c (= row pivot of A^T, reading R2): the same with rows and columns exchanged.
#include <algorithm>
#include <cstdint>
#include <atomic>
#include <cstdlib>
#include <mutex>


#include "common.cuh"

namespace sperm {
namespace {

constexpr int kExpThreads = 256;

struct Child {
  int del_row, del_col;
  int merge;  // 0 none, 1 column merge (keep col := al*col(del_col) + be*col(keep)), 2 row merge
  int keep;
  int32_t al, be;
  int64_t coef;
  bool valid;  // false if an entry or the coefficient overflowed
};

struct Plan {
  int nkids;  // 0..2 candidate children (before the zero-line test)
  int early;  // 1: s >= 5, node kept unsplit
  Child kid[2];
};

// A staged node: shared-memory copy with row stride ns = n | 1 (odd), so that a warp reading
// one column (lane = row) and a warp reading one row (lane = column) both hit 32 distinct banks.
struct NodeView {
  const int32_t* a;
  int n, ns;
  __device__ __forceinline__ int32_t at(int i, int j) const { return a[i * ns + j]; }
};

__host__ __device__ __forceinline__ int stage_stride(int n) { return n | 1; }

// Pivot selection and the Eq. (2) children of one node (warp-uniform result).  Line counts by
// lane-per-line scans (lane l counts row l and column l; lanes loop for n > 32), written to
// rowcnt/colcnt for the survival test.
__device__ Plan plan_node(const NodeView& A, int64_t coef, int lane, int* rowcnt, int* colcnt) {
  const int n = A.n;
  int best_row_key = 0x7fffffff;  // (count << 8) | index, min = fewest nonzeros, lowest index
  int best_col_key = 0x7fffffff;
  for (int l = lane; l < n; l += 32) {
    int rc = 0, cc = 0;
#pragma unroll 4
    for (int j = 0; j < n; ++j) {
      rc += A.at(l, j) != 0;
      cc += A.at(j, l) != 0;
    }
    rowcnt[l] = rc;
    colcnt[l] = cc;
    best_row_key = min(best_row_key, (rc << 8) | l);
    best_col_key = min(best_col_key, (cc << 8) | l);
  }
  for (int o = 16; o; o >>= 1) {
    best_row_key = min(best_row_key, __shfl_xor_sync(0xffffffffu, best_row_key, o));
    best_col_key = min(best_col_key, __shfl_xor_sync(0xffffffffu, best_col_key, o));
  }
  __syncwarp();
  Plan pl;
  pl.nkids = 0;
  pl.early = 0;
  const int srow = best_row_key >> 8, scol = best_col_key >> 8;
  const bool colpiv = scol < srow;  // rows first; a column only if strictly fewer (R2)
  const int s = colpiv ? scol : srow;
  const int idx = colpiv ? (best_col_key & 0xff) : (best_row_key & 0xff);
  if (s == 0) return pl;
  if (s >= 5) {
    pl.early = 1;
    return pl;
  }
  // positions and values of the pivot line's nonzeros, ascending
  int pos[4];
  int32_t val[4];
  int cnt = 0;
  for (int c0 = 0; c0 < n; c0 += 32) {
    const int t = c0 + lane;
    int32_t v = 0;
    if (t < n) v = colpiv ? A.at(t, idx) : A.at(idx, t);
    unsigned b = __ballot_sync(0xffffffffu, v != 0);
    while (b) {
      const int l = __ffs(b) - 1;
      b &= b - 1;
      const int32_t vv = __shfl_sync(0xffffffffu, v, l);
#pragma unroll
      for (int t = 0; t < 4; ++t)  // static indices: pos/val stay in registers
        if (cnt == t) {
          pos[t] = c0 + l;
          val[t] = vv;
        }
      ++cnt;
    }
  }
  auto merge_child = [&](int pa, int pb, int32_t al, int32_t be) {
    Child ch;
    ch.merge = colpiv ? 2 : 1;
    ch.del_row = colpiv ? pb : idx;
    ch.del_col = colpiv ? idx : pb;
    ch.keep = pa;
    ch.al = al;
    ch.be = be;
    ch.coef = coef;
    ch.valid = true;
    return ch;
  };
  auto minor_child = [&](int p, int32_t v) {
    Child ch;
    ch.merge = 0;
    ch.del_row = colpiv ? p : idx;
    ch.del_col = colpiv ? idx : p;
    ch.keep = -1;
    ch.al = ch.be = 0;
    const __int128 r = (__int128)coef * v;
    ch.valid = r <= (__int128)INT64_MAX && r >= (__int128)INT64_MIN;
    ch.coef = (int64_t)r;
    return ch;
  };
  if (s == 1) {
    pl.kid[0] = minor_child(pos[0], val[0]);
    pl.nkids = 1;
  } else {
    pl.kid[0] = merge_child(pos[0], pos[1], val[0], val[1]);
    pl.nkids = 1;
    if (s == 3) {
      pl.kid[1] = minor_child(pos[2], val[2]);
      pl.nkids = 2;
    } else if (s == 4) {
      pl.kid[1] = merge_child(pos[2], pos[3], val[2], val[3]);
      pl.nkids = 2;
    }
  }
  return pl;
}

// Survival test of a child (reading R4: no zero row or column) from the parent's line counts
// and the few lines the child changes — O(n) per child instead of rebuilding it.  Row i of a
// column-merge child is nonzero iff it keeps a nonzero outside the two merged columns or its
// merged entry is nonzero; an unmerged column is nonzero iff it has a nonzero outside the
// deleted row; the merged column iff some merged entry is nonzero (and symmetrically for a
// row merge, which is a column pivot).  Also flags int32 overflow of merged entries.
__device__ int survives(const NodeView& A, const Child& ch, const int* __restrict__ rowcnt,
                        const int* __restrict__ colcnt, int lane, bool* ovf) {
  const int n = A.n;
  bool ok = true, over = false, merged_nz = false;
  if (ch.merge == 0) {
    const int r = ch.del_row, p = ch.del_col;
    for (int i = lane; i < n; i += 32) {
      if (i != r && rowcnt[i] - (A.at(i, p) != 0) == 0) ok = false;
      if (i != p && colcnt[i] - (A.at(r, i) != 0) == 0) ok = false;
    }
    merged_nz = true;
  } else if (ch.merge == 1) {  // row pivot r: column keep := al*col(del_col) + be*col(keep)
    const int r = ch.del_row, ka = ch.keep, kb = ch.del_col;
    for (int i = lane; i < n; i += 32) {
      if (i != r) {
        const int32_t va = A.at(i, ka), vb = A.at(i, kb);
        const long long mv = (long long)ch.al * vb + (long long)ch.be * va;
        if (mv > INT32_MAX || mv < INT32_MIN) over = true;
        if (mv != 0) merged_nz = true;
        else if (rowcnt[i] - (va != 0) - (vb != 0) == 0) ok = false;
      }
      if (i != ka && i != kb && colcnt[i] - (A.at(r, i) != 0) == 0) ok = false;
    }
  } else {  // column pivot c: row keep := al*row(del_row) + be*row(keep)
    const int c = ch.del_col, ka = ch.keep, kb = ch.del_row;
    for (int j = lane; j < n; j += 32) {
      if (j != c) {
        const int32_t va = A.at(ka, j), vb = A.at(kb, j);
        const long long mv = (long long)ch.al * vb + (long long)ch.be * va;
        if (mv > INT32_MAX || mv < INT32_MIN) over = true;
        if (mv != 0) merged_nz = true;
        else if (colcnt[j] - (va != 0) - (vb != 0) == 0) ok = false;
      }
      if (j != ka && j != kb && rowcnt[j] - (A.at(j, c) != 0) == 0) ok = false;
    }
  }
  ok = __all_sync(0xffffffffu, ok) && __any_sync(0xffffffffu, merged_nz);
  if (__any_sync(0xffffffffu, over)) *ovf = true;
  return ok ? 1 : 0;
}

// Staging moves US words per lane per batch: all of a batch's loads are issued before its
// stores, so a node's whole transfer is in flight at once instead of one dependent load round
// trip per row.  The kernel is instantiated for US = 4, 8, 12, 16 and launched with the
// smallest that covers the node in one batch (n <= 22), so few predicated-off slots are issued.

// Copies the warp's node (dense, row-major in global memory) into its shared-memory slot with
// row stride stage_stride(n); `stage_words` = the slot size in words.
template <int US>
__device__ __forceinline__ NodeView stage_node(const int32_t* __restrict__ g, int n, int stage_words, int lane) {
  extern __shared__ int32_t esm[];
  int32_t* s = esm + (threadIdx.x >> 5) * stage_words;
  const int nn = n * n, ns = stage_stride(n);
  const uint32_t magic = (uint32_t)(0xffffffffull / (uint32_t)n) + 1u;  // e / n for e * n < 2^32
  if (!(n & 1) && !(reinterpret_cast<uintptr_t>(g) & 15)) {
    // even order: n^2 is a multiple of 4 and every node of the level is 16-byte aligned, so a
    // lane moves 4 consecutive entries per 16-byte load (a quarter of the load instructions)
    constexpr int UV = US / 4 > 0 ? US / 4 : 1;
    const int nv = nn >> 2;
    const int4* g4 = reinterpret_cast<const int4*>(g);
    for (int base = 0; base < nv; base += 32 * UV) {
      int4 r[UV];
#pragma unroll
      for (int u = 0; u < UV; ++u) {
        const int v = base + u * 32 + lane;
        r[u] = v < nv ? g4[v] : make_int4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < UV; ++u) {
        const int v = base + u * 32 + lane;
        if (v < nv) {
          const int e = 4 * v, i = (int)__umulhi((uint32_t)e, magic), j = e - i * n;
          const int32_t x[4] = {r[u].x, r[u].y, r[u].z, r[u].w};
#pragma unroll
          for (int t = 0; t < 4; ++t) {  // a vector may cross one row boundary (n = 2 mod 4)
            const bool wrap = j + t >= n;
            s[(i + wrap) * ns + j + t - (wrap ? n : 0)] = x[t];
          }
        }
      }
    }
    __syncwarp();
    NodeView v;
    v.a = s;
    v.n = n;
    v.ns = ns;
    return v;
  }
  for (int base = 0; base < nn; base += 32 * US) {
    int32_t r[US];
#pragma unroll
    for (int u = 0; u < US; ++u) {
      const int e = base + u * 32 + lane;
      r[u] = e < nn ? g[e] : 0;
    }
#pragma unroll
    for (int u = 0; u < US; ++u) {
      const int e = base + u * 32 + lane;
      const int i = (int)__umulhi((uint32_t)e, magic);
      if (e < nn) s[i * ns + (e - i * n)] = r[u];
    }
  }
  __syncwarp();
  NodeView v;
  v.a = s;
  v.n = n;
  v.ns = ns;
  return v;
}

// Writes the n x n block of a staged node, or child `ch` of it (order m = n - 1), densely to
// `out`, output-element parallel: lane l produces elements l, l+32, ... so every store is
// coalesced and a lane's loads are independent.  Child element (ii, jj) is parent element
// (ii + [ii >= del_row], jj + [jj >= del_col]), merged as in Eq. (2) (al * deleted line +
// be * kept line).  The count pass has already rejected any level with an overflowing merged
// entry, so the merge is computed modulo 2^32 (exact whenever the result fits, as it then does).
template <bool CHILD>
__device__ __forceinline__ void write_dense(const NodeView& A, const Child& ch, int32_t* __restrict__ out, int lane) {
  const int m = CHILD ? A.n - 1 : A.n, mm = m * m;
  const int dr = CHILD ? ch.del_row : 0x7fff, dc = CHILD ? ch.del_col : 0x7fff;
  if (m <= 32 && (32 / m) * m >= 22) {
    // row-blocked: lane = (sub, jj) writes column jj of rows sub, sub + R, ... (R = 32 / m rows
    // per step, each step's stores contiguous); the source column and the column-merge test are
    // per lane, the source row and the row-merge test per step — no per-element division.  Used
    // when a step keeps >= 22 of the 32 lanes busy (measured: order-17 and -24 levels 2-5 %
    // faster than the flattened loop below, order 20 (m = 19, 19 lanes) 2.5 % slower)
    const int R = 32 / m, sub = lane / m, jj = lane - sub * m;
    if (sub >= R) return;
    const int j = jj + (jj >= dc);
    const bool colmerge = CHILD && ch.merge == 1 && j == ch.keep;
    const bool rowmerge = CHILD && ch.merge == 2;
#pragma unroll 4
    for (int ii = sub; ii < m; ii += R) {
      const int i = ii + (ii >= dr);
      int32_t v = A.at(i, j);
      if (colmerge)
        v = (int32_t)((uint32_t)ch.al * (uint32_t)A.at(i, ch.del_col) + (uint32_t)ch.be * (uint32_t)v);
      else if (rowmerge && i == ch.keep)
        v = (int32_t)((uint32_t)ch.al * (uint32_t)A.at(ch.del_row, j) + (uint32_t)ch.be * (uint32_t)v);
      out[ii * m + jj] = v;
    }
    return;
  }
  // floor(e / m) = umulhi(e, ceil(2^32 / m)) exactly for e * m < 2^32 (e < 2^14 here)
  const uint32_t magic = (uint32_t)(0xffffffffull / (uint32_t)m) + 1u;
  // batches of 4 elements per lane: the loads come from shared memory and the stores need no
  // round trip, so short batches cost no latency and waste fewer predicated-off slots
  constexpr int UW = 4;
  for (int base = 0; base < mm; base += 32 * UW) {
    int32_t r[UW];
#pragma unroll
    for (int u = 0; u < UW; ++u) {
      const int e = base + u * 32 + lane;
      int32_t v = 0;
      if (e < mm) {
        const int ii = (int)__umulhi((uint32_t)e, magic), jj = e - ii * m;
        const int i = ii + (ii >= dr), j = jj + (jj >= dc);
        v = A.at(i, j);
        if (CHILD) {
          if (ch.merge == 1 && j == ch.keep)
            v = (int32_t)((uint32_t)ch.al * (uint32_t)A.at(i, ch.del_col) + (uint32_t)ch.be * (uint32_t)v);
          else if (ch.merge == 2 && i == ch.keep)
            v = (int32_t)((uint32_t)ch.al * (uint32_t)A.at(ch.del_row, j) + (uint32_t)ch.be * (uint32_t)v);
        }
      }
      r[u] = v;
    }
#pragma unroll
    for (int u = 0; u < UW; ++u) {
      const int e = base + u * 32 + lane;
      if (e < mm) out[e] = r[u];
    }
  }
}

// Tile status of the single-pass scan (decoupled look-back): flag (2 bits: 0 empty,
// 1 aggregate, 2 inclusive prefix) | surviving children (31 bits) | early nodes (31 bits).
constexpr unsigned long long kStFlagAgg = 1ull << 62, kStFlagPre = 2ull << 62;
constexpr unsigned long long kSt31 = (1ull << 31) - 1;
__device__ __forceinline__ unsigned long long st_pack(unsigned long long flag, long long kids, long long early) {
  return flag | ((unsigned long long)kids << 31) | (unsigned long long)early;
}

// One expansion level in a single pass.  A CTA takes the next tile of `wpb` consecutive
// nodes (ticket order = node order), one warp per node: stage it, pick the pivot, test which
// children survive; the tile's child / early counts get their output offsets from the
// preceding tiles by a decoupled look-back, and every warp then writes its children (and
// early node) in natural order.  The node is read from HBM once.  err bits: 1 overflow of a
// merged entry or coefficient, 2 output capacity exceeded or output buffer missing.
//
// ORDERED = false (the H_per recursion below the job level, where only each job's SUM matters,
// not the order of its leaves): the tile's output offsets come from one atomicAdd on the level
// totals instead of the look-back — no waiting on the preceding tiles.
template <int US, bool ORDERED>
__global__ void __launch_bounds__(kExpThreads, 5) expand_level_kernel(
    const int32_t* __restrict__ mats, const int64_t* __restrict__ coef, const int32_t* __restrict__ job,
    int n, int64_t count, int stage_words,
    int32_t* __restrict__ out_mats, int64_t* __restrict__ out_coef, int32_t* __restrict__ out_job, int64_t cap_out,
    int32_t* __restrict__ early_mats, int64_t* __restrict__ early_coef, int32_t* __restrict__ early_job,
    int64_t cap_early, unsigned long long* __restrict__ tile_status, unsigned* __restrict__ ticket,
    long long* __restrict__ totals, int* __restrict__ err) {
  __shared__ int s_tile;
  __shared__ int s_kids[kExpThreads / 32], s_early[kExpThreads / 32];
  __shared__ long long s_base[2];
  __shared__ int s_cnt[kExpThreads / 32][2 * SPERM_EXPAND_NMAX];  // row and column counts per warp
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  if (threadIdx.x == 0) s_tile = (int)atomicAdd(ticket, 1u);
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t node = tile * wpb + w;
  const bool live = node < count;
  NodeView A;
  Plan pl;
  pl.nkids = 0;
  pl.early = 0;
  int kids = 0, mask = 0;
  int64_t cf = 1;
  if (live) {
    A = stage_node<US>(mats + node * (int64_t)n * n, n, stage_words, lane);
    cf = coef ? coef[node] : 1;
    int* rowcnt = s_cnt[w];
    int* colcnt = rowcnt + SPERM_EXPAND_NMAX;
    pl = plan_node(A, cf, lane, rowcnt, colcnt);
    bool ovf = false;
#pragma unroll
    for (int c = 0; c < 2; ++c) {  // static bound: the plan stays in registers
      if (c >= pl.nkids) break;
      if (!pl.kid[c].valid) ovf = true;
      if (survives(A, pl.kid[c], rowcnt, colcnt, lane, &ovf)) {
        ++kids;
        mask |= 1 << c;
      }
    }
    if (ovf && lane == 0) atomicOr(err, 1);
  }
  if (lane == 0) {
    s_kids[w] = kids;
    s_early[w] = pl.early;
  }
  __syncthreads();
  if (w == 0) {
    // warp 0: tile aggregate, publish it, then look back over the preceding tiles 32 at a time
    // (lane l reads tile j - l): aggregates are summed until the nearest inclusive prefix
    long long ak = 0, ae = 0;
    for (int i = 0; i < wpb; ++i) {
      ak += s_kids[i];
      ae += s_early[i];
    }
    long long ek = 0, ee = 0;  // exclusive prefix of this tile
    if (!ORDERED) {
      if (lane == 0) {
        unsigned long long* tu = reinterpret_cast<unsigned long long*>(totals);
        ek = ak ? (long long)atomicAdd(tu, (unsigned long long)ak) : 0;
        ee = ae ? (long long)atomicAdd(tu + 1, (unsigned long long)ae) : 0;
      }
    } else if (tile == 0) {
      if (lane == 0) atomicExch(tile_status, st_pack(kStFlagPre, ak, ae));
    } else {
      if (lane == 0) atomicExch(tile_status + tile, st_pack(kStFlagAgg, ak, ae));
      int64_t j = tile - 1;  // newest tile of the current window
      while (true) {
        const int64_t t = j - lane;
        unsigned long long v = 2ull << 62;  // before tile 0: an empty inclusive prefix
        if (t >= 0) v = *(volatile unsigned long long*)(tile_status + t);
        // wait until every tile of the window up to the nearest prefix has published
        unsigned pre = __ballot_sync(0xffffffffu, (v & (3ull << 62)) == kStFlagPre);
        const unsigned upto = pre ? (pre & (0u - pre)) * 2u - 1u : 0xffffffffu;  // lanes <= first prefix
        if (__ballot_sync(0xffffffffu, (v & (3ull << 62)) == 0ull) & upto) continue;  // re-read the window
        long long k_ = 0, e_ = 0;
        if ((upto >> lane) & 1u && t >= 0) {
          k_ = (long long)((v >> 31) & kSt31);
          e_ = (long long)(v & kSt31);
        }
        for (int o = 16; o; o >>= 1) {
          k_ += __shfl_xor_sync(0xffffffffu, k_, o);
          e_ += __shfl_xor_sync(0xffffffffu, e_, o);
        }
        ek += k_;
        ee += e_;
        if (pre) break;
        j -= 32;
      }
      if (lane == 0) atomicExch(tile_status + tile, st_pack(kStFlagPre, ek + ak, ee + ae));
    }
    if (lane == 0) {
      s_base[0] = ek;
      s_base[1] = ee;
      if (ORDERED && (tile + 1) * wpb >= count) {  // the last tile: level totals
        totals[0] = ek + ak;
        totals[1] = ee + ae;
      }
    }
  }
  __syncthreads();
  if (!live) return;
  long long ok_ = s_base[0], oe = s_base[1];
  for (int i = 0; i < w; ++i) {
    ok_ += s_kids[i];
    oe += s_early[i];
  }
  const int32_t jb = job ? job[node] : (int32_t)node;
  if (pl.early) {
    if (oe >= cap_early || !early_mats || !early_coef || !early_job) {
      if (lane == 0) atomicOr(err, 2);
      return;
    }
    write_dense<false>(A, pl.kid[0], early_mats + oe * (int64_t)n * n, lane);
    if (lane == 0) {
      early_coef[oe] = cf;
      early_job[oe] = jb;
    }
    return;
  }
  if (!kids) return;
  if (ok_ + kids > cap_out || !out_mats || !out_coef || !out_job) {
    if (lane == 0) atomicOr(err, 2);
    return;
  }
  const int64_t m2 = (int64_t)(n - 1) * (n - 1);
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    if ((mask >> c) & 1) {
      write_dense<true>(A, pl.kid[c], out_mats + ok_ * m2, lane);
      if (lane == 0) {
        out_coef[ok_] = pl.kid[c].coef;
        out_job[ok_] = jb;
      }
      ++ok_;
    }
  }
}

// nonzeros of each node (one warp per node, coalesced 4-byte loads, warp-sum): the "size" key of
// the load-balance comparison (the paper's |D| / S regressors, Tables 5-7's
// alternatives to the estimate order)
__global__ void nnz_kernel(const int32_t* __restrict__ mats, int n, int64_t count, int64_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= count) return;
  const int32_t* m = mats + w * (int64_t)n * n;
  int c = 0;
  for (int e = lane; e < n * n; e += 32) c += m[e] != 0;
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) out[w] = c;
}

}  // namespace
}  // namespace sperm

using namespace sperm;

extern "C" int sperm_nnz(const int32_t* d_mats, int n, int64_t count, int64_t* d_out, void* stream) {
  if (n < 0 || n > SPERM_EXPAND_NMAX || count < 0) return set_error(SPERM_ERR_ARG, "sperm_nnz: bad sizes");
  if (count == 0) return SPERM_OK;
  if (!d_out || (n > 0 && !d_mats)) return set_error(SPERM_ERR_ARG, "sperm_nnz: NULL pointer");
  count_launch();
  nnz_kernel<<<(unsigned)((count + 7) / 8), 256, 0, (cudaStream_t)stream>>>(d_mats, n, count, d_out);
  const cudaError_t le = cudaGetLastError();
  return le == cudaSuccess ? SPERM_OK : cuda_check(le, "nnz_kernel");
}

static std::mutex g_exp_mu;
static double g_exp_bytes = 0.0, g_exp_nodes = 0.0;

static int expand_level(bool ordered, const int32_t* d_in_mats, const int64_t* d_in_coef, const int32_t* d_in_job,
                        int n, int64_t count, int32_t* d_out_mats, int64_t* d_out_coef, int32_t* d_out_job,
                        int64_t cap_out, int32_t* d_early_mats, int64_t* d_early_coef, int32_t* d_early_job,
                        int64_t cap_early, int64_t* h_out_count, int64_t* h_early_count, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  keep_pool_memory();
  if (!h_out_count || !h_early_count) return set_error(SPERM_ERR_ARG, "sperm_expand: NULL count outputs");
  *h_out_count = 0;
  *h_early_count = 0;
  if (n < 2 || n > SPERM_EXPAND_NMAX) return set_error(SPERM_ERR_ARG, "sperm_expand: n out of range [2, 128]");
  if (count < 0) return set_error(SPERM_ERR_ARG, "sperm_expand: count < 0");
  if (count >= (int64_t)1 << 30) return set_error(SPERM_ERR_ARG, "sperm_expand: count >= 2^30 (split the level)");
  if (count == 0) return SPERM_OK;
  if (!d_in_mats) return set_error(SPERM_ERR_ARG, "sperm_expand: d_in_mats is NULL");
  // shared-memory staging of each warp's node (row stride n | 1): up to 8 warps per CTA within 200 KB
  const int stage_words = ((n * stage_stride(n) + 3) / 4) * 4;
  const int wpb = std::max(1, std::min(8, (int)((200 * 1024) / (stage_words * 4))));
  const size_t esmem = (size_t)wpb * stage_words * 4;
  const int64_t tiles = (count + wpb - 1) / wpb;
  // workspace: tile status [tiles] u64 | totals [2] i64 | ticket u32, err i32
  unsigned long long* ws = nullptr;
  SPERM_CUDA(cudaMallocAsync((void**)&ws, sizeof(unsigned long long) * (tiles + 3), st));
  SPERM_CUDA(cudaMemsetAsync(ws, 0, sizeof(unsigned long long) * (tiles + 3), st));
  long long* totals = reinterpret_cast<long long*>(ws + tiles);
  unsigned* ticket = reinterpret_cast<unsigned*>(ws + tiles + 2);
  int* err = reinterpret_cast<int*>(ticket + 1);
  const int per_lane = (n * n + 31) / 32;
  auto kern = ordered ? (per_lane <= 4 ? expand_level_kernel<4, true> : per_lane <= 8 ? expand_level_kernel<8, true>
                         : per_lane <= 12 ? expand_level_kernel<12, true> : expand_level_kernel<16, true>)
                      : (per_lane <= 4 ? expand_level_kernel<4, false> : per_lane <= 8 ? expand_level_kernel<8, false>
                         : per_lane <= 12 ? expand_level_kernel<12, false> : expand_level_kernel<16, false>);
  {  // the attribute once per device and kernel, at the 200 KB staging budget (host time per level)
    static std::atomic<unsigned> attr_done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const unsigned bit = 1u << (dev & 31);
    if (!(attr_done.load() & bit)) {
      for (auto k : {expand_level_kernel<4, true>, expand_level_kernel<8, true>, expand_level_kernel<12, true>,
                     expand_level_kernel<16, true>, expand_level_kernel<4, false>, expand_level_kernel<8, false>,
                     expand_level_kernel<12, false>, expand_level_kernel<16, false>})
        SPERM_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      attr_done.fetch_or(bit);
    }
  }
  {
    TimingScope ts("expand", st);
    count_launch();
    kern<<<(unsigned)tiles, 32u * wpb, esmem, st>>>(
        d_in_mats, d_in_coef, d_in_job, n, count, stage_words, d_out_mats, d_out_coef, d_out_job, cap_out,
        d_early_mats, d_early_coef, d_early_job, cap_early, ws, ticket, totals, err);
  }
  cudaError_t le = cudaGetLastError();
  if (le != cudaSuccess) {
    cudaFreeAsync(ws, st);
    return cuda_check(le, "expand_level_kernel");
  }
  long long tot[2] = {0, 0};
  int herr = 0;
  SPERM_CUDA(cudaMemcpyAsync(tot, totals, sizeof(tot), cudaMemcpyDeviceToHost, st));
  SPERM_CUDA(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, st));
  cudaFreeAsync(ws, st);
  le = cudaStreamSynchronize(st);
  if (le != cudaSuccess) return cuda_check(le, "sperm_expand read-back");
  *h_out_count = tot[0];
  *h_early_count = tot[1];
  if (herr & 1) return set_error(SPERM_ERR_RANGE, "sperm_expand: merged entry or coefficient overflow");
  if (tot[0] > cap_out || tot[1] > cap_early)
    return set_error(SPERM_ERR_CAPACITY, "sperm_expand: output capacity too small");
  if (herr & 2) return set_error(SPERM_ERR_ARG, "sperm_expand: NULL output buffer");
  {
    // algorithmic bytes of the level: every parent read once (matrix + coef + job), every
    // child and early node written once
    std::lock_guard<std::mutex> lk(g_exp_mu);
    g_exp_bytes += (double)count * (4.0 * n * n + 12.0) + (double)tot[0] * (4.0 * (n - 1) * (n - 1) + 12.0) +
                   (double)tot[1] * (4.0 * n * n + 12.0);
    g_exp_nodes += (double)count;
  }
  return SPERM_OK;
}

extern "C" int sperm_expand(const int32_t* d_in_mats, const int64_t* d_in_coef, const int32_t* d_in_job, int n,
                            int64_t count, int32_t* d_out_mats, int64_t* d_out_coef, int32_t* d_out_job,
                            int64_t cap_out, int32_t* d_early_mats, int64_t* d_early_coef, int32_t* d_early_job,
                            int64_t cap_early, int64_t* h_out_count, int64_t* h_early_count, void* stream) {
  return expand_level(true, d_in_mats, d_in_coef, d_in_job, n, count, d_out_mats, d_out_coef, d_out_job, cap_out,
                      d_early_mats, d_early_coef, d_early_job, cap_early, h_out_count, h_early_count, stream);
}

extern "C" int sperm_expand_unordered(const int32_t* d_in_mats, const int64_t* d_in_coef, const int32_t* d_in_job,
                                      int n, int64_t count, int32_t* d_out_mats, int64_t* d_out_coef,
                                      int32_t* d_out_job, int64_t cap_out, int32_t* d_early_mats,
                                      int64_t* d_early_coef, int32_t* d_early_job, int64_t cap_early,
                                      int64_t* h_out_count, int64_t* h_early_count, void* stream) {
  return expand_level(false, d_in_mats, d_in_coef, d_in_job, n, count, d_out_mats, d_out_coef, d_out_job, cap_out,
                      d_early_mats, d_early_coef, d_early_job, cap_early, h_out_count, h_early_count, stream);
}

extern "C" int sperm_expand_stats(double* h_bytes, double* h_nodes, int reset) {
  std::lock_guard<std::mutex> lk(g_exp_mu);
  if (h_bytes) *h_bytes = g_exp_bytes;
  if (h_nodes) *h_nodes = g_exp_nodes;
  if (reset) g_exp_bytes = g_exp_nodes = 0.0;
  return SPERM_OK;
}
