// expand.cu — one breadth-first level of Algorithm PH Step 2:
// every node is split by Eq. (2) on its pivot line (Algorithm
// H_per Step 1) into at most two children of order n-1.
//
// One warp per node.  Pass 1 (count) stages the node in shared memory, picks the pivot
// (lane l holds columns l, l+32, ... of the row being scanned) and tests from the line
// counts whether each child survives (no zero line, reading R4); an exclusive scan of the
// per-node child counts gives every child its output slot in natural order (parents in
// order, A1 before A2 — stable, reading R6); pass 2 (emit) writes the surviving children
// output-element parallel (write_child).
//
// A child is described by the lines it deletes and the merge it performs:
//   row pivot r, merge of p_a,p_b:  delete row r, column p_b; column p_a := al*col(p_b) + be*col(p_a)
//   row pivot r, cofactor at p:     delete row r, column p;   coef *= a_rp
//   column pivot c (= row pivot of A^T, reading R2): the same with rows and columns exchanged.
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include <cub/device/device_scan.cuh>

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
      if (cnt < 4) {
        pos[cnt] = c0 + l;
        val[cnt] = vv;
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

// Words each lane moves per batch: all of a batch's loads are issued before its stores, so a
// node's whole transfer is in flight at once (a node of order <= 22 is one batch) instead of
// one dependent load round trip per row — the expansion levels are latency-bound otherwise.
constexpr int kStageU = 16;

// Copies the warp's node (dense, row-major in global memory) into its shared-memory slot with
// row stride stage_stride(n); `stage_words` = the slot size in words.
__device__ __forceinline__ NodeView stage_node(const int32_t* __restrict__ g, int n, int stage_words, int lane) {
  extern __shared__ int32_t esm[];
  int32_t* s = esm + (threadIdx.x >> 5) * stage_words;
  const int nn = n * n, ns = stage_stride(n);
  const uint32_t magic = (uint32_t)(0xffffffffull / (uint32_t)n) + 1u;  // e / n for e * n < 2^32
  for (int base = 0; base < nn; base += 32 * kStageU) {
    int32_t r[kStageU];
#pragma unroll
    for (int u = 0; u < kStageU; ++u) {
      const int e = base + u * 32 + lane;
      r[u] = e < nn ? g[e] : 0;
    }
#pragma unroll
    for (int u = 0; u < kStageU; ++u) {
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
  // floor(e / m) = umulhi(e, ceil(2^32 / m)) exactly for e * m < 2^32 (e < 2^14 here)
  const uint32_t magic = (uint32_t)(0xffffffffull / (uint32_t)m) + 1u;
  for (int base = 0; base < mm; base += 32 * kStageU) {
    int32_t r[kStageU];
#pragma unroll
    for (int u = 0; u < kStageU; ++u) {
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
    for (int u = 0; u < kStageU; ++u) {
      const int e = base + u * 32 + lane;
      if (e < mm) out[e] = r[u];
    }
  }
}

__global__ void __launch_bounds__(kExpThreads) expand_count_kernel(
    const int32_t* __restrict__ mats, const int64_t* __restrict__ coef, int n, int64_t count,
    int* __restrict__ kid_count, int* __restrict__ early_count, int* __restrict__ kid_mask,
    int* __restrict__ err, int stage_words, Plan* __restrict__ plans) {
  const int lane = threadIdx.x & 31;
  const int64_t node = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (node >= count) return;
  const NodeView A = stage_node(mats + node * (int64_t)n * n, n, stage_words, lane);
  const int64_t cf = coef ? coef[node] : 1;
  __shared__ int s_cnt[kExpThreads / 32][2 * SPERM_EXPAND_NMAX];  // row and column counts per warp
  int* rowcnt = s_cnt[threadIdx.x >> 5];
  int* colcnt = rowcnt + SPERM_EXPAND_NMAX;
  Plan pl = plan_node(A, cf, lane, rowcnt, colcnt);
  int kids = 0, mask = 0;
  bool ovf = false;
  for (int c = 0; c < pl.nkids; ++c) {
    if (!pl.kid[c].valid) ovf = true;
    if (survives(A, pl.kid[c], rowcnt, colcnt, lane, &ovf)) {
      ++kids;
      mask |= 1 << c;
    }
  }
  if (lane == 0) {
    kid_count[node] = kids;
    kid_mask[node] = mask;
    plans[node] = pl;  // the emit pass reuses the pivot and children (no second scan)
    early_count[node] = pl.early;
    if (ovf) atomicOr(err, 1);
  }
}

__global__ void __launch_bounds__(kExpThreads) expand_emit_kernel(
    const int32_t* __restrict__ mats, const int64_t* __restrict__ coef, const int32_t* __restrict__ job,
    int n, int64_t count, const int* __restrict__ kid_mask, const int64_t* __restrict__ kid_off,
    const int64_t* __restrict__ early_off,
    int32_t* __restrict__ out_mats, int64_t* __restrict__ out_coef, int32_t* __restrict__ out_job,
    int32_t* __restrict__ early_mats, int64_t* __restrict__ early_coef, int32_t* __restrict__ early_job,
    int stage_words, const Plan* __restrict__ plans) {
  const int lane = threadIdx.x & 31;
  const int64_t node = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (node >= count) return;
  const int mask = kid_mask[node];
  const Plan pl = plans[node];
  if (!mask && !pl.early) return;  // no surviving child: nothing to read
  const NodeView A = stage_node(mats + node * (int64_t)n * n, n, stage_words, lane);
  const int64_t cf = coef ? coef[node] : 1;
  const int32_t jb = job ? job[node] : (int32_t)node;
  if (pl.early) {
    const int64_t o = early_off[node];
    write_dense<false>(A, pl.kid[0], early_mats + o * (int64_t)n * n, lane);
    if (lane == 0) {
      early_coef[o] = cf;
      early_job[o] = jb;
    }
    return;
  }
  int64_t o = kid_off[node];
  const int64_t m2 = (int64_t)(n - 1) * (n - 1);
  for (int c = 0; c < pl.nkids; ++c) {
    if ((mask >> c) & 1) {  // survivors found by the count pass
      write_dense<true>(A, pl.kid[c], out_mats + o * m2, lane);
      if (lane == 0) {
        out_coef[o] = pl.kid[c].coef;
        out_job[o] = jb;
      }
      ++o;
    }
  }
}

}  // namespace
}  // namespace sperm

using namespace sperm;

static std::mutex g_exp_mu;
static double g_exp_bytes = 0.0, g_exp_nodes = 0.0;

extern "C" int sperm_expand(const int32_t* d_in_mats, const int64_t* d_in_coef, const int32_t* d_in_job, int n,
                            int64_t count, int32_t* d_out_mats, int64_t* d_out_coef, int32_t* d_out_job,
                            int64_t cap_out, int32_t* d_early_mats, int64_t* d_early_coef, int32_t* d_early_job,
                            int64_t cap_early, int64_t* h_out_count, int64_t* h_early_count, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  keep_pool_memory();
  if (!h_out_count || !h_early_count) return set_error(SPERM_ERR_ARG, "sperm_expand: NULL count outputs");
  *h_out_count = 0;
  *h_early_count = 0;
  if (n < 2 || n > SPERM_EXPAND_NMAX) return set_error(SPERM_ERR_ARG, "sperm_expand: n out of range [2, 128]");
  if (count < 0) return set_error(SPERM_ERR_ARG, "sperm_expand: count < 0");
  if (count == 0) return SPERM_OK;
  if (!d_in_mats) return set_error(SPERM_ERR_ARG, "sperm_expand: d_in_mats is NULL");
  // scratch: kid_count[count] int, early_count[count] int, offsets 2*count int64, err int, totals
  int* kc = nullptr;
  SPERM_CUDA(cudaMallocAsync((void**)&kc, sizeof(int) * (3 * count + 4), st));
  int* ec = kc + count;
  int* km = kc + 2 * count;
  int* err = kc + 3 * count;
  int64_t* off = nullptr;
  SPERM_CUDA(cudaMallocAsync((void**)&off, sizeof(int64_t) * (2 * count + 2), st));
  int64_t* eoff = off + count + 1;
  Plan* plans = nullptr;  // per-node pivot and children, count pass -> emit pass
  SPERM_CUDA(cudaMallocAsync((void**)&plans, sizeof(Plan) * count, st));
  SPERM_CUDA(cudaMemsetAsync(err, 0, sizeof(int) * 4, st));
  // shared-memory staging of each warp's node (row stride n | 1): up to 8 warps per CTA within 200 KB
  const int stage_words = ((n * stage_stride(n) + 3) / 4) * 4;
  const int wpb = std::max(1, std::min(8, (int)((200 * 1024) / (stage_words * 4))));
  const size_t esmem = (size_t)wpb * stage_words * 4;
  SPERM_CUDA(cudaFuncSetAttribute(expand_count_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)esmem));
  SPERM_CUDA(cudaFuncSetAttribute(expand_emit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)esmem));
  const unsigned bthreads = 32u * wpb;
  const unsigned blocks = (unsigned)((count * 32 + bthreads - 1) / bthreads);
  int rc = SPERM_OK;
  auto cleanup = [&]() {
    cudaFreeAsync(kc, st);
    cudaFreeAsync(off, st);
    cudaFreeAsync(plans, st);
  };
  {
    TimingScope ts("expand", st);
    count_launch();
    expand_count_kernel<<<blocks, bthreads, esmem, st>>>(d_in_mats, d_in_coef, n, count, kc, ec, km, err,
                                                         stage_words, plans);
  }
  cudaError_t le = cudaGetLastError();
  if (le != cudaSuccess) { cleanup(); return cuda_check(le, "expand_count_kernel"); }
  // exclusive scans (count+1 entries: the last one is the total)
  SPERM_CUDA(cudaMemsetAsync(off, 0, sizeof(int64_t) * (2 * count + 2), st));
  size_t tmp_bytes = 0, tmp2 = 0;
  cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, kc, off + 1, count, st);
  cub::DeviceScan::InclusiveSum(nullptr, tmp2, ec, eoff + 1, count, st);
  tmp_bytes = std::max(tmp_bytes, tmp2);
  void* tmp = nullptr;
  SPERM_CUDA(cudaMallocAsync(&tmp, tmp_bytes, st));
  cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, kc, off + 1, count, st);
  cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, ec, eoff + 1, count, st);
  cudaFreeAsync(tmp, st);
  int64_t tot[2] = {0, 0};
  int herr = 0;
  SPERM_CUDA(cudaMemcpyAsync(&tot[0], off + count, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  SPERM_CUDA(cudaMemcpyAsync(&tot[1], eoff + count, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  SPERM_CUDA(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, st));
  le = cudaStreamSynchronize(st);
  if (le != cudaSuccess) { cleanup(); return cuda_check(le, "sperm_expand count readback"); }
  *h_out_count = tot[0];
  *h_early_count = tot[1];
  if (herr) { cleanup(); return set_error(SPERM_ERR_RANGE, "sperm_expand: merged entry or coefficient overflow"); }
  if (tot[0] > cap_out || tot[1] > cap_early) {
    cleanup();
    return set_error(SPERM_ERR_CAPACITY, "sperm_expand: output capacity too small");
  }
  if ((tot[0] > 0 && (!d_out_mats || !d_out_coef || !d_out_job)) ||
      (tot[1] > 0 && (!d_early_mats || !d_early_coef || !d_early_job))) {
    cleanup();
    return set_error(SPERM_ERR_ARG, "sperm_expand: NULL output buffer");
  }
  {
    TimingScope ts("expand", st);
    count_launch();
    // the emit pass stages the parent too (read once, then once per child from shared memory;
    // measured on the config-5 fullerene: 1.46 s staged vs 1.73 s reading global memory)
    expand_emit_kernel<<<blocks, bthreads, esmem, st>>>(d_in_mats, d_in_coef, d_in_job, n, count, km, off, eoff,
                                                        d_out_mats, d_out_coef, d_out_job, d_early_mats, d_early_coef,
                                                        d_early_job, stage_words, plans);
  }
  le = cudaGetLastError();
  cleanup();
  if (le != cudaSuccess) return cuda_check(le, "expand_emit_kernel");
  {
    // algorithmic bytes of the level: every parent read once (matrix + coef + job), every
    // child and early node written once
    std::lock_guard<std::mutex> lk(g_exp_mu);
    g_exp_bytes += (double)count * (4.0 * n * n + 12.0) + (double)tot[0] * (4.0 * (n - 1) * (n - 1) + 12.0) +
                   (double)tot[1] * (4.0 * n * n + 12.0);
    g_exp_nodes += (double)count;
  }
  return rc;
}

extern "C" int sperm_expand_stats(double* h_bytes, double* h_nodes, int reset) {
  std::lock_guard<std::mutex> lk(g_exp_mu);
  if (h_bytes) *h_bytes = g_exp_bytes;
  if (h_nodes) *h_nodes = g_exp_nodes;
  if (reset) g_exp_bytes = g_exp_nodes = 0.0;
  return SPERM_OK;
}
