/* Row-frontier dynamic programme for per(A) in plain C — TEST INFRASTRUCTURE ONLY.
 *
 * The same algorithm as oracle/frontier.py (not a method of the paper; an independent exact
 * algorithm used to pin per(A) of the workloads the Python version is too slow for, e.g.
 * the configs[4] n = 96 matrices of BASELINE.json).  Called through oracle/cfrontier.py.
 *
 * per(A) = sum over perfect matchings rows -> columns (Eq. (1)).  Rows are
 * processed in the given order; a state is the set of columns already used that some later
 * row can still reach ("open"), with the signed sum of the partial products leading to it.
 * A column whose last nonzero row has just been processed must be used by then, otherwise
 * the partial assignment can never be completed: such states are discarded and the column's
 * bit is cleared from the survivors.
 *
 * States are kept as a sorted array (key = 128-bit column mask, value = signed 128-bit sum):
 * each row generates every child (state, nonzero column not yet used), the children are
 * sorted by key and equal keys merged.  No hashing, no blocking: slow but obvious.
 *
 * Exactness: every product and sum is checked for signed 128-bit overflow
 * (__builtin_mul_overflow / __builtin_add_overflow); an overflow is an error, never a wrap.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef __int128 i128;
typedef struct {
    uint64_t lo, hi;
    i128 val;
} state_t;

static int cmp_state(const void *x, const void *y) {
    const state_t *a = (const state_t *)x, *b = (const state_t *)y;
    if (a->hi != b->hi) return a->hi < b->hi ? -1 : 1;
    if (a->lo != b->lo) return a->lo < b->lo ? -1 : 1;
    return 0;
}

static int has_bit(const state_t *s, int j) {
    return j < 64 ? (int)((s->lo >> j) & 1u) : (int)((s->hi >> (j - 64)) & 1u);
}
static void set_bit(state_t *s, int j) {
    if (j < 64) s->lo |= (uint64_t)1 << j; else s->hi |= (uint64_t)1 << (j - 64);
}
static void clear_bit(state_t *s, int j) {
    if (j < 64) s->lo &= ~((uint64_t)1 << j); else s->hi &= ~((uint64_t)1 << (j - 64));
}

/* per(A) for an n x n int64 matrix (row-major), rows processed in `order` (a permutation of
 * 0..n-1).  Writes the value as two's-complement 128 bits into out[0] (low) / out[1] (high)
 * and the largest state count seen into *max_states.
 * Returns 0 on success, -1 bad arguments, -2 signed 128-bit overflow, -3 out of memory. */
int frontier_per(int n, const int64_t *a, const int *order, uint64_t out[2], uint64_t *max_states) {
    if (n < 0 || n > 128) return -1;
    if (n == 0) { out[0] = 1; out[1] = 0; *max_states = 1; return 0; }
    /* last step at which each column has a nonzero */
    int last[128];
    for (int j = 0; j < n; ++j) last[j] = -1;
    for (int step = 0; step < n; ++step) {
        int i = order[step];
        if (i < 0 || i >= n) return -1;
        for (int j = 0; j < n; ++j)
            if (a[(size_t)i * n + j] != 0) last[j] = step;
    }
    for (int j = 0; j < n; ++j)
        if (last[j] < 0) { out[0] = out[1] = 0; *max_states = 0; return 0; }

    size_t cap = 1024, count = 1;
    state_t *cur = (state_t *)malloc(cap * sizeof(state_t));
    if (!cur) return -3;
    cur[0].lo = cur[0].hi = 0;
    cur[0].val = 1;
    uint64_t maxs = 1;
    for (int step = 0; step < n && count > 0; ++step) {
        int i = order[step];
        int nzj[128];
        int64_t nzx[128];
        int nnz = 0;
        for (int j = 0; j < n; ++j)
            if (a[(size_t)i * n + j] != 0) { nzj[nnz] = j; nzx[nnz] = a[(size_t)i * n + j]; ++nnz; }
        size_t ncap = count * (size_t)nnz + 1;
        state_t *nxt = (state_t *)malloc(ncap * sizeof(state_t));
        if (!nxt) { free(cur); return -3; }
        size_t m = 0;
        for (size_t s = 0; s < count; ++s) {
            for (int t = 0; t < nnz; ++t) {
                if (has_bit(&cur[s], nzj[t])) continue;
                nxt[m] = cur[s];
                set_bit(&nxt[m], nzj[t]);
                if (__builtin_mul_overflow(cur[s].val, (i128)nzx[t], &nxt[m].val)) {
                    free(cur); free(nxt); return -2;
                }
                ++m;
            }
        }
        free(cur);
        /* close the columns whose last row is this one: keep states that used them */
        size_t w = 0;
        for (size_t s = 0; s < m; ++s) {
            int ok = 1;
            for (int j = 0; j < n && ok; ++j)
                if (last[j] == step && !has_bit(&nxt[s], j)) ok = 0;
            if (!ok) continue;
            for (int j = 0; j < n; ++j)
                if (last[j] == step) clear_bit(&nxt[s], j);
            nxt[w++] = nxt[s];
        }
        qsort(nxt, w, sizeof(state_t), cmp_state);
        size_t u = 0;
        for (size_t s = 0; s < w; ++s) {
            if (u > 0 && nxt[u - 1].lo == nxt[s].lo && nxt[u - 1].hi == nxt[s].hi) {
                if (__builtin_add_overflow(nxt[u - 1].val, nxt[s].val, &nxt[u - 1].val)) {
                    free(nxt); return -2;
                }
            } else
                nxt[u++] = nxt[s];
        }
        cur = nxt;
        count = u;
        if (count > maxs) maxs = count;
    }
    i128 total = 0;
    for (size_t s = 0; s < count; ++s)
        if (__builtin_add_overflow(total, cur[s].val, &total)) { free(cur); return -2; }
    free(cur);
    out[0] = (uint64_t)total;
    out[1] = (uint64_t)((unsigned __int128)total >> 64);
    *max_states = maxs;
    return 0;
}
