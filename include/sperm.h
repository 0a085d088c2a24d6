/* sperm.h — C ABI of libsperm.so, the B200 (sm_100a) hot path of the
 * parallel hybrid algorithm for exact sparse permanents.
 *
 * Paper: Wang, Liang, Bai, Huo, "A load balancing strategy for parallel
 * computation of sparse permanents" (arXiv 1112.6072), cited as PAPER.md:<line>.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Matrices are square, DENSE, int32, row-major, stored back to back:
 *    mats[m*n*n + i*n + j] = a_ij of matrix m.  All matrices of one call have
 *    the same order n (the BFS levels of Algorithm PH, have
 *    a single order per level).
 *  - Pointers named d_* are DEVICE pointers (cudaMalloc / torch CUDA
 *    tensors); h_* are HOST pointers.  The library never frees caller memory;
 *    internal temporaries are stream-ordered (cudaMallocAsync) and released
 *    before the call returns or in stream order.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Calls are asynchronous with respect to the host unless stated otherwise.
 *  - Return value: SPERM_OK (0) or a negative SPERM_ERR_* code; the message
 *    of the last error on the calling thread is sperm_last_error().
 *  - Exact results are produced as residues modulo the primes of
 *    sperm_prime(): p_0 > p_1 > ... all in (2^30, 2^31).  A value x with
 *    |x| < (p_0 ... p_{k-1}) / 2 is recovered by sperm_crt().
 */
#ifndef SPERM_H_
#define SPERM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPERM_KMAX 8     /* maximal number of CRT primes per value        */
#define SPERM_NMAX 48    /* maximal order of an R-NW leaf (2^47 terms)    */
#define SPERM_EXPAND_NMAX 128 /* maximal order of an expanded node        */

enum {
  SPERM_OK = 0,
  SPERM_ERR_ARG = -1,       /* invalid argument (size, NULL pointer, n > max)   */
  SPERM_ERR_CUDA = -2,      /* a CUDA runtime call or a kernel launch failed    */
  SPERM_ERR_RANGE = -3,     /* entries too large for exact int32 evaluation     */
  SPERM_ERR_CAPACITY = -4,  /* output buffer too small; see the *_needed output */
  SPERM_ERR_PRIMES = -5     /* bound needs more than SPERM_KMAX primes          */
};

/* ---------------------------------------------------------------- utility */
int sperm_version(void);
const char* sperm_last_error(void);

/* The i-th CRT prime (0 <= i < SPERM_KMAX), or 0 if i is out of range. */
uint32_t sperm_prime(int i);

/* Chinese remaindering (host, synchronous).  residues[q] is x mod p_q for
 * q < k.  Writes the unique x with -M/2 < x <= M/2, M = p_0 ... p_{k-1}, as a
 * sign (-1, 0, +1) and a magnitude of `limbs` little-endian uint32 words
 * (limbs >= k+1 suffices).  Garner's algorithm. */
int sperm_crt(const uint32_t* h_residues, int k, uint32_t* h_mag, int limbs, int* h_sign);

/* sperm_crt over `count` rows (host, synchronous): row r has residues
 * h_residues[r*stride .. r*stride + h_k[r]) (h_k NULL: every row uses k_all primes) and
 * writes h_mag[r*limbs .. (r+1)*limbs) and h_sign[r]. */
int sperm_crt_batch(const uint32_t* h_residues, int64_t count, int stride, const int32_t* h_k, int k_all,
                    uint32_t* h_mag, int limbs, int* h_sign);

/* sperm_crt_batch on the device (asynchronous on `stream`): the same Garner CRT per row, one
 * thread per row; d_out[r*(limbs+1) .. r*(limbs+1)+limbs) receives the magnitude's little-endian
 * uint32 limbs and d_out[r*(limbs+1)+limbs] the sign (-1, 0, +1), so one device-to-host copy
 * returns a whole batch.  d_residues [count][stride] uint32, d_k [count] int32 or NULL (k_all
 * primes per row), k + 1 <= limbs <= SPERM_KMAX + 2.  Errors: SPERM_ERR_ARG. */
int sperm_crt_device(const uint32_t* d_residues, int64_t count, int stride, const int32_t* d_k, int k_all,
                     uint32_t* d_out, int limbs, void* stream);

/* Number of CRT primes that reconstruct per(A) of one HOST matrix h_mat [n][n] (host,
 * synchronous): |per(A)| <= min(prod_i sum_j |a_ij|, prod_j sum_i |a_ij|), and for a 0/1
 * matrix the Bregman-Minc bound prod_i (r_i!)^(1/r_i) (rows and columns).  SPERM_ERR_PRIMES
 * if more than SPERM_KMAX primes would be needed. */
int sperm_bound_primes(const int32_t* h_mat, int n, int* h_k);

/* ---------------------------------------------------------------- R-NW */
/* sperm_permanent — batched exact permanents of the leaves of Algorithm
 * H_per ("return by R-NW(A)"), by Ryser's formula with the
 * Nijenhuis-Wilf refinement in binary-reflected Gray-code order (R-NW,
 * PAPER.md:61-65), evaluated in exact arithmetic modulo k primes:
 *
 *   per(A) = (-1)^(n-1) 2^(1-n) sum_{t=0}^{2^(n-1)-1} (-1)^t prod_i w_i(g(t)),
 *   w_i(S) = 2 a_{i,n-1} - sum_j a_ij + 2 sum_{j in S} a_ij,   g(t) = t ^ (t>>1).
 *
 * (Rows and columns may be renumbered first: per(A) is invariant.  The device sums each
 * aligned block of 2^B Gray-code terms in closed form when B low columns have disjoint
 * supports — the same exact sum.)
 *
 *  d_mats     [count][n][n] int32 leaves (device), 0 <= n <= SPERM_NMAX.
 *  d_coef     [count] int64 leaf coefficients (device) or NULL (all 1): the
 *             leaf contributes coef * per(leaf) (the scalars Eq. (2),
 *             PAPER.md:105-112, leaves on its children).
 *  d_order    [count] int32 evaluation order (device) or NULL (natural order):
 *             leaves are grouped by their evaluation plan (one persistent grid
 *             per group, the groups running concurrently, largest work first),
 *             and each group's work queue hands out its leaves in this order
 *             (stable grouping; improved Step 3: the pipeline
 *             expands a rank's jobs in non-increasing-estimate order, so the
 *             natural leaf order already follows it).  Must be a permutation
 *             of 0..count-1.  (Measurement knob SPERM_RNW_SUBKEY=1: batches of
 *             more than 4096 leaves are ordered, inside a group, by prime class
 *             and exact-E mode first and by this order within those; off by
 *             default.)
 *  d_job      [count] int32 job id of each leaf (device) or NULL (every leaf
 *             belongs to job 0, so d_job_acc[0] accumulates the total).
 *  num_jobs   size of d_job_acc's first dimension (>= 1 when d_job_acc is set).
 *  min_primes every leaf uses at least this many primes (so that sums over
 *             leaves can be reconstructed); each leaf also uses as many as
 *             its own bound |coef| * B(leaf) requires, B = the Bregman-Minc bound
 *             prod_i (r_i!)^(1/r_i) for a 0/1 leaf, else min(prod_i sum_j |a_ij|,
 *             prod_j sum_i |a_ij|).  1 <= min_primes <= SPERM_KMAX.
 *  max_primes 0, or a cap (>= min_primes) on the primes per leaf: the caller
 *             asserts that only sums it knows to be small (e.g. the total of a
 *             nonnegative matrix) will be reconstructed, so an individual leaf
 *             above the cap is then known only modulo the capped primes.
 *  d_leaf_res [count][SPERM_KMAX] uint32 out (device) or NULL:
 *             coef * per(leaf) mod p_q for q < d_leaf_k[m], 0 beyond.
 *  d_leaf_k   [count] int32 out (device) or NULL: primes used per leaf.
 *  d_job_acc  [num_jobs + 1][SPERM_KMAX] uint64 in/out (device) or NULL: the
 *             leaf residues (each < 2^31) are ADDED to the accumulator of their
 *             job and to the last row (the total, Algorithm PH Step 4,
 *             PAPER.md:179), so sums over many calls, GPUs (an NCCL sum) and
 *             leaves stay exact below 2^64; reduce mod p_q before sperm_crt.
 *             With d_job NULL only row 0 is used (it is the total).
 *  d_leaf_cycles [count] uint64 in/out (device) or NULL: SM clock cycles the
 *             R-NW kernel spent on each leaf's work items are ADDED here (the
 *             measured job cost T_i of the paper's load-balance study,
 *             PAPER.md:420-423).
 *  stream     cudaStream_t.
 * Errors: SPERM_ERR_ARG (n > SPERM_NMAX, count < 0), SPERM_ERR_RANGE (some
 * row or column abs sum >= 2^30), SPERM_ERR_PRIMES.  RANGE/PRIMES are
 * detected on the device and reported synchronously (the call waits once for
 * the read-back of the bound pass and plan histogram; when the calling thread's
 * previous call had the same device, n, count and prime bounds, the previous
 * plan groups are launched before that wait and run only if the device finds
 * the same histogram — results are identical either way; SPERM_SPECULATE=0
 * turns this off). */
int sperm_permanent(const int32_t* d_mats, int n, int64_t count, const int64_t* d_coef,
                    const int32_t* d_order, const int32_t* d_job, int64_t num_jobs,
                    int min_primes, int max_primes, uint32_t* d_leaf_res, int32_t* d_leaf_k,
                    uint64_t* d_job_acc, uint64_t* d_leaf_cycles, void* stream);

/* sperm_permanent_host — sperm_permanent on HOST buffers, synchronous: copies h_mats
 * [count][n][n] int32 (host; pinned memory makes the copy asynchronous DMA) to the device,
 * evaluates every matrix's exact permanent (R-NW mod the primes its bound needs, at least
 * min_primes), reconstructs it on the device (sperm_crt_device) and copies back h_out
 * [count][limbs + 1] uint32 (host): limbs little-endian magnitude words, then the sign (-1, 0,
 * +1).  limbs >= (primes needed) + 1; limbs = SPERM_KMAX + 2 always suffices.  The public
 * end-to-end call of the batched R-NW (configs[1] in bench.py's e2e figure).  Errors: those of
 * sperm_permanent and sperm_crt_device; SPERM_ERR_ARG for bad sizes / NULL buffers. */
int sperm_permanent_host(const int32_t* h_mats, int n, int64_t count, int min_primes, uint32_t* h_out,
                         int limbs, void* stream);

/* Number of Gray-code terms sperm_permanent evaluates for `count` leaves of
 * order n: count * 2^(n-1) (as double; exact for n <= 53). */
double sperm_rnw_terms(int n, int64_t count);

/* Cumulative work model of the sperm_permanent calls since the last reset (host):
 * Gray-code terms evaluated, multiply-pipe units (IMAD = 1, IMAD.WIDE / IMAD.HI = 2)
 * and ALU-pipe lane-operations of the kernels' formulation, for the
 * roofline.  reset != 0 clears the counters after reading. */
int sperm_rnw_stats(double* h_terms, double* h_fma_units, double* h_alu_ops, int reset);

/* Reduce accumulators mod the primes: out[r][q] = acc[r][q] mod p_q (device). */
int sperm_reduce_mod(const uint64_t* d_acc, int64_t rows, uint32_t* d_out, void* stream);

/* Fold accumulators mod the primes IN PLACE: acc[r][q] := acc[r][q] mod p_q (device,
 * asynchronous on `stream`).  d_job_acc of sperm_permanent gains < 2^31 per leaf and row, so a
 * caller accumulating more than 2^32 leaves (PH Step 4's sum, over a long run) or
 * summing accumulators over GPUs folds them first; the residues mod p_q are unchanged.
 * Errors: SPERM_ERR_ARG (rows < 0, NULL d_acc). */
int sperm_fold_mod(uint64_t* d_acc, int64_t rows, void* stream);

/* ---------------------------------------------------------------- expansion */
/* sperm_expand — one breadth-first level of Algorithm PH Step 2
 * (PAPER.md:161-174): every node (coef, A) of order n is split by Eq. (2)
 * on the line with the minimal number of nonzeros s
 * (Algorithm H_per Step 1), into its children of order n-1:
 *   s = 1: the single child  a * minor(pivot row, p0);
 *   s = 2: A1 = merge of p0,p1: column p0 := a*col(p1) + b*col(p0), column p1
 *          and the pivot row deleted (A2 has a zero column);
 *   s = 3: A1 as above, plus c * minor(pivot row, p2);
 *   s = 4: A1 and A2 = the same merge of p2,p3 with scalars c,d;
 * with p0 < p1 < p2 < p3 the pivot line's nonzero positions and a,b,c,d their
 * values.  Pivot tie-break: rows before columns, lowest index; a column pivot
 * acts on the transpose (reading R2).  Children with a zero row or
 * column are dropped (per = 0).  Nodes with s >= 5 are not split; they are
 * copied unchanged (order n) to the `early` outputs.  Nodes with s = 0 vanish.
 * Children are written in natural order (parents in order, A1 before A2) —
 * stable, so the job list equals the oracle's.
 *
 *  d_in_mats/coef/job  [count] nodes of order n (device).  d_in_job may be
 *                      NULL: the node index is used as its job id.
 *  d_out_mats/coef/job [cap_out] children of order n-1 (device).
 *  d_early_*           [cap_early] unsplit nodes of order n (device; may be
 *                      NULL when cap_early == 0).
 *  h_out_count, h_early_count  host outputs: numbers written (or needed).
 * count < 2^30 per call.  Synchronous w.r.t. the host (the counts are read
 * back).  Returns SPERM_ERR_CAPACITY if a capacity is too small (counts still
 * report the needed sizes), SPERM_ERR_RANGE if a merged entry or coefficient
 * overflows; after either error the output buffers' contents are unspecified. */
int sperm_expand(const int32_t* d_in_mats, const int64_t* d_in_coef, const int32_t* d_in_job,
                 int n, int64_t count,
                 int32_t* d_out_mats, int64_t* d_out_coef, int32_t* d_out_job, int64_t cap_out,
                 int32_t* d_early_mats, int64_t* d_early_coef, int32_t* d_early_job,
                 int64_t cap_early, int64_t* h_out_count, int64_t* h_early_count, void* stream);

/* sperm_expand_unordered — sperm_expand with the children of the level in an UNSPECIFIED order
 * (each tile of nodes takes its output range with one atomic add instead of the order-preserving
 * look-back scan).  Every child, coefficient and job id is the same; only their positions differ
 * from run to run.  For the H_per recursion below the job level, where a job's
 * value is the sum over its leaves and their order does not matter; the PH job list itself
 * (Step 2) uses the ordered sperm_expand.  Same arguments, outputs and errors as sperm_expand. */
int sperm_expand_unordered(const int32_t* d_in_mats, const int64_t* d_in_coef, const int32_t* d_in_job,
                           int n, int64_t count,
                           int32_t* d_out_mats, int64_t* d_out_coef, int32_t* d_out_job, int64_t cap_out,
                           int32_t* d_early_mats, int64_t* d_early_coef, int32_t* d_early_job,
                           int64_t cap_early, int64_t* h_out_count, int64_t* h_early_count, void* stream);

/* sperm_expand_subtree — Algorithm H_per's recursion (Step 1's pivot line and
 * Eq. (2)'s split) applied DEPTH FIRST below the job level: every node of order
 * n is expanded by the same splits as sperm_expand (pivot reading R2, zero-line children dropped
 * per R4, s >= 5 nodes not split per R5) down to its leaves of order leaf_order, in one call — one
 * warp per node walks the node's whole subtree in shared memory, so no intermediate level touches
 * HBM.  The leaves are the same multiset (matrix, coefficient, job id) as repeated
 * sperm_expand_unordered calls produce, in an UNSPECIFIED order: for the H_per recursion below
 * the job level, where a job's value is the sum over its leaves.
 *
 *  d_in_mats/coef/job  [count] nodes of order n, 2 <= n <= 32 (device).  d_in_job may be NULL
 *                      (node index = job id); d_in_coef may be NULL (coefficient 1).
 *  leaf_order          L, 1 <= L < n: the leaves have order exactly L.
 *  d_out_mats/coef/job [cap_out] leaves [L][L] (device).
 *  d_early_*           [cap_early] the s >= 5 nodes met on the way, each padded to order n by an
 *                      identity block: diag(X, I_{n-o}) for a node X of order o (same permanent),
 *                      so all have order n (device; may be NULL when cap_early == 0).
 *  h_out_count, h_early_count  host outputs: numbers written (or needed, see below).
 * Synchronous w.r.t. the host (the counts are read back).  Errors: SPERM_ERR_ARG (sizes, NULL
 * pointers, a stack too large for shared memory: sum_{m=L}^{n-1} m(m+1) + 2 n (n|1) words per
 * warp must fit 56 KB); SPERM_ERR_RANGE (a merged entry or coefficient overflows);
 * SPERM_ERR_CAPACITY: the leaves exceeded cap_out — the kernel stops taking new nodes, so the
 * outputs are incomplete and *h_out_count is only a lower bound (re-run on fewer nodes) — or
 * only the early nodes exceeded cap_early (the leaf outputs and both counts are then exact:
 * re-run with cap_early = *h_early_count). */
int sperm_expand_subtree(const int32_t* d_in_mats, const int64_t* d_in_coef, const int32_t* d_in_job,
                         int n, int64_t count, int leaf_order,
                         int32_t* d_out_mats, int64_t* d_out_coef, int32_t* d_out_job, int64_t cap_out,
                         int32_t* d_early_mats, int64_t* d_early_coef, int32_t* d_early_job,
                         int64_t cap_early, int64_t* h_out_count, int64_t* h_early_count, void* stream);

/* Cumulative algorithmic traffic of the completed sperm_expand_subtree calls since the last reset
 * (host): bytes = every root read once + every leaf / early node written once (matrix,
 * coefficient, job id); roots = nodes taken.  reset != 0 clears the counters after reading. */
int sperm_expand_subtree_stats(double* h_bytes, double* h_roots, int reset);

/* sperm_nnz — number of nonzero entries of each node (device, asynchronous): d_out[m] =
 * |{(i, j) : a_ij != 0}| of matrix m of d_mats [count][n][n].  The "size" scheduling key the
 * load-balance comparison orders jobs by (the paper's alternatives to the estimate order:
 * natural order, and the size regressors of PAPER.md:293-349).  Errors: SPERM_ERR_ARG. */
int sperm_nnz(const int32_t* d_mats, int n, int64_t count, int64_t* d_out, void* stream);

/* Cumulative algorithmic traffic of the completed sperm_expand calls since the last reset
 * (host): bytes = every parent read once + every child / early node written once (matrix,
 * coefficient, job id); nodes = parents processed.  For the HBM roofline of the expansion.
 * reset != 0 clears the counters after reading. */
int sperm_expand_stats(double* h_bytes, double* h_nodes, int reset);

/* ---------------------------------------------------------------- estimator */
/* sperm_estimate — Algorithm KKLLL on the 0/1 pattern of
 * each matrix: B_ij = 0 where a_ij = 0, else an
 * independent uniform cube root of unity; X = det(B) conj(det(B)); the
 * estimate is the mean of `trials` X's (0 -> n^2).  Theorem 1
 * (PAPER.md:218-220): E[X] = per(pattern).  Randomness is the counter-based
 * generator of DESIGN.md reading K1 keyed by (seed, d_ids[m] or m, trial, i, j);
 * det by complex LU with partial pivoting in IEEE fp64 without contraction
 * (reading K2), so estimates are reproducible bit for bit.  Orders >= 48 run a
 * frontal LU (one warp per trial over the rows and columns pivoting can still change; the
 * same operations per entry) and re-run jobs that overflow its front in a CTA-per-trial LU;
 * the call then synchronizes once (the overflow flags are read back).
 *  d_mats    [count][n][n] int32 (device); d_ids [count] int32 or NULL.
 *  d_est     [count] double out (device).
 *  d_trials_out [count][trials] double out (device) or NULL: every X.  */
int sperm_estimate(const int32_t* d_mats, int n, int64_t count, const int32_t* d_ids,
                   int trials, uint64_t seed, double* d_est, double* d_trials_out,
                   void* stream);


/* Jobs that went through sperm_estimate's frontal warp-per-trial kernel (orders >= 48) since the
 * last reset, and how many of them it handed to the CTA kernel (front > 24 rows, window > 64
 * columns, or a row with > 12 nonzeros).  Host; reset != 0 clears the counters after reading. */
int sperm_estimate_stats(double* h_jobs, double* h_redo, int reset);

/* ---------------------------------------------------------------- schedule */
/* sperm_schedule — the improved Step 3 and LPT
 * on the host: jobs are ordered by non-increasing weight
 * (ties: lower job id), then each goes to the currently least-loaded of
 * `machines` machines (ties: lowest machine id).
 *  policy 0 = estimate order (weights as given, LPT),
 *         1 = natural order (list scheduling in index order),
 *         2 = random order (seeded Fisher-Yates with `seed`),
 *  h_weights [count] double (host); h_machine [count] int32 out;
 *  h_order [count] int32 out: the order jobs were dealt in;
 *  h_loads [machines] double out (planned loads, may be NULL). */
int sperm_schedule(const double* h_weights, int64_t count, int machines, int policy,
                   uint64_t seed, int32_t* h_machine, int32_t* h_order, double* h_loads);

/* sperm_list_schedule — Algorithm LS with the jobs' ACTUAL costs: jobs in
 * the order h_order (a permutation of 0..count-1), each to the machine with the least
 * accumulated cost so far (ties: lowest id).  This is Step 3 of Algorithm PH as it runs ("the
 * currently least loaded processor") replayed with measured job times,
 * for the natural / exact-time / estimated orders of Tables 5-7.
 *  h_cost [count] double (host); h_machine [count] int32 out or NULL; h_loads [machines] out.
 * Errors: SPERM_ERR_ARG. */
int sperm_list_schedule(const double* h_cost, const int32_t* h_order, int64_t count, int machines,
                        int32_t* h_machine, double* h_loads);

/* sperm_interpolate_mod — the polynomial P of degree < npts through the points (x_j, v_j),
 * modulo each of the first k CRT primes (host, synchronous): h_values [npts][stride] uint32 with
 * v_j mod p_q at column q < k (e.g. the residue rows of sperm_permanent), h_x [npts] distinct
 * integer points, h_coef [npts][coef_stride] out: coefficient of x^t mod p_q at row t, column q.
 * Newton divided differences mod p.  With the values of per(xI - A) at n + 1 points this gives
 * the permanental polynomial's coefficients (Eq. (11)) modulo the primes;
 * sperm_crt_batch then recovers them exactly when prod p_q > 2 max |coefficient|.
 * Errors: SPERM_ERR_ARG (bad sizes, points not distinct mod some p_q). */
int sperm_interpolate_mod(const uint32_t* h_values, int stride, const int64_t* h_x, int npts, int k,
                          uint32_t* h_coef, int coef_stride);

/* ---------------------------------------------------------------- box-wide queue */
/* A dynamic work queue shared by the GPUs of one node: the improved Step 3's "currently least
 * loaded processor" across GPUs — every rank claims the next chunk of
 * the shared (estimate) job order when it runs out of work.  The counter lives in rank 0's device
 * memory; peers map it through CUDA IPC and claim with a system-scope atomicAdd over
 * NVLink / NVSwitch.
 *  sperm_queue_create  (rank 0) allocates a zeroed uint64 counter on the current device; writes
 *                      its IPC handle (SPERM_QUEUE_HANDLE_BYTES bytes) to h_handle, which the
 *                      caller sends to the peers (e.g. through the process group's store).
 *  sperm_queue_open    (peers) maps the counter from the handle (another process; same or
 *                      another device of the node).
 *  sperm_queue_claim   start = atomicAdd(counter, chunk) (a one-thread kernel on `stream`),
 *                      through the caller's 8-byte DEVICE scratch d_scratch (on the current
 *                      device); synchronous: *h_start receives the claimed range's first index.
 *  sperm_queue_close   owner != 0: frees the counter (after every peer closed it); else unmaps.
 * Errors: SPERM_ERR_ARG, SPERM_ERR_CUDA. */
#define SPERM_QUEUE_HANDLE_BYTES 64
int sperm_queue_create(void** d_counter, void* h_handle);
int sperm_queue_open(const void* h_handle, void** d_counter);
int sperm_queue_claim(void* d_counter, int64_t chunk, void* d_scratch, int64_t* h_start, void* stream);
int sperm_queue_close(void* d_counter, int owner);

/* ---------------------------------------------------------------- statistics */
/* sperm_kendall_tau — Kendall's rank correlation of (x_i, y_i), i < m, with the tie correction
 * of Eq. (10) (Eqs. (7)-(9)): S = sum_{i<j} sign(x_j - x_i) sign(y_j - y_i),
 * T / U = pairs tied in x / in y, tau = S / (sqrt(m(m-1)/2 - T) sqrt(m(m-1)/2 - U)); NaN if a
 * ranking is constant.  The paper's measure of how well a key (estimate, permanent, size)
 * ranks the measured job times (Tables 2-4).  Host, synchronous, O(m log m).
 *  h_x, h_y  [m] double (host); h_tau out; h_counts [4] int64 out or NULL: S, T, U, m(m-1)/2.
 * Errors: SPERM_ERR_ARG (m < 0, NULL, NaN input). */
int sperm_kendall_tau(const double* h_x, const double* h_y, int64_t m, double* h_tau, int64_t* h_counts);

/* ---------------------------------------------------------------- timing */
/* Number of libsperm kernels launched (its own kernels; CUB scans/sorts it calls are not
 * counted) since the last reset; reset != 0 clears the counter after reading. */
int64_t sperm_launch_count(int reset);

/* Device-side kernel timing: when enabled, the library records CUDA events
 * around each launch of its kernels (on the launching stream).
 * sperm_timing_get synchronizes those events and returns the summed
 * milliseconds and launch count of kernel `name` ("rnw", "expand",
 * "kklll", "rnw_prep", "rnw_finalize") since the last reset. */
void sperm_timing_enable(int on);
void sperm_timing_reset(void);
int sperm_timing_get(const char* name, double* h_ms, int64_t* h_launches);

#ifdef __cplusplus
}
#endif
#endif /* SPERM_H_ */
