"""Host orchestration of the hot path (Algorithm PH with the improved Step 3).

    per(A) = PH(A):  pre-expand (Step 2)  -> sperm_expand per level
                     weights   (improved Step 3) -> sperm_estimate (KKLLL)
                     schedule  (LPT over GPUs)  -> sperm_schedule
                     per GPU: expand each job to leaves of order <= L (H_per)
                              and evaluate the leaves by R-NW        -> sperm_expand, sperm_permanent
                     sum       (Step 4): residue accumulators summed over GPUs by
                               one NCCL all-reduce, then host CRT   -> torch.distributed, sperm_crt

This module only sequences C-ABI calls and moves tensors; every arithmetic step of
the method runs inside libsperm.so.  Nodes are kept grouped by order (one dense
[count, n, n] int32 tensor per order), which is how the kernels take them.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

from . import sperm as S


@dataclass
class NodeSet:
    """Nodes of one order n: mats [count,n,n] int32, coef [count] int64, job [count] int32."""
    n: int
    mats: "object"
    coef: "object"
    job: "object"

    @property
    def count(self) -> int:
        return int(self.mats.shape[0])


@dataclass
class PHResult:
    value: int
    job_values: List[int]
    num_jobs: int
    job_order_n: Dict[int, int]
    leaves: int
    terms: float
    estimates: Optional[np.ndarray] = None
    machine: Optional[np.ndarray] = None
    job_cycles: Optional[np.ndarray] = None  # measured SM cycles per job (measure_jobs=True)
    job_sizes: Optional[np.ndarray] = None   # nonzeros per job (the "size" ordering key)
    stats: Dict[str, float] = field(default_factory=dict)


def job_sizes(jobsets: List["NodeSet"], num_jobs: int) -> np.ndarray:
    """Number of nonzero entries of every job (sperm_nnz; the "size" scheduling key)."""
    out = np.zeros(num_jobs, dtype=np.int64)
    for s in jobsets:
        out[s.job.cpu().numpy()] = S.sperm_nnz(s.mats).cpu().numpy()
    return out


def root_nodeset(a, device="cuda") -> NodeSet:
    import torch
    a = np.asarray(a, dtype=np.int64)
    if np.abs(a).max(initial=0) >= 2**31:
        raise ValueError("entries must fit int32")
    n = a.shape[0]
    return NodeSet(n, torch.tensor(a, dtype=torch.int32, device=device).reshape(1, n, n),
                   torch.ones(1, dtype=torch.int64, device=device),
                   torch.zeros(1, dtype=torch.int32, device=device))


def _cat(sets: List[NodeSet]) -> List[NodeSet]:
    """Merge node sets of equal order, keeping their relative order."""
    import torch
    by: Dict[int, List[NodeSet]] = {}
    for s in sets:
        if s.count:
            by.setdefault(s.n, []).append(s)
    out = []
    for n in sorted(by, reverse=True):
        ss = by[n]
        if len(ss) == 1:
            out.append(ss[0])
        else:
            out.append(NodeSet(n, torch.cat([s.mats for s in ss]), torch.cat([s.coef for s in ss]),
                               torch.cat([s.job for s in ss])))
    return out


def pre_expand(root: NodeSet, jobs_at_least: int = 1, job_order: int = 1) -> List[NodeSet]:
    """Algorithm PH Step 2 (reading R6): BFS levels in natural order until the job
    count reaches jobs_at_least or the order reaches job_order.  Returns the job list
    as [level nodes, early (s >= 5) nodes in order of appearance], each NodeSet
    carrying its jobs' global ids (level jobs first, then early jobs)."""
    import torch
    level = root
    early: List[NodeSet] = []
    order = root.n
    while (level.count and level.count + sum(e.count for e in early) < jobs_at_least
           and order > job_order and order >= 2):
        (km, kc, kj), (em, ec, ej) = S.sperm_expand(level.mats, level.coef, level.job)
        if em.shape[0]:
            early.append(NodeSet(order, em, ec, ej))
        level = NodeSet(order - 1, km, kc, kj)
        order -= 1
    jobs = [level] + early
    nid = 0
    out = []
    for s in jobs:
        if s.count == 0:
            continue
        ids = torch.arange(nid, nid + s.count, dtype=torch.int32, device=s.mats.device)
        out.append(NodeSet(s.n, s.mats, s.coef, ids))
        nid += s.count
    return out


def expand_to_leaves(jobs: NodeSet, L: int) -> List[NodeSet]:
    """H_per's recursion applied breadth-first to a batch of jobs until every node has
    order <= L or s >= 5 (readings R5/R6).  Job ids are inherited by the leaves."""
    level = jobs
    early: List[NodeSet] = []
    while level.count and level.n > L and level.n >= 2:
        (km, kc, kj), (em, ec, ej) = S.sperm_expand(level.mats, level.coef, level.job)
        if em.shape[0]:
            early.append(NodeSet(level.n, em, ec, ej))
        level = NodeSet(level.n - 1, km, kc, kj)
    return _cat([level] + early)


# Below the job level only each job's sum matters, so the recursion's levels are expanded
# without the order-preserving scan (sperm_expand_unordered); SPERM_EXPAND_ORDERED=1 keeps it (A-B).
# Nodes of order <= L + SUBTREE_DEPTH (<= 32) are expanded depth first to their leaves in one
# sperm_expand_subtree call (no intermediate level in HBM); SPERM_SUBTREE_DEPTH=0 turns it off.
import os as _os
_LEAF_ORDERED = _os.environ.get("SPERM_EXPAND_ORDERED", "0") == "1"
SUBTREE_DEPTH = int(_os.environ.get("SPERM_SUBTREE_DEPTH", "32"))


def subtree_root_order(L: int, depth: int = None) -> int:
    """Order from which sperm_expand_subtree takes over (0: never): L + depth, at most 32 (one
    lane per line)."""
    depth = SUBTREE_DEPTH if depth is None else depth
    if depth <= 0 or L < 1 or L >= 32:
        return 0
    return min(32, L + depth)


def iter_leaves(jobs: NodeSet, L: int, budget_bytes: int = 16 << 30, stats=None, subtree_depth: int = None):
    """The same H_per recursion as expand_to_leaves, streamed: a level whose children could
    exceed `budget_bytes` of HBM is split into chunks that are expanded to their leaves one
    after another (depth first over chunks), so the live node sets stay bounded however many
    leaves a job has.  Yields NodeSets of leaves (order <= L) and of s >= 5 nodes (those met
    below the subtree order come padded to that order by an identity block, same permanent)."""
    # A level is expanded whole (breadth first: the largest, best-utilised launches) while its own
    # expansion fits the budget.  A level that does not is split into chunks sized so that a
    # chunk's whole subtree down to order L is projected to fit (growth per level = children /
    # parents seen so far at that order, else the largest at any order, else 2; 25% margin), so a
    # chunk normally reaches its leaves without nested splits, which would each keep their parent
    # level alive: the live memory stays ~ the chunked level + one chunk's two current levels.
    # Only the first chunk is cut at a time; the rest is re-split with the growth seen by then.
    # Levels of order <= n0 = subtree_root_order(L) go to sperm_expand_subtree whole (chunked by
    # the leaves per root seen so far, else the 2^(n0-L) worst case); a chunk whose leaves overflow
    # its output is re-run in halves.
    n0 = subtree_root_order(L, subtree_depth)
    seen: Dict[int, List[int]] = {}  # order -> [parents expanded, children produced]
    seen_sub: List[int] = [0, 0]  # subtree roots taken, leaves produced
    leaf_bytes = 4 * L * L + 12

    def g_at(m: int) -> float:
        if m in seen:
            return seen[m][1] / seen[m][0]
        return max(c / p for p, c in seen.values()) if seen else 2.0

    def leaves_per_root() -> float:
        return seen_sub[1] / seen_sub[0] if seen_sub[0] else float(2 ** (n0 - L))

    stack = [jobs]
    while stack:
        level = stack.pop()
        if level.count == 0:
            continue
        if level.n <= L or level.n < 2:
            yield level
            continue
        if n0 and level.n <= n0:
            # depth first below order n0: one call per chunk of roots
            lpr = leaves_per_root()
            cap_roots = max(1, int(budget_bytes // (leaf_bytes * 1.25 * max(lpr, 1.0))))
            if level.count > cap_roots:
                stack.append(NodeSet(level.n, level.mats[cap_roots:], level.coef[cap_roots:], level.job[cap_roots:]))
                stack.append(NodeSet(level.n, level.mats[:cap_roots], level.coef[:cap_roots], level.job[:cap_roots]))
                continue
            cap = max(1, min(int(budget_bytes // leaf_bytes), int(1.25 * lpr * level.count) + 1024))
            if stats is not None:
                import time
                t0 = time.perf_counter()
            r = S.sperm_expand_subtree(level.mats, L, cap, level.coef, level.job)
            if stats is not None:
                stats["subtree_calls"] = stats.get("subtree_calls", 0) + 1
                stats["expand_host_s"] = stats.get("expand_host_s", 0.0) + time.perf_counter() - t0
            if r is None:  # more leaves than projected: halves
                if stats is not None:
                    stats["subtree_retries"] = stats.get("subtree_retries", 0) + 1
                if level.count == 1:
                    raise S.SpermError(S.ERR_CAPACITY, "one node's leaves exceed the leaf budget")
                h = level.count // 2
                stack.append(NodeSet(level.n, level.mats[h:], level.coef[h:], level.job[h:]))
                stack.append(NodeSet(level.n, level.mats[:h], level.coef[:h], level.job[:h]))
                continue
            (lm, lc, lj), (em, ec, ej) = r
            seen_sub[0] += level.count
            seen_sub[1] += lm.shape[0]
            if em.shape[0]:
                yield NodeSet(level.n, em, ec, ej)
            if lm.shape[0]:
                yield NodeSet(L, lm, lc, lj)
            continue
        # bytes per node of one level of order m: its parents (4 m^2 each) and sperm_expand's
        # output slots (2 children of order m-1 and 1 early node of order m per parent)
        per_level = lambda m: 8 * m * m + 8 * (m - 1) ** 2  # noqa: E731
        cap = max(1, budget_bytes // per_level(level.n))
        if level.count > cap:
            peak, mult = 0.0, 1.0
            for m in range(level.n, L, -1):
                if n0 and m <= n0:  # the subtree call: its roots and its leaves
                    peak = max(peak, mult * (4 * m * m + 1.25 * leaves_per_root() * leaf_bytes))
                    break
                peak = max(peak, mult * per_level(m))
                mult *= g_at(m)
                if mult * 8 * L * L > budget_bytes:  # one node's subtree alone exceeds the budget
                    break
            cap = max(1, min(cap, int(budget_bytes // (1.25 * peak))))
        if level.count > cap:
            # the first chunk now; the rest is re-split when popped, with the growth its
            # predecessor's subtree has shown by then
            stack.append(NodeSet(level.n, level.mats[cap:], level.coef[cap:], level.job[cap:]))
            stack.append(NodeSet(level.n, level.mats[:cap], level.coef[:cap], level.job[:cap]))
            continue
        if stats is not None:
            import time
            t0 = time.perf_counter()
        (km, kc, kj), (em, ec, ej) = S.sperm_expand(level.mats, level.coef, level.job, ordered=_LEAF_ORDERED)
        if stats is not None:
            stats["expand_calls"] = stats.get("expand_calls", 0) + 1
            stats["expand_host_s"] = stats.get("expand_host_s", 0.0) + time.perf_counter() - t0
        pc = seen.setdefault(level.n, [0, 0])
        pc[0] += level.count
        pc[1] += km.shape[0]
        if em.shape[0]:
            yield NodeSet(level.n, em, ec, ej)
        stack.append(NodeSet(level.n - 1, km, kc, kj))


def bound_primes(a) -> int:
    """Primes needed to reconstruct per(A): host C (sperm_bound_primes) — the row/column
    abs-sum bound, and Bregman-Minc for 0/1 matrices."""
    return S.sperm_bound_primes(a)


def rank_positions(machine, order, rank: int) -> np.ndarray:
    """Position of every job in this rank's queue (-1 if another rank's): the jobs LPT
    dealt to `rank`, in the order they were dealt (non-increasing estimate, S1)."""
    machine = np.asarray(machine)
    order = np.asarray(order)
    mine = order[machine[order] == rank].astype(np.int64)
    pos = np.full(len(machine), -1, dtype=np.int64)
    pos[mine] = np.arange(len(mine))
    return pos


def estimate_owner(job_ids, world: int):
    """Rank that computes the KKLLL estimate of each job: job id mod world."""
    return job_ids % world


def _allreduce_sum(t, group=None):
    """SUM all-reduce of a CUDA tensor over `group`: in place over NCCL; a gloo group (the CPU
    multi-process tests, or ranks sharing one device) stages it through host memory."""
    import torch.distributed as dist
    if group is None or dist.get_world_size(group) <= 1:
        return t
    if t.is_cuda and dist.get_backend(group) == "gloo":
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def gather_estimates(est_part, group=None):
    """Every rank's estimates from per-rank partial vectors (0.0 at the jobs other ranks own):
    one SUM all-reduce, exact since x + 0.0 = x for the nonnegative estimates."""
    return _allreduce_sum(est_part, group)


def dynamic_chunks(order, chunk: int, claim):
    """The paper's dynamic Step 3 across ranks (each job goes to the
    first free processor, in estimate order): every rank repeatedly claims the next `chunk` jobs
    of the shared order — claim(chunk) returns the first index of a fresh range of the shared
    counter — so a rank that finishes early takes more.  Yields the claimed job ids; over all
    ranks every job is claimed exactly once."""
    order = np.asarray(order)
    while True:
        start = int(claim(chunk))
        if start >= len(order):
            return
        yield order[start:start + chunk]


def store_claimer(store, key: str):
    """claim() through the torch.distributed store's atomic add (a host TCP round trip)."""
    return lambda chunk: int(store.add(key, chunk)) - chunk


class DeviceClaimer:
    """claim() through the box-wide device queue (sperm_queue_*): rank 0 creates the counter in
    its HBM and publishes the IPC handle in the store; the other ranks map it and claim with a
    system-scope atomicAdd over NVLink.  close() unmaps (peers) / frees (owner, after a barrier)."""

    def __init__(self, store, key: str, rank: int, group=None):
        self.group, self.rank = group, rank
        if rank == 0:
            self.q = S.DeviceQueue()
            store.set(key, self.q.handle)
        else:
            self.q = S.DeviceQueue(handle=store.get(key))
        self.claims = 0
        self.claim_s = 0.0

    def __call__(self, chunk: int) -> int:
        import time
        t0 = time.perf_counter()
        v = self.q.claim(chunk)
        self.claim_s += time.perf_counter() - t0
        self.claims += 1
        return v

    def close(self):
        import torch.distributed as dist
        if self.rank != 0:
            self.q.close()
        if self.group is not None and dist.get_world_size(self.group) > 1:
            dist.barrier(group=self.group)  # every peer has unmapped the counter
        if self.rank == 0:
            self.q.close()


_dynamic_calls = 0

# leaves added to the accumulators between folds: each adds < 2^31 to its job row and to the
# total row, so 2^32 leaves keep every uint64 entry below 2^63
FOLD_EVERY = 1 << 32


def allreduce_accumulators(acc, group=None):
    """Algorithm PH Step 4 across GPUs: one SUM all-reduce of the
    [jobs + 1][8] residue accumulators (NCCL on GPUs).  Each rank added residues < 2^31
    per leaf, so the int64 (wrap-around) sum equals the exact uint64 sum."""
    return _allreduce_sum(acc, group)


def reconstruct(res, k: int):
    """Host CRT (sperm_crt) of the reduced accumulators: (job values, total)."""
    return [S.sperm_crt(res[j], k) for j in range(res.shape[0] - 1)], S.sperm_crt(res[-1], k)


def _eval_jobs(jobsets, jobs, L, num_jobs, k_total, nonneg, device, acc):
    """Expand the given job ids to leaves of order <= L and evaluate them (R-NW) into `acc`."""
    import torch
    starts = np.cumsum([0] + [s.count for s in jobsets])
    jobs = np.asarray(jobs)
    which = np.searchsorted(starts, jobs, side="right") - 1
    for si, s in enumerate(jobsets):
        mine = jobs[which == si] - starts[si]
        if not len(mine):
            continue
        idx = torch.tensor(mine, dtype=torch.int64, device=device)
        batch = NodeSet(s.n, s.mats.index_select(0, idx), s.coef.index_select(0, idx), s.job.index_select(0, idx))
        for lv in iter_leaves(batch, L):
            if lv.n > S.NMAX:
                return False
            S.sperm_permanent(lv.mats, coef=lv.coef, job=lv.job, num_jobs=num_jobs, min_primes=k_total,
                              max_primes=k_total if nonneg else 0, job_acc=acc)
    return True


def choose_leaf_order(jobsets, order, num_jobs, k_total, nonneg, device, sample_frac: float = 0.01,
                      start: int = 16, lo: int = 8, hi: int = 32):
    """Reading R5's leaf order L chosen per workload by measurement (NEXT-1): the jobs at evenly
    spaced positions of the estimate order (about `sample_frac` of them, at least 2) are expanded
    to leaves of order <= L and evaluated, timed with CUDA events, for L = start and then one
    step at a time in the direction that got faster (hill climbing) until it stops improving.
    H_per's own rule stops at order 2 and never reaches s >= 5 on 3-regular
    inputs; the balance between the expansion's node count and the R-NW's 2^(L-1)
    terms per leaf is machine-dependent, so it is measured.  Returns (L, {L: seconds})."""
    import torch
    order = np.asarray(order)
    m = max(2, int(round(sample_frac * len(order))))
    pick = order[np.linspace(0, len(order) - 1, num=min(m, len(order))).round().astype(int)]
    scratch = torch.zeros((num_jobs + 1, S.KMAX), dtype=torch.int64, device=device)
    times = {}

    def t_of(L):
        if L not in times:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            ok = _eval_jobs(jobsets, pick, L, num_jobs, k_total, nonneg, device, scratch)
            e1.record()
            torch.cuda.synchronize()
            times[L] = e0.elapsed_time(e1) * 1e-3 if ok else float("inf")
        return times[L]

    L = max(lo, min(hi, start))
    best = t_of(L)
    for step in (-1, 1):
        moved = False
        while lo <= L + step <= hi and t_of(L + step) < best:
            L += step
            best = times[L]
            moved = True
        if moved:
            break
    return L, {str(k): v for k, v in sorted(times.items())}


def permanent(a, jobs_at_least: int = 1, job_order: int = 1, leaf_order=20, trials: int = 0,
              seed: int = 1, policy: str = "estimate", batch_jobs: int = 4096, group=None,
              device="cuda", measure_jobs: bool = False, leaf_budget_bytes: int = None,
              assignment: str = "static", store=None, dynamic_chunk: int = 0,
              fold_every: int = FOLD_EVERY, queue: str = "device") -> PHResult:
    """per(A) by Algorithm PH with the improved Step 3 on one or more GPUs.

    With a torch.distributed `group` of world size G, every rank replicates the
    (cheap, deterministic) pre-expansion and scheduling, estimates its share of the jobs,
    evaluates only the jobs assigned to it, and one all-reduce sums the residue accumulators.
    assignment="static": the LPT plan of sperm_schedule (S1); "dynamic": ranks claim chunks of
    the policy's job order from one shared counter as they finish — the paper's first-free-
    processor rule across GPUs; queue="device": the counter is in rank 0's HBM, claimed with
    system-scope atomics through CUDA IPC (sperm_queue_*; the IPC handle travels through
    `store`, default the process group's store); queue="store": the store's own atomic add.
    leaf_order: L of reading R5, or "auto" (choose_leaf_order: measured on a sample of the jobs).
    policy: "estimate" (KKLLL weights, the improved Step 3), "natural", "random", or "size"
    (the job's nonzero count as the LPT weight).  The uint64 accumulators gain < 2^31 per leaf, so they are folded mod p (sperm_fold_mod)
    before more than `fold_every` leaves have been added since the last fold, and before the
    all-reduce (so the sum over ranks stays below 2^64)."""
    import torch
    import torch.distributed as dist
    rank, world = (dist.get_rank(group), dist.get_world_size(group)) if group is not None else (0, 1)
    if leaf_budget_bytes is None:  # HBM budget of the streamed leaf sets (SPERM_LEAF_BUDGET_GB, default 16)
        leaf_budget_bytes = int(float(_os.environ.get("SPERM_LEAF_BUDGET_GB", "16")) * (1 << 30))
    k_total = bound_primes(a)
    # nonnegative A: every leaf term is >= 0, so each job value and the total lie in
    # [0, per(A)] and k_total primes reconstruct all of them; leaves may be capped at k_total
    nonneg = bool((np.asarray(a) >= 0).all())
    root = root_nodeset(a, device)
    jobsets = pre_expand(root, jobs_at_least, job_order)
    num_jobs = sum(s.count for s in jobsets)
    # improved Step 3: KKLLL weights.  Each rank estimates the jobs it owns (job id mod world);
    # one all-reduce gives every rank every estimate, bit-identical to a replicated run (a job's
    # trials depend only on (seed, job id, trial)).
    est_dev = torch.zeros(num_jobs, dtype=torch.float64, device=device)
    for s in jobsets:
        ids = s.job
        mats = s.mats
        if world > 1:
            idx = torch.nonzero(estimate_owner(ids, world) == rank).flatten()
            ids, mats = ids.index_select(0, idx), mats.index_select(0, idx)
        if ids.shape[0] == 0:
            continue
        if s.n <= 112:
            est_dev[ids.long()] = S.sperm_estimate(mats, trials=trials, seed=seed, ids=ids)
        else:
            est_dev[ids.long()] = float("inf")
    est = gather_estimates(est_dev, group).cpu().numpy()
    sizes = job_sizes(jobsets, num_jobs)
    if policy == "size":  # LPT on the job's nonzero count instead of its estimate
        machine, order, _ = S.sperm_schedule(sizes.astype(np.float64), world, "estimate", seed=seed)
    else:
        machine, order, _ = S.sperm_schedule(est, world, policy, seed=seed)
    acc = torch.zeros((num_jobs + 1, S.KMAX), dtype=torch.int64, device=device)
    job_cycles = torch.zeros(num_jobs, dtype=torch.int64, device=device) if measure_jobs else None
    pos = rank_positions(machine, order, rank)
    if leaf_order == "auto":
        leaf_order, stats_auto = choose_leaf_order(jobsets, order, num_jobs, k_total, nonneg, device)
        if world > 1:  # every rank uses rank 0's choice
            box = [leaf_order]
            dist.broadcast_object_list(box, src=0, group=group)
            leaf_order = int(box[0])
    else:
        stats_auto = None
    leaves = 0
    terms = 0.0
    import time
    stats = {"rnw_calls": 0, "rnw_host_s": 0.0, "leaf_sets": 0, "t_loop_s": 0.0, "leaf_order": leaf_order}
    if stats_auto is not None:
        stats["leaf_order_auto"] = stats_auto
    t_loop = time.perf_counter()
    # Every stage runs on the caller's stream.  SPERM_PIPELINE_OVERLAP=1 puts the R-NW batches on
    # a stream of their own instead, so that the next chunk's expansion could overlap them; the
    # persistent R-NW grids fill every SM, though, and per(C100) at L = 15 measured 45.9 s with
    # the second stream against 33.1 s without (the expansion kernels queue behind the R-NW CTAs
    # while the host waits on their count read-back).
    main = torch.cuda.current_stream()
    import os
    rnw_stream = torch.cuda.Stream() if os.environ.get("SPERM_PIPELINE_OVERLAP", "0") == "1" else main
    acc.record_stream(rnw_stream)
    if measure_jobs:
        job_cycles.record_stream(rnw_stream)
    # the job batches this rank evaluates: (jobset, indices within it), in evaluation order
    def static_batches():
        for s in jobsets:
            ids = s.job.cpu().numpy()
            sel = np.nonzero(pos[ids] >= 0)[0]
            sel = sel[np.argsort(pos[ids[sel]], kind="stable")]
            for b0 in range(0, len(sel), batch_jobs):
                yield s, sel[b0:b0 + batch_jobs]

    claimer = None

    def dynamic_batches():
        nonlocal claimer
        global _dynamic_calls
        _dynamic_calls += 1
        st = store if store is not None else dist.distributed_c10d._get_default_store()
        key = f"sperm_dynamic_{_dynamic_calls}"
        claimer = DeviceClaimer(st, key, rank, group) if queue == "device" else store_claimer(st, key)
        starts = np.cumsum([0] + [s.count for s in jobsets])  # job ids are numbered set by set
        chunk = dynamic_chunk or max(1, num_jobs // (16 * world))
        for jobs in dynamic_chunks(order, chunk, claimer):
            which = np.searchsorted(starts, jobs, side="right") - 1
            for si, s in enumerate(jobsets):
                mine = jobs[which == si] - starts[si]
                if len(mine):
                    yield s, mine

    dynamic = assignment == "dynamic" and (world > 1 or store is not None)
    since_fold = 0
    for s, sel in (dynamic_batches() if dynamic else static_batches()):
        idx = torch.tensor(sel, dtype=torch.int64, device=device)
        batch = NodeSet(s.n, s.mats.index_select(0, idx), s.coef.index_select(0, idx),
                        s.job.index_select(0, idx))
        for lv in iter_leaves(batch, leaf_order, leaf_budget_bytes, stats):
            if lv.n > S.NMAX:
                raise S.SpermError(S.ERR_ARG, f"leaf of order {lv.n} > {S.NMAX} (s >= 5 node)")
            stats["leaf_sets"] += 1
            if since_fold + lv.count > fold_every:  # keep every accumulator below 2^63
                S.sperm_fold_mod(acc, stream=rnw_stream)
                stats["folds"] = stats.get("folds", 0) + 1
                since_fold = 0
            since_fold += lv.count
            t_r = time.perf_counter()
            rnw_stream.wait_stream(main)  # the leaves were written on the main stream
            for t in (lv.mats, lv.coef, lv.job):
                t.record_stream(rnw_stream)  # keep them alive until the R-NW batch is done
            with torch.cuda.stream(rnw_stream):
                cyc = torch.zeros(lv.count, dtype=torch.int64, device=device) if measure_jobs else None
                S.sperm_permanent(lv.mats, coef=lv.coef, job=lv.job, num_jobs=num_jobs, min_primes=k_total,
                                  max_primes=k_total if nonneg else 0, job_acc=acc, leaf_cycles=cyc,
                                  stream=rnw_stream)
                if measure_jobs:  # measured job cost T_i = SM cycles of its leaves
                    job_cycles.index_add_(0, lv.job.long(), cyc)
            stats["rnw_calls"] += 1
            stats["rnw_host_s"] += time.perf_counter() - t_r
            leaves += lv.count
            terms += S.sperm_rnw_terms(lv.n, lv.count)
    if isinstance(claimer, DeviceClaimer):
        stats["claims"], stats["claim_s"] = claimer.claims, claimer.claim_s
        claimer.close()
    if world > 1:
        S.sperm_fold_mod(acc, stream=rnw_stream)  # each rank's rows < 2^31: the G-rank sum fits
    main.wait_stream(rnw_stream)
    stats["t_loop_s"] = time.perf_counter() - t_loop
    allreduce_accumulators(acc, group)
    res = S.sperm_reduce_mod(acc).cpu().numpy().view(np.uint32)
    job_values, value = reconstruct(res, k_total)
    return PHResult(value=value, job_values=job_values, num_jobs=num_jobs,
                    job_order_n={s.n: s.count for s in jobsets}, leaves=leaves, terms=terms,
                    estimates=est, machine=machine,
                    job_cycles=job_cycles.cpu().numpy() if measure_jobs else None,
                    job_sizes=sizes, stats=stats)


def permanental_polynomial(a, device="cuda"):
    """The permanental polynomial P(x) = per(xI - A) = sum_t c_t x^t (Eq. (11)),
    exactly: returns [c_0, ..., c_n] as Python ints.

    The n + 1 values P(x_j), x_j = j - floor(n/2), are evaluated in ONE batched sperm_permanent
    call (R-NW of every x_j I - A) modulo the k primes the coefficients need — sum_t |c_t| <=
    per(I + |A|) (every term of per(xI - A) expands into terms of per(|x| I + |A|) at |x| = 1),
    whose bound sperm_bound_primes gives — then interpolated modulo each prime
    (sperm_interpolate_mod, Newton) and reconstructed by CRT (sperm_crt_batch).  The paper
    evaluates P at the (n+1)-th roots of unity in complex floating point;
    integer points and modular arithmetic make every coefficient exact.  Direct R-NW limits n to
    SPERM_NMAX (48): through the expansion, merged entries of x I - A grow like |x|^depth
    (NEXT-3), so larger graphs are out of this function's reach."""
    import torch
    a = np.asarray(a, dtype=np.int64)
    n = a.shape[0]
    if a.ndim != 2 or a.shape[1] != n:
        raise ValueError("square matrix expected")
    if n > S.NMAX:
        raise ValueError(f"permanental_polynomial: n = {n} > {S.NMAX} (direct R-NW only)")
    if n == 0:
        return [1]
    k = S.sperm_bound_primes(np.abs(a) + np.eye(n, dtype=np.int64))
    xs = np.arange(n + 1, dtype=np.int64) - n // 2
    mats = xs[:, None, None] * np.eye(n, dtype=np.int64)[None] - a[None]
    if np.abs(mats).max() >= 2**31:
        raise ValueError("entries must fit int32")
    res, _ = S.sperm_permanent(torch.tensor(mats, dtype=torch.int32, device=device), min_primes=k, max_primes=k)
    coef = S.sperm_interpolate_mod(res.cpu().numpy().view(np.uint32), xs, k)
    return S.residues_to_ints(coef, k)
