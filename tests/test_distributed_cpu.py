"""Multi-rank host logic of the hot path on CPU (-m "not gpu"): world_size 2 over gloo.

Each rank estimates the jobs it owns (pipeline.estimate_owner) and one all-reduce gives all
ranks every estimate (pipeline.gather_estimates); each rank replicates the LPT schedule (host
C++, sperm_schedule), takes the jobs dealt to it (pipeline.rank_positions), adds its jobs' residues to the [jobs + 1][8] accumulators,
and one all-reduce (pipeline.allreduce_accumulators — NCCL on GPUs, gloo here) forms
Algorithm PH Step 4; host CRT (pipeline.reconstruct) must give the exact total and every
job value.  The per-job values come from the oracle (test infrastructure) in place of the
GPU R-NW, so the test isolates the distributed logic."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1112_6072_b200 as P
from paper_1112_6072_b200 import pipeline


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, policy, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.hybrid import node_permanent, pre_expand, to_dense
        from oracle.kklll import kklll_estimate
        from workloads import dodecahedron
        a = dodecahedron()
        jobs = pre_expand(a, jobs_at_least=30)
        J = len(jobs)
        vals = [node_permanent(j) for j in jobs]
        est_all = [kklll_estimate((np.array(to_dense(m, k)) != 0).astype(int), 16, 7, i)
                   for i, (c, m, k) in enumerate(jobs)]
        # sharded estimation: this rank fills only the jobs it owns, one all-reduce combines
        owner = pipeline.estimate_owner(torch.arange(J), world)
        part = torch.zeros(J, dtype=torch.float64)
        for i in range(J):
            if int(owner[i]) == rank:
                part[i] = est_all[i]
        est = pipeline.gather_estimates(part, dist.group.WORLD).numpy()
        est_ok = est.tolist() == est_all  # bit-identical to the replicated estimates
        machine, order, _ = P.sperm_schedule(est, world, policy, seed=5)
        pos = pipeline.rank_positions(machine, order, rank)
        k = P.sperm_bound_primes(a)
        acc = torch.zeros((J + 1, P.KMAX), dtype=torch.int64)
        for j in range(J):
            if pos[j] >= 0:
                for qq in range(k):
                    r = vals[j] % P.sperm_prime(qq)
                    acc[j, qq] += r
                    acc[J, qq] += r
        pipeline.allreduce_accumulators(acc, dist.group.WORLD)
        red = np.zeros((J + 1, P.KMAX), dtype=np.uint32)
        for qq in range(k):
            red[:, qq] = (acc[:, qq].numpy() % P.sperm_prime(qq)).astype(np.uint32)
        job_values, total = pipeline.reconstruct(red, k)
        owned = torch.tensor((pos >= 0).astype(np.int64))
        dist.all_reduce(owned)
        sched = torch.tensor(np.asarray(machine, dtype=np.int64))
        gathered = [torch.zeros_like(sched) for _ in range(world)]
        dist.all_gather(gathered, sched)
        q.put((rank, total, job_values == vals and est_ok, bool((owned == 1).all()),
               all(torch.equal(g, gathered[0]) for g in gathered)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("policy", ["estimate", "natural", "random"])
def test_two_rank_partition_and_residue_allreduce(policy):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, policy, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, total, jobs_ok, owned_once, same_sched in out:
        assert total == 1392  # per(C20) (tests/golden/oracle_values.txt)
        assert jobs_ok and owned_once and same_sched


def _dyn_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import time
        from oracle.hybrid import node_permanent, pre_expand
        from workloads import dodecahedron
        jobs = pre_expand(dodecahedron(), jobs_at_least=60)
        J = len(jobs)
        vals = [node_permanent(j) for j in jobs]
        order = np.argsort(-np.array([abs(v) for v in vals]), kind="stable")  # any shared order
        store = dist.distributed_c10d._get_default_store()
        mine = []
        for chunk in pipeline.dynamic_chunks(order, 3, pipeline.store_claimer(store, "test_dynamic")):
            mine.extend(int(j) for j in chunk)
            time.sleep(0.002 * (rank + 1))  # ranks of different speed: the faster claims more
        k = P.sperm_bound_primes(dodecahedron())
        acc = torch.zeros((J + 1, P.KMAX), dtype=torch.int64)
        for j in mine:
            for qq in range(k):
                r = vals[j] % P.sperm_prime(qq)
                acc[j, qq] += r
                acc[J, qq] += r
        pipeline.allreduce_accumulators(acc, dist.group.WORLD)
        red = np.zeros((J + 1, P.KMAX), dtype=np.uint32)
        for qq in range(k):
            red[:, qq] = (acc[:, qq].numpy() % P.sperm_prime(qq)).astype(np.uint32)
        job_values, total = pipeline.reconstruct(red, k)
        claimed = [None] * world
        dist.all_gather_object(claimed, mine)
        q.put((rank, total, job_values == vals, sorted(sum(claimed, [])) == list(range(J)), len(mine)))
    finally:
        dist.destroy_process_group()


def test_two_rank_dynamic_assignment():
    """pipeline.dynamic_chunks over the process group's store: every job claimed by exactly one
    rank (the faster rank claims more), and the residue all-reduce still gives per(C20)."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dyn_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, total, jobs_ok, all_once, n_mine in out:
        assert total == 1392 and jobs_ok and all_once and n_mine > 0
