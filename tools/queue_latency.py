"""Claim latency of the box-wide device queue (sperm_queue_*, NEXT-2): rank 0 creates the
counter in its HBM, rank 1 maps it through CUDA IPC (both on this node's GPUs; on a one-GPU pod
both processes share cuda:0), each claims `--claims` chunks of size 1 from its own stream.
Reports microseconds per claim and that every index was claimed exactly once.

    python tools/queue_latency.py --claims 2000
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, world, port, claims, out):
    import time
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import paper_1112_6072_b200 as P
    torch.cuda.set_device(rank % torch.cuda.device_count())
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    store = dist.distributed_c10d._get_default_store()
    if rank == 0:
        q = P.DeviceQueue()
        store.set("q", q.handle)
    else:
        q = P.DeviceQueue(handle=store.get("q"))
    got = [q.claim(1)]  # warm-up claim (counted in the coverage check)
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(claims):
        got.append(q.claim(1))
    dt = time.perf_counter() - t0
    dist.barrier()
    res = [None] * world
    dist.all_gather_object(res, {"rank": rank, "us_per_claim": 1e6 * dt / claims, "got": got})
    if rank != 0:
        q.close()
    dist.barrier()
    if rank == 0:
        q.close()
        allgot = sorted(g for r in res for g in r["got"])
        print(json.dumps({"ranks": world, "claims_per_rank": claims,
                          "us_per_claim": [round(r["us_per_claim"], 2) for r in res],
                          "each_index_once": allgot == list(range(world * (claims + 1))),
                          "devices": torch.cuda.device_count()}), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--claims", type=int, default=2000)
    ap.add_argument("--ranks", type=int, default=2)
    args = ap.parse_args()
    import socket
    import torch.multiprocessing as mp
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    mp.start_processes(worker, args=(args.ranks, port, args.claims, None), nprocs=args.ranks, join=True,
                       start_method="spawn")


if __name__ == "__main__":
    main()
