"""One configs[1] bench step (sperm_permanent over the 256 x n=24 batch) bracketed by
cudaProfilerStart/Stop, after warm-up steps: for `ncu --profile-from-start off --set full`
captures of exactly the step's kernels (tools/ncu_traffic.py sums their DRAM bytes).

    ncu --set full --profile-from-start off -o gpurun_out/step python tools/rnw_step_probe.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_1112_6072_b200 as P
    from workloads import random_3perm_batch
    d = torch.tensor(random_3perm_batch(256, 24, seed=2024), dtype=torch.int32, device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
    for _ in range(4):
        P.sperm_permanent(d, min_primes=1)
    flush.fill_(1)  # the bench flushes L2 before every timed step
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    P.sperm_permanent(d, min_primes=1)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("step done")


if __name__ == "__main__":
    main()
