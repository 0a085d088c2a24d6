"""bench.py — R-NW Gray-code throughput of the hot path on BASELINE.json configs[1].

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

Workload (configs[1]): 256 seeded n=24 matrices, each the sum of 3 disjoint random
permutation matrices (half 0/1, half with nonzeros uniform in [1,7]); "direct batched
R-NW, no expansion".  One step = the persistent R-NW kernels over all 256 x 2^23
Gray-code terms in exact multi-prime arithmetic -> residues (then D2H + host CRT of the
256 exact permanents, inside the e2e timing).
Metric: Gray-code terms per second (whole job, all ranks).  With --gpus N > 1 the script
re-launches itself under torch.distributed.run (one process per GPU, NCCL) unless WORLD_SIZE is
already set; each rank evaluates its own seeded batch of 256 (weak scaling, no data-path
collective) for `value`, and the line adds `strong_scaling`: configs[4] (the n = 96 spiral
fullerene and random 3-regular matrix) through pipeline.permanent over the NCCL group — per(A)
wall time on N GPUs (device events, max over ranks) per scheduling policy, against the same
job on rank 0 alone, with the exact per(A) checked against the oracle's golden value.
At N = 1 the line carries `ph` (configs[2], per(C60)), `configs4` (both n = 96 permanents,
1 GPU), `ph_c100` (the paper's C100 case study) and the roofline / cpu_baseline blocks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("R-NW Gray-code terms/s, closed-form-equivalent (2^(n-1) terms per n x n matrix; configs[1]: "
          "256 x n=24 3-regular, exact per(A))")
UNIT = "terms/s"
N_MATS, ORDER, SEED = 256, 24, 2024
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ph", action="store_true", help="skip the whole-path per(C60) measurement")
    ap.add_argument("--ph-leaf", type=int, default=32, help="leaf order L of the per(C60) run")
    ap.add_argument("--no-c100", action="store_true", help="skip the per(C100) run (the paper's case study)")
    ap.add_argument("--no-strong", action="store_true", help="skip the configs[4] runs (strong scaling at N > 1)")
    ap.add_argument("--strong-jobs", type=int, default=160, help="configs[4]: PH jobs (jobs_at_least)")
    ap.add_argument("--strong-leaf", type=int, default=16, help="configs[4]: leaf order L")
    return ap.parse_args()


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled through NVML (pynvml, in-process: no
    nvidia-smi processes competing with the host launch path) every 2 ms of the timed region,
    plus one sample at start and stop; falls back to nvidia-smi if NVML is unavailable."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None
        self.source = "nvml"
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
            self.source = "nvidia-smi"

    def _sample(self):
        if self.nv is not None:
            nv = self.nv
            sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
            bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            self.rows.append((float(sm), float(self.max_mhz),
                              [name for name, attr in self.REASONS if bits & getattr(nv, attr)]))
        else:
            out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                                  "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                                  "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5).stdout
            r = [x.strip() for x in out.strip().split(",")]
            if len(r) >= 6:
                self.rows.append((float(r[0]), float(r[1]), [self.REASONS[i][0] for i in range(4)
                                                             if "Active" in r[2 + i] and "Not" not in r[2 + i]]))

    def start(self):
        self._sample()

        def run():
            while not self._stop.wait(0.002 if self.nv is not None else 0.2):
                try:
                    self._sample()
                except Exception:
                    pass
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        try:
            self._sample()
        except Exception:
            pass
        sm = [r[0] for r in self.rows]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(r[1] for r in self.rows) if sm else None,
                "reasons": sorted({x for r in self.rows for x in r[2]}), "samples": len(self.rows),
                "source": self.source}


def peaks():
    try:
        with open(PEAKS) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def relaunch(args):
    """--gpus N > 1 outside torchrun: start N ranks on this node (torch.distributed.run,
    rendezvous on 127.0.0.1) running this script with the same arguments."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def device_index(local: int) -> int:
    """LOCAL_RANK's GPU.  SPERM_BENCH_SHARE_DEVICE=1 maps every rank to GPU local % count (a
    functional check of the N > 1 path on a one-GPU box with SPERM_BENCH_BACKEND=gloo; its
    timings mean nothing); otherwise one GPU per rank, and too few GPUs is an error."""
    import torch
    cnt = torch.cuda.device_count()
    if os.environ.get("SPERM_BENCH_SHARE_DEVICE") == "1":
        return local % max(cnt, 1)
    if local >= cnt:
        raise RuntimeError(f"rank with LOCAL_RANK={local} but only {cnt} visible GPU(s)")
    return local


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        sys.exit(relaunch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, max(world, args.gpus))
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1112_6072_b200 as P
    from workloads import random_3perm_batch

    didx = device_index(local)
    torch.cuda.set_device(didx)
    dev = torch.device("cuda", didx)
    backend = os.environ.get("SPERM_BENCH_BACKEND", "nccl")
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    # each rank: its own seeded batch (rank 0 is exactly configs[1])
    h_np = random_3perm_batch(N_MATS, ORDER, seed=SEED + rank)
    h_mats = torch.tensor(h_np, dtype=torch.int32).pin_memory()
    d_mats = h_mats.to(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)  # 256 MB > 126 MB L2
    stream = torch.cuda.current_stream()
    jobs = torch.arange(N_MATS, dtype=torch.int32, device=dev)

    def step(mats):
        # configs[1] is the direct batched R-NW (no expansion): one sperm_permanent call
        res, k = P.sperm_permanent(mats, min_primes=1)
        return res, k

    def finish(res, k):
        # exact per(A) of every matrix: CRT on the GPU (sperm_crt_device), one D2H of the
        # [256][limbs + 1] magnitude/sign words, marshalling to Python ints
        return P.residues_to_ints_device(res, k)

    for _ in range(max(args.warmup, 3)):
        vals = finish(*step(d_mats))
    # device-timed region: K steps, L2 flushed before each (outside the events)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    sampler = ClockSampler(didx)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    P.sperm_rnw_stats(reset=True)
    P.sperm_launch_count(reset=True)
    for i in range(args.steps):
        flush.fill_(i)
        ev[i][0].record(stream)
        res, k = step(d_mats)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    st_terms, st_fma, st_alu = P.sperm_rnw_stats(reset=True)
    launches = P.sperm_launch_count(reset=True)
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    vals = finish(res, k)
    # the same K steps again with the library's per-launch CUDA-event timers on (they add host
    # work per launch, so the headline loop above runs without them): the R-NW kernels' device
    # time per step, for the roofline
    P.sperm_timing_enable(True)
    P.sperm_timing_reset()
    evi = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        flush.fill_(i)
        evi[i][0].record(stream)
        step(d_mats)
        evi[i][1].record(stream)
    torch.cuda.synchronize()
    rnw_ms, rnw_launches = P.sperm_timing_get("rnw")
    P.sperm_timing_enable(False)
    instr_ms = sum(a.elapsed_time(b) for a, b in evi)
    # the same K steps with the speculative plan-group launch OFF: it only pays on repeated
    # same-shape batches (this loop); pipeline leaf sets change shape every call
    os.environ["SPERM_SPECULATE"] = "0"
    ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        flush.fill_(i)
        ev2[i][0].record(stream)
        step(d_mats)
        ev2[i][1].record(stream)
    torch.cuda.synchronize()
    os.environ.pop("SPERM_SPECULATE", None)
    clocks = sampler.stop()  # sampled over both loops (same host conditions for the A-B)
    nospec_ms = sum(a.elapsed_time(b) for a, b in ev2)
    # end to end through the public API on HOST buffers: sperm_permanent_host (one C call: H2D of
    # the pinned input batch, R-NW, device CRT, D2H of the exact values) + marshalling to ints
    h_in = h_mats.numpy()
    h_out = torch.empty((N_MATS, P.KMAX + 3), dtype=torch.int32).pin_memory().numpy().view(np.uint32)
    e2e_ms = []
    for i in range(args.steps):
        flush.fill_(i)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        vals = P.sperm_permanent_host(h_in, min_primes=1, out=h_out, stream=stream)
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_total = sum(e2e_ms)
    assert vals == finish(res, k), "host-buffer call disagrees with the device-buffer call"
    if world > 1:
        t = torch.tensor([total_ms, e2e_total, rnw_ms], dtype=torch.float64,
                         device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, e2e_total, rnw_ms = [float(x) for x in t.cpu()]
    terms_step = P.sperm_rnw_terms(ORDER, N_MATS) * world
    value = terms_step * args.steps / (total_ms * 1e-3)
    e2e_value = terms_step * args.steps / (e2e_total * 1e-3)
    # dram read + write bytes of the step's R-NW launches from the committed ncu --set full capture
    # of this build's bench step (tools/ncu_traffic.py -> profiles_bench/rnw_traffic.json; profiles/ does not travel to the GPU box)
    traffic, traffic_note = None, "no ncu capture committed for this build"
    try:
        with open(os.path.join(ROOT, "profiles_bench", "rnw_traffic.json")) as f:
            tj = json.load(f)
        traffic = tj["bytes_per_step"]
        traffic_note = (f"dram__bytes_read.sum + dram__bytes_write.sum of the step's R-NW launches, ncu --set full "
                        f"({tj['source']}, {tj['launches_per_step']} launches per step)")
    except Exception:
        pass
    # roofline of the dominant kernel (rnw_main) on this rank
    pk, pk_kind = peaks()
    sm_mhz = float(pk.get("sm_max_mhz", 1965.0))
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    # integer-pipe roofline: the library's op model of the kernels it ran (sperm_rnw_stats):
    # multiply-pipe units (IMAD 1, IMAD.WIDE/IMAD.HI 2) at 64 / clk / SM and ALU lane-ops at
    # 64 / clk / SM (both measured, tools/microbench); the bound is the busier pipe.
    clk = sm_mhz * 1e6
    t_min = max(st_fma, st_alu) / (64.0 * nsm * clk)
    rnw_s = rnw_ms * 1e-3
    achieved = (st_fma + st_alu) / rnw_s
    peak_ops = (st_fma + st_alu) / t_min if t_min > 0 else 0.0
    rnw_avg_s = rnw_s / max(args.steps, 1)
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int32 (exact mod 2^31 primes)", "data": "synthetic",
        "config": {"workload": "configs[1]: 256 x n=24 sum of 3 disjoint permutation matrices, half 0/1, "
                               "half weights U[1,7], seed 2024(+rank); direct batched R-NW -> residues -> CRT",
                   "matrices_per_gpu": N_MATS, "n": ORDER, "terms_per_step_per_gpu": terms_step / world,
                   "l2": "flushed (256 MB write) before every timed step", "parallelism": f"dp{world} weak"},
        "roofline": {"bound": "alu", "achieved": achieved / 1e9, "peak": peak_ops / 1e9, "unit": "Gop/s",
                     "frac": (achieved / peak_ops) if peak_ops else None,
                     "traffic": traffic, "traffic_note": traffic_note,
                     "kernel": "rnw_tree_kernel / rnw_generic_kernel (all R-NW launches of the step)",
                     "kernel_ms_per_step": rnw_avg_s * 1e3, "launches_per_step": rnw_launches / max(args.steps, 1),
                     "kernel_share_of_step": rnw_ms / instr_ms,
                     "kernel_timing": "library CUDA-event timers on the launching streams, over a second "
                                      "pass of the same K steps (timers on; the headline pass runs without them)",
                     "mul_pipe_units_per_term": st_fma / max(st_terms, 1), "alu_ops_per_term": st_alu / max(st_terms, 1),
                     "terms_per_s_kernel": st_terms / rnw_s if rnw_s else None,
                     "peak_note": f"{nsm} SM x 64 lane-ops/clk per int pipe (mul, alu; measured tools/microbench) "
                                  f"x {sm_mhz:.0f} MHz ({pk_kind} sm_max); bound = busier pipe"},
        "per_A": {"batch_ms_device": total_ms / args.steps, "matrices_per_s": N_MATS * world * args.steps / (total_ms * 1e-3),
                  "batch_ms_e2e": e2e_total / args.steps,
                  "note": "exact per(A) of every matrix of the 256-matrix batch per step (the headline terms/s count "
                          "2^(n-1) equivalent Gray-code terms per matrix; the closed-form block sums evaluate 2^B "
                          "of them per block, DESIGN.md 5.1)"},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h_mats.numel() * 4),
                "d2h_bytes_per_step": int(N_MATS * (P.KMAX + 3) * 4),  # [256][limbs + 1] CRT words
                "api": "sperm_permanent_host (host buffers; H2D + R-NW + device CRT + D2H in one C call)"},
        "without_speculation": {"value": terms_step / world * args.steps / (nospec_ms * 1e-3),
                                "ms_per_step": nospec_ms / args.steps,
                                "note": "same K steps with SPERM_SPECULATE=0 (rank 0): no launch of the previous "
                                        "call's plan groups before the histogram read-back; the speculative launch "
                                        "only pays on repeated same-shape batches like this loop's"},
        "gpu_launches": launches,
        "clocks": clocks,
        "check": {"per_first": str(vals[0]), "per_last": str(vals[-1])},
    }
    if world > 1 and not args.no_strong:
        out["strong_scaling"] = bench_strong(P, torch, dist, rank, world, dev, args.strong_jobs, args.strong_leaf)
    if rank == 0 and world == 1 and not args.no_strong:
        try:
            out["configs4"] = bench_configs4(P, torch, args.strong_jobs, args.strong_leaf)
        except Exception as e:
            out["configs4"] = {"error": repr(e)[:300]}
    if rank == 0 and world == 1 and not args.no_ph:
        out["ph"] = bench_ph(P, torch, leaf_order=args.ph_leaf)
    if rank == 0 and world == 1 and not args.no_ph:
        try:
            out["expand_roofline"] = bench_expand(P, torch)
        except Exception as e:
            out["expand_roofline"] = {"error": repr(e)[:300]}
    if rank == 0 and world == 1 and not args.no_c100:
        try:
            out["ph_c100"] = bench_c100(P, torch)
        except Exception as e:  # reported, never fatal for the main line
            out["ph_c100"] = {"error": repr(e)[:300]}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(h_np)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def configs4_workloads():
    """configs[4]: the seeded n = 96 spiral fullerene (isomer 0) and the n = 96 union of three
    disjoint random permutation matrices (PCG64([2024, 96])), with their oracle golden values."""
    import numpy as np
    from workloads import random_3perm, random_fullerene
    rng = np.random.default_rng(np.random.PCG64([2024, 96]))
    return [("fullerene_n96_seed2024_iso0", random_fullerene(96, 2024, 0)[0]),
            ("random3reg_n96_seed2024_96", random_3perm(96, rng))]


def golden_value(name):
    try:
        for ln in open(os.path.join(ROOT, "tests", "golden", "oracle_values.txt")):
            if ln.startswith(name + " "):
                return int(ln.split()[1])
    except OSError:
        pass
    return None


def _timed_permanent(torch, pipeline, a, **kw):
    """pipeline.permanent between two CUDA events on the current stream (device time of the
    whole call, host gaps included) and a synchronize on both sides."""
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    r = pipeline.permanent(a, **kw)
    e1.record(st)
    torch.cuda.synchronize()
    return r, e0.elapsed_time(e1) * 1e-3


def bench_configs4(P, torch, jobs, leaf):
    """configs[4] on one GPU: per(A) wall time of both n = 96 matrices (estimate-LPT order),
    exact values against the oracle's (tests/golden/oracle_values.txt)."""
    from paper_1112_6072_b200 import pipeline
    out = {}
    for name, a in configs4_workloads():
        r, t = _timed_permanent(torch, pipeline, a, jobs_at_least=jobs, leaf_order=leaf)
        g = golden_value(name)
        out[name] = {"per": str(r.value), "matches_oracle_golden": (r.value == g) if g is not None else None,
                     "wall_s_device": t, "jobs": r.num_jobs, "leaves": r.leaves, "terms": r.terms}
    out["config"] = f"J >= {jobs} PH jobs, leaves of order <= {leaf}, estimate-LPT, 1 GPU"
    return out


def bench_strong(P, torch, dist, rank, world, dev, jobs, leaf):
    """configs[4] strong scaling: each n = 96 matrix through pipeline.permanent on the whole
    group (improved Step 3 across the GPUs, NCCL estimate / residue all-reduces), per policy:
    estimate-LPT static (the paper's contribution, reading S1), estimate dynamic (chunks of the
    estimate order claimed as ranks free up), size-LPT, natural and random order (static).
    T_1 = the same job on rank 0 alone (group=None) while the others wait; T_N = device time of
    the group run, max over ranks; efficiency = T_1 / (N T_N) (Tables 5-7's definition,
    PAPER.md:736-790).  Every group run's per(A) is checked against the golden value."""
    import torch.distributed as dist_
    from paper_1112_6072_b200 import pipeline
    pg = dist_.group.WORLD
    policies = [("estimate", "static"), ("estimate", "dynamic"), ("size", "static"), ("natural", "static"),
                ("random", "static")]
    res = {"config": f"configs[4]: J >= {jobs} PH jobs, leaves of order <= {leaf}; {world} ranks",
           "timing": "device time (CUDA events around the whole call on each rank), max over ranks",
           "workloads": {}}
    from workloads import dodecahedron
    pipeline.permanent(dodecahedron(), jobs_at_least=8, leaf_order=12, group=pg)  # warm-up, all ranks
    for name, a in configs4_workloads():
        g = golden_value(name)
        w = {"golden": str(g) if g is not None else None}
        t1 = torch.zeros(1, dtype=torch.float64, device=dev)
        dist.barrier()
        if rank == 0:
            r1, t = _timed_permanent(torch, pipeline, a, jobs_at_least=jobs, leaf_order=leaf)
            t1[0] = t
            w["per_1gpu"] = str(r1.value)
            w["jobs"] = r1.num_jobs
        dist.barrier()
        pipeline._allreduce_sum(t1, pg)
        w["T1_s"] = float(t1[0])
        for pol, asg in policies:
            dist.barrier()
            r, t = _timed_permanent(torch, pipeline, a, jobs_at_least=jobs, leaf_order=leaf, policy=pol,
                                    group=pg, assignment=asg)
            tt = torch.tensor([t], dtype=torch.float64, device=dev if dist.get_backend(pg) == "nccl" else "cpu")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            tn = float(tt[0])
            w[f"{pol}_{asg}"] = {"TN_s": tn, "efficiency": w["T1_s"] / (world * tn) if tn else None,
                                 "speedup": w["T1_s"] / tn if tn else None, "per": str(r.value),
                                 "exact": (r.value == g) if g is not None else None}
            if asg == "dynamic":  # rank 0's claims on the box-wide device queue (CUDA IPC counter)
                c = r.stats.get("claims", 0)
                w[f"{pol}_{asg}"]["queue"] = {"claims_rank0": c, "us_per_claim": 1e6 * r.stats.get("claim_s", 0.0) / max(c, 1)}
        res["workloads"][name] = w
    return res


def bench_expand(P, torch, jobs_at_least: int = 200000, reps: int = 3):
    """HBM roofline of one Eq. (2) expansion level (sperm_expand: count + scan + emit kernels):
    C100 pre-expanded to >= 2e5 nodes, that level expanded `reps` times (library event timers)."""
    from paper_1112_6072_b200 import pipeline
    from workloads import paper_graph
    s = pipeline.pre_expand(pipeline.root_nodeset(paper_graph("C100")), jobs_at_least=jobs_at_least)[0]
    P.sperm_expand(s.mats, s.coef, s.job)  # warm-up
    torch.cuda.synchronize()
    P.sperm_timing_enable(True)
    P.sperm_timing_reset()
    P.sperm_expand_stats(reset=True)
    for _ in range(reps):
        P.sperm_expand(s.mats, s.coef, s.job)
    torch.cuda.synchronize()
    ms, launches = P.sperm_timing_get("expand")
    nbytes, nodes = P.sperm_expand_stats(reset=True)
    P.sperm_timing_enable(False)
    pk, pk_kind = peaks()
    gbs = nbytes / (ms * 1e-3) / 1e9
    return {"bound": "hbm", "achieved": gbs, "peak": pk.get("hbm_gbs"), "unit": "GB/s",
            "frac": gbs / pk["hbm_gbs"] if pk.get("hbm_gbs") else None, "traffic": None,
            "kernel": "expand_level_kernel (one pass per level)", "level": {"n": s.n, "nodes": s.count},
            "ms_per_level": ms / reps, "algorithmic_bytes_per_level": nbytes / reps,
            "peak_note": f"{pk_kind} MEASURED_PEAKS.json hbm_gbs (copy)"}


def bench_c100(P, torch, leaf_order: int = 15, jobs_at_least: int = 159):
    """per(C100) — the paper's own case study (§4.1): the appendix graph by the whole
    path, checked against Table T12's printed Total (tests/golden/paper_pins.txt).
    The paper: 118413.21 s on one Pentium III (Table 5), 3796.85 s on 32 (Table 6)."""
    from paper_1112_6072_b200 import pipeline
    from workloads import paper_graph
    pin = None
    for ln in open(os.path.join(ROOT, "tests", "golden", "paper_pins.txt")):
        if ln.startswith("per_C100 "):
            pin = int(ln.split()[1])
    P.sperm_timing_enable(True)
    P.sperm_timing_reset()
    P.sperm_rnw_stats(reset=True)
    P.sperm_expand_stats(reset=True)
    P.sperm_expand_subtree_stats(reset=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = pipeline.permanent(paper_graph("C100"), jobs_at_least=jobs_at_least, leaf_order=leaf_order,
                           measure_jobs=True)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    stages = {name: P.sperm_timing_get(name)[0] for name in ("expand", "kklll", "rnw_prep", "rnw", "rnw_finalize")}
    terms = P.sperm_rnw_stats(reset=True)[0]
    lvl_bytes, lvl_nodes = P.sperm_expand_stats(reset=True)
    sub_bytes, sub_roots = P.sperm_expand_subtree_stats(reset=True)
    P.sperm_timing_enable(False)
    # the paper's load-balance study on this run's measured job costs T_i (SM cycles of each job's
    # R-NW leaves): Kendall tau (Eq. 10, Table 3) and Tables 5-7's efficiencies of Step 3 at m
    # processors in natural / exact-time / estimated order (LS replayed with the actual costs)
    import numpy as np
    T = r.job_cycles.astype(np.float64)
    est = r.estimates
    tau_est = P.sperm_kendall_tau(T, est)
    tau_size = P.sperm_kendall_tau(T, r.job_sizes.astype(np.float64))
    orders = {"natural": np.arange(len(T)), "exact": np.argsort(-T, kind="stable"),
              "estimated": np.argsort(-est, kind="stable")}
    eff = {str(m): {k: P.replay_efficiency(T, o, m) for k, o in orders.items()} for m in (8, 16, 32)}
    return {"workload": f"per(C100), PAPER.md appendix graph; J>={jobs_at_least}, leaves of order <= {leaf_order}",
            "per": str(r.value), "paper_table_T12_total": str(pin), "matches_paper": r.value == pin,
            "wall_s": wall, "jobs": r.num_jobs, "leaves": r.leaves, "terms": terms,
            "stage_ms": stages, "stage_note": "device time per stage (library CUDA-event timers, one stream); "
                                              "per-job cycle counters on (measure_jobs); 'expand' = the level "
                                              "kernels down to order 32 + the depth-first subtree kernel below",
            "expansion_bytes": {"level_kernels": lvl_bytes, "level_parents": lvl_nodes, "subtree_kernel": sub_bytes,
                                "subtree_roots": sub_roots,
                                "note": "algorithmic bytes: parents/roots read once, children/leaves written once"},
            "leaves_per_s": r.leaves / (wall if wall else 1.0),
            "kendall_tau_T_estimate": tau_est, "kendall_tau_T_size": tau_size,
            "tau_z_estimate": P.tau_z(tau_est, len(T)),
            "paper_tau_T_AP_table3": 0.4919, "paper_tau_T_P_table3": 0.5334,
            "replay_efficiency": eff,
            "paper_efficiency_32": {"natural": 0.8434, "exact": 0.9746, "estimated": 0.9461},
            "paper_T1_s": 118413.21, "paper_T32_s": 3796.85}


def bench_ph(P, torch, leaf_order: int = 32, jobs_at_least: int = 992):
    """Whole hot path on configs[2] (C60, the truncated icosahedron): PH pre-expansion
    to >= 992 jobs, KKLLL weights, LPT order, expansion of every job to leaves of order
    <= L, batched R-NW, residue sums, CRT.  One warm-up run, one timed run; per-stage
    device times from the library's event timers; exactness checked against the value
    tests/golden/oracle_values.txt holds (written by oracle/ via tools/make_golden.py)."""
    from paper_1112_6072_b200 import pipeline
    from workloads import dodecahedron, truncated_icosahedron
    a = truncated_icosahedron()
    pipeline.permanent(dodecahedron(), jobs_at_least=8, leaf_order=12)  # warm-up (tiny)
    torch.cuda.synchronize()
    P.sperm_timing_enable(True)
    P.sperm_timing_reset()
    P.sperm_rnw_stats(reset=True)
    P.sperm_expand_stats(reset=True)
    t0 = time.perf_counter()
    r = pipeline.permanent(a, jobs_at_least=jobs_at_least, leaf_order=leaf_order)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    stages = {name: P.sperm_timing_get(name)[0] for name in ("expand", "kklll", "rnw_prep", "rnw", "rnw_finalize")}
    terms, fma, alu = P.sperm_rnw_stats(reset=True)
    exp_bytes, exp_nodes = P.sperm_expand_stats(reset=True)
    P.sperm_timing_enable(False)
    pk, pk_kind = peaks()
    exp_gbs = exp_bytes / (stages["expand"] * 1e-3) / 1e9 if stages["expand"] else None
    gold = None
    try:
        for ln in open(os.path.join(ROOT, "tests", "golden", "oracle_values.txt")):
            if ln.startswith("C60_truncated_icosahedron "):
                gold = int(ln.split()[1])
    except OSError:
        pass
    return {"workload": f"configs[2]: per(C60) by PH, J>={jobs_at_least} jobs, leaves of order <= {leaf_order}",
            "per": str(r.value), "matches_oracle_golden": (r.value == gold) if gold is not None else None,
            "wall_s": wall, "jobs": r.num_jobs, "leaves": r.leaves, "terms": terms,
            "terms_per_s_rnw": terms / (stages["rnw"] * 1e-3) if stages["rnw"] else None,
            "stage_ms": stages,
            "expand_roofline": {"bound": "hbm", "achieved": exp_gbs, "peak": pk.get("hbm_gbs"), "unit": "GB/s",
                                "frac": (exp_gbs / pk["hbm_gbs"]) if exp_gbs and pk.get("hbm_gbs") else None,
                                "algorithmic_bytes": exp_bytes, "parents": exp_nodes,
                                "peak_note": f"{pk_kind} MEASURED_PEAKS.json hbm_gbs (copy)"}}


def cpu_baseline(mats, seconds: float = 12.0):
    """The oracle (oracle/ryser_nw.c, exact multi-limb R-NW, 1 thread) on a bounded
    sample of the same workload: whole matrices alternately from the 0/1 and the
    weighted half until ~`seconds` of CPU time."""
    from oracle.cryser import per_ryser_nw_c
    t0 = time.perf_counter()
    done = []
    i = 0
    while time.perf_counter() - t0 < seconds and i < len(mats):
        idx = (i // 2) if i % 2 == 0 else len(mats) // 2 + i // 2
        per_ryser_nw_c(mats[idx])
        done.append(idx)
        i += 1
    dt = time.perf_counter() - t0
    terms = len(done) * 2 ** (mats.shape[1] - 1)
    return {"value": terms / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{len(done)} of the 256 configs[1] matrices (alternating 0/1 / weighted), "
                      f"oracle/ryser_nw.c exact multi-limb R-NW, {dt:.1f} s"}


def run_reference(args, rank, world):
    """Reference arm = the CPU oracle, as it stands, on this arm's config and metric."""
    if rank != 0:
        return
    sys.path.insert(0, ROOT)
    from workloads import random_3perm_batch
    from oracle.cryser import build_oracle_c, per_ryser_nw_c
    build_oracle_c()
    mats = random_3perm_batch(N_MATS, ORDER, seed=SEED)
    per_step = 2  # bounded sample per step: one 0/1 and one weighted matrix (~2 s)
    times = []
    for s in range(max(args.warmup, 3) + args.steps):
        t0 = time.perf_counter()
        for i in range(per_step):
            idx = (s % (N_MATS // 2)) + (N_MATS // 2) * (i % 2)
            per_ryser_nw_c(mats[idx])
        if s >= max(args.warmup, 3):
            times.append(time.perf_counter() - t0)
    tot = sum(times)
    terms = per_step * 2 ** (ORDER - 1) * args.steps
    v = terms / tot
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": tot / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "exact multi-limb int (CPU)", "data": "synthetic",
        "config": {"workload": "configs[1] (same batch, seed 2024); each step a bounded sample of 2 matrices"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"{per_step} matrices per step (one 0/1, one weighted), oracle/ryser_nw.c"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


if __name__ == "__main__":
    main()
