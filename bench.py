#!/usr/bin/env python
"""Benchmark of the GaloisSAT GPU stage on B200 (contract: see DESIGN.md §Measurement).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C2] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...     (one process per GPU, NCCL)

A "step" is one pass of the whole hot path over the batch: sample, clause forward,
straight-through signal + Adam update + rounding (fused), exact check, best tracking
(and the NCCL MIN all-reduce of the best key when N > 1). Metric: literal-evaluations/s
(L x B x steps / time, one "literal evaluation" = one (slot, member) pair of one step),
whole job over all ranks; weak scaling (B = 4096 per GPU for C2). Prints ONE JSON line
on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "literal-evals/sec"
UNIT = "literal-evals/s"

# per-GPU batch of each workload (BASELINE.json configs)
WORKLOADS = {
    "C1": dict(desc="uniform random 3-SAT n=50 m=213 (ratio 4.26), seed 0", batch=1024),
    "C2": dict(desc="uniform random 3-SAT n=10000 m=42000 (ratio 4.2), seed 0", batch=4096),
    "C3a": dict(desc="random 5-SAT n=2000 m=42000 (ratio 21), seed 0", batch=16384),
    "C3b": dict(desc="random 7-SAT n=500 m=43895 (ratio 87.79), seed 0", batch=16384),
    "C4": dict(desc="industrial-like n=1M m=4.2M widths 2-30 power-law occurrences, seed 0", batch=1024),
    "C5": dict(desc="cube-split random 3-SAT n=100k m=426k, 16 cube pins, seed 0", batch=65536),
}


def make_instance(name):
    from paper_2603_28796_b200 import instances as I
    return I.CONFIGS[name][0]()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(workload):
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu --set full
    summary (profiles/ncu_traffic.json), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f)
    e = d.get(workload, {}).get("update")
    return None if e is None else e.get("dram_bytes_per_launch")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"galois_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def oracle_sample(inst, batch, seconds=12.0, rank_b0=0):
    """The fp64 oracle as it stands, timed on the host cores on a bounded sample of the
    same workload: whole steps of up to 64 members, repeated until `seconds` elapse."""
    from oracle import oracle as O
    f = O.Cnf(inst.n, inst.offsets, inst.lits)
    cfg = O.Config(seed=0)
    nb = min(batch, max(16, 4 * O.num_threads()))
    st = O.State.init(inst.n, rank_b0, nb, 0)
    steps = 0
    t0 = time.perf_counter()
    while True:
        O.step(f, cfg, st)
        steps += 1
        el = time.perf_counter() - t0
        if el >= seconds or steps >= 1000:
            break
    value = inst.L * nb * steps / el
    return {"value": value, "unit": UNIT, "cores": O.num_threads(), "kind": "oracle",
            "sample": f"{nb} members x {steps} steps of the {batch}-member workload "
                      f"(fp64 C oracle, OpenMP over members), {el:.1f} s"}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def run_reference(args):
    """--impl reference: the oracle (the reference arm of this tier), rank 0 only."""
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    inst = make_instance(args.workload)
    per_gpu = WORKLOADS[args.workload]["batch"]
    B = per_gpu * args.gpus
    samples = []
    for i in range(args.warmup + args.steps):
        s = oracle_sample(inst, B, seconds=args.ref_seconds)
        if i >= args.warmup:
            samples.append(s)
    value = statistics.median(s["value"] for s in samples)
    cb = dict(samples[-1])
    cb["value"] = value
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload, "instance": WORKLOADS[args.workload]["desc"],
                       "global_batch": B, "n": inst.n, "m": inst.m, "L": inst.L},
            "cpu_baseline": cb,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="C2", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--tts", default=None, help="only measure time-to-first-SAT on this config's SAT set")
    ap.add_argument("--tts-seeds", type=int, default=10)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    from paper_2603_28796_b200 import galois as G

    rank, world, local = dist_env()
    if world != args.gpus:
        args.gpus = world if world > 1 else args.gpus
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if args.tts:
        print(json.dumps({"time_to_first_sat": time_to_sat(G, torch, dev, args.tts, range(args.tts_seeds))}),
              flush=True)
        return 0
    pg = None
    nccl_id = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        pg = dist
        obj = [G.galois_comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]

    inst = make_instance(args.workload)
    per_gpu = WORKLOADS[args.workload]["batch"]
    B = per_gpu * world
    T = args.warmup + args.steps
    stream = torch.cuda.Stream(dev)          # a real stream (not the legacy default one)
    torch.cuda.set_stream(stream)
    cnf = G.Cnf.from_instance(inst)
    info = cnf.info()
    eng = G.Engine(cnf, B, T, 0.5, 0, cubes=inst.pins, stream=stream.cuda_stream, rank=rank, world=world,
                   nccl_id=nccl_id)
    eng.enqueue(args.warmup)
    torch.cuda.synchronize(dev)
    eng.set_profiling(True)
    eng.kernel_times()                       # reset
    clocks = ClockSampler(local)
    clocks.start()
    if pg:
        pg.barrier()
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    eng.enqueue(args.steps)
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    if pg:
        pg.barrier()
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    kt = eng.kernel_times()
    st = eng.info()
    completed = st["steps_done"] == T and not st["stopped"]
    t_all = torch.tensor([ms], dtype=torch.float64, device=dev)
    if pg:
        pg.all_reduce(t_all, op=pg.ReduceOp.MAX)
    ms_max = float(t_all.item())
    L = info["L"]
    value = L * B * args.steps / (ms_max / 1e3)

    # dominant kernel: the fused update (a6 + a7); algorithmic bytes per launch
    n, W, b_pad = inst.n, (eng.info()["local_batch"] + 31) // 32, ((eng.info()["local_batch"] + 31) // 32) * 32
    upd_ms, upd_n = kt["update"]
    hub = info["num_hubs"] > 0
    bytes_update = (L * W * 4          # read E (CSC order), one bit per member per slot
                    + 24 * n * b_pad   # z, m, v read + write (fp32)
                    + 2 * n * W * 4    # X, R bit rows written
                    + 4 * (2 * n + 1)) # CSC offsets
    fwd_ms, fwd_n = kt["forward"]
    bytes_forward = L * W * 4 * 2 + 8 * L + 4 * (inst.m + 1)
    peak, peak_src = peaks()
    achieved = bytes_update / (upd_ms / upd_n / 1e3) / 1e9 if upd_n else None
    gpu_launches = int(sum(c for _, c in kt.values()))
    total_kernel_ms = sum(t for t, _ in kt.values())

    line = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = oracle_sample(inst, B, seconds=args.ref_seconds)
        e2e = None
        if world == 1 and not args.no_e2e:
            e2e = run_e2e(G, inst, B, args, torch, dev)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32-bits+f32", "data": "synthetic",
            "config": {"workload": args.workload, "instance": WORKLOADS[args.workload]["desc"],
                       "global_batch": B, "batch_per_gpu": per_gpu, "n": n, "m": inst.m, "L": L,
                       "check_interval": 1, "lr": 0.5, "tau": 1.0, "optimizer": "adam",
                       "l2": f"inputs larger than L2 (fp32 state {3 * 4 * n * b_pad / 1e6:.0f} MB per GPU > 126 MB)",
                       "parallelism": f"dp{world} (batch sharding, NCCL MIN all-reduce of the best key per step)"},
            "roofline": {"bound": "hbm", "kernel": "k_update_tma (fused signal reduction + Adam + round + sample)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None,
                         "traffic": ncu_traffic(args.workload), "algorithmic_bytes_per_launch": bytes_update,
                         "peak_source": peak_src,
                         "ms_per_launch": upd_ms / upd_n if upd_n else None,
                         "share_of_kernel_time": upd_ms / total_kernel_ms if total_kernel_ms else None},
            "kernels_ms_per_step": {k: (t / args.steps) for k, (t, c) in kt.items() if c},
            "forward": {"ms_per_launch": fwd_ms / fwd_n if fwd_n else None,
                        "achieved_gbs": bytes_forward / (fwd_ms / fwd_n / 1e3) / 1e9 if fwd_n else None,
                        "algorithmic_bytes_per_launch": bytes_forward},
            "gpu_launches": gpu_launches,
            "clocks": clk,
            "completed_all_steps": completed,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
    eng.free()
    cnf.free()
    if pg:
        pg.barrier()
        pg.destroy_process_group()
    if line is not None:
        print(json.dumps(line), flush=True)
    return 0


def time_to_sat(G, torch, dev, which="C1", seeds=range(10), batch=None, steps=None):
    """Time-to-first-SAT through the public API (galois_engine_run; host wall clock
    bracketed by device syncs; CNF already loaded, engine create + init included),
    per instance: SAT-set instances of the config's shape (C1: G1(50, 213, 3, seed);
    C2: planted G2(10000, 42000, 3, seed); C4: planted G3)."""
    from paper_2603_28796_b200 import instances as I
    make = {"C1": lambda s: I.random_ksat(50, 213, 3, s),
            "C2": lambda s: I.random_ksat(10_000, 42_000, 3, s, planted=True),
            "C3a": lambda s: I.random_ksat(2_000, 42_000, 5, s, planted=True),
            "C4": lambda s: I.industrial(1_000_000, 4_200_000, s, planted=True)}[which]
    B = batch or WORKLOADS[which]["batch"]
    T = steps or (100 if which == "C1" else 200)
    out = []
    for s in seeds:
        inst = make(s)
        cnf = G.Cnf.from_instance(inst)
        for rep in range(2):               # the first repetition warms up
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            eng = G.Engine(cnf, B, T, 0.5, 0)
            rc = eng.run()
            best = eng.best_assignment()
            torch.cuda.synchronize(dev)
            el = time.perf_counter() - t0
            eng.free()
        out.append({"seed": s, "sat": rc == G.SAT, "seconds": el, "step": best["step"], "member": best["global_b"],
                    "best_unsat": best["unsat"]})
        cnf.free()
    solved = [o for o in out if o["sat"]]
    return {"instances": which, "batch": B, "steps_budget": T, "n": len(out), "solved": len(solved),
            "median_seconds_solved": statistics.median(o["seconds"] for o in solved) if solved else None,
            "median_step_solved": statistics.median(o["step"] for o in solved) if solved else None,
            "per_instance": out}


def run_e2e(G, inst, B, args, torch, dev):
    """Same metric end to end through the public C ABI with HOST buffers: CNF upload
    (host -> device), device CSR/CSC build, engine create + init, galois_engine_run of
    the timed steps (host polls the device stop flag), and the results read back
    (unsat counts + best assignment). Host wall clock bracketed by device syncs."""
    import numpy as np
    off = np.ascontiguousarray(inst.offsets, dtype=np.int64)
    lits = np.ascontiguousarray(inst.lits, dtype=np.int32)
    results = []
    for rep in range(2):                       # first pass warms the context / allocator
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        cnf = G.Cnf(inst.n, off, lits)
        eng = G.Engine(cnf, B, args.steps, 0.5, 0, cubes=inst.pins)
        eng.run()
        counts, _ = eng.unsat_counts()
        best = eng.best_assignment()
        torch.cuda.synchronize(dev)
        el = time.perf_counter() - t0
        done = eng.info()["steps_done"]
        eng.free()
        cnf.free()
        results.append((el, done))
    el, done = results[-1]
    h2d = off.nbytes + lits.nbytes + 8 * (args.steps + 2) + 64
    polls = (args.steps + 3) // 4 + 2
    d2h = 64 * polls + 4 * B + inst.n
    return {"value": inst.L * B * done / el, "unit": UNIT, "steps": done,
            "h2d_bytes_per_step": h2d / max(done, 1), "d2h_bytes_per_step": d2h / max(done, 1),
            "wall_s": el, "includes": "cnf upload + CSR/CSC build + create/init + run + read-back"}


if __name__ == "__main__":
    sys.exit(main())
