#!/usr/bin/env python3
"""Benchmark of the per-record FFT hot path (arXiv 1407.6915) on B200.

Default workload (N=1): BASELINE.json configs[1] — a 4 GiB in-HBM batch of
8192 records x 65536-point complex64, forward transform.  A "step" is one
fft_exec over the whole batch (every §8(a) kernel row the plan runs).
Multi-GPU (torchrun, one process per GPU): every rank transforms its own
4 GiB batch (records are independent: no collective on the data path,
"scaling": "weak"); the step time is the max over ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 1|2|3|5]

Prints ONE JSON line on rank 0.
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

L2_BYTES = 126 * 2 ** 20

CONFIGS = {
    1: dict(n=1024, batch=16, name="config1: 16 x 1024-pt complex64 forward (latency case)"),
    2: dict(n=65536, batch=8192, name="config2: 4 GiB in-HBM batch of 8192 x 65536-pt complex64, forward"),
    3: dict(n=1 << 20, batch=2048, name="config3: 16 GiB batch of 2048 x 2^20-pt complex64, forward (four-step)"),
}


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy_ read+write)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.rows = []
        self.proc = None
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.t:
            self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                mx.append(float(r[2]))
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def ncu_traffic(kernel_substr, n, batch):
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu
    summary (profiles/ncu_summary.json), if it matches this workload."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None, None
    with open(p) as f:
        d = json.load(f)
    for k in d.get("kernels", []):
        if kernel_substr in k.get("name", "") and k.get("n") == n and k.get("batch") == batch:
            return k.get("dram_bytes_per_launch"), k.get("source")
    # same kernel and N captured at another batch: per-record DRAM bytes scale with the batch
    for k in d.get("kernels", []):
        if kernel_substr in k.get("name", "") and k.get("n") == n and k.get("batch"):
            per = k["dram_bytes_per_launch"] / k["batch"]
            return per * batch, f"{k.get('source')} (captured at batch {k['batch']}, scaled per record)"
    return None, None


# ------------------------------------------------------------------ oracle arm
def host_cores():
    """Host cores available to this process (torchrun sets OMP_NUM_THREADS=1
    per rank, so the OpenMP default is not the machine)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def oracle_rate(n, seconds=10.0, threads=0, min_records=None):
    """Time the CPU oracle (as it stands) on a bounded sample of records of
    length n, all host cores; returns (records/s, cores, sample description)."""
    import oracle
    import synth
    cores = host_cores() if threads <= 0 else threads
    per = max(cores, 1) if min_records is None else min_records
    x = synth.random_records(synth.DEFAULT_SEED, n, 0, per)
    done, t0 = 0, time.perf_counter()
    while True:
        oracle.records_c64(x, oracle.FORWARD, "fft", cores)
        done += per
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return done / el, cores, f"{done} records of {n} points (recursive radix-2, fp64), {el:.1f} s, {cores} threads"


def run_reference(args, cfg):
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    n = cfg["n"]
    import oracle
    cores = host_cores()
    steps = []
    per_step = max(cores, 8)
    import synth
    x = synth.random_records(synth.DEFAULT_SEED, n, 0, per_step)
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        oracle.records_c64(x, oracle.FORWARD, "fft", cores)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            steps.append(dt)
    tot = sum(steps)
    rate = per_step * len(steps) / tot
    out = {
        "impl": "reference", "metric": "records_per_s", "value": rate, "unit": "records/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / len(steps), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded SplitMix64, uniform [-1,1))",
        "config": {"workload": cfg["name"], "n": n, "records_per_step": per_step,
                   "sample": "each step = a bounded sample of the workload's records"},
        "cpu_baseline": {"value": rate, "unit": "records/s", "cores": cores, "kind": "oracle",
                         "sample": f"{per_step} records x {len(steps)} steps of {n} points"},
        "e2e": {"value": rate, "unit": "records/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3])
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist

    import paper_1407_6915_b200 as bf
    from paper_1407_6915_b200 import dist as bd
    from synth import gpu as sg
    import synth

    ri = bd.rank_info()
    world, rank, local = ri.world, ri.rank, ri.local_rank
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    n, batch = cfg["n"], cfg["batch"]
    if args.config == 3 and world > 1:       # strong scaling of the 16 GiB batch
        first, batch = bf.partition(cfg["batch"], world, rank)
        scaling = "strong"
    else:
        first = rank * batch                  # each rank its own records
        scaling = "weak"
    x = torch.empty((batch, n), dtype=torch.complex64, device=dev)
    sg.fill_random(x, synth.DEFAULT_SEED, first_sample=first * n)
    y = torch.empty_like(x)
    plan = bf.Plan(n, batch, bf.FFT_FORWARD, args.variant)
    info = plan.info()
    stream = torch.cuda.current_stream()

    for _ in range(args.warmup):
        plan.exec(x, y)
    torch.cuda.synchronize()
    bd.barrier(dev)
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    t_begin = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_begin.record(stream)
    for i in range(args.steps):
        starts[i].record(stream)
        plan.exec(x, y)                      # one kernel launch on this stream
        ends[i].record(stream)
    t_end.record(stream)
    torch.cuda.synchronize()
    bd.barrier(dev)
    torch.cuda.synchronize()
    clk = clocks.stop()
    total_ms = t_begin.elapsed_time(t_end)
    launch_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    max_ms = bd.max_over_ranks(total_ms, dev)
    recs_total = batch * world if scaling == "weak" else cfg["batch"]
    ms_per_step = max_ms / args.steps
    value = recs_total * args.steps / (max_ms * 1e-3)

    # roofline of the dominant kernel: algorithmic bytes 16 N per record
    peak, peak_src = load_peaks()
    alg_bytes = 16.0 * n * batch
    avg_launch_s = statistics.mean(launch_ms) * 1e-3
    kernels_per_exec = info["kernels_per_exec"]
    achieved = alg_bytes / avg_launch_s / 1e9
    kname = {"cluster": "k_cluster", "single": "k_rows", "fourstep": "k_fs", "identity": "k_copy",
             "pipe": "k_pipe2"}[info["variant_name"]]   # the default pipelined kernel (impl 2)
    traffic, traffic_src = ncu_traffic(kname, n, batch)

    # end to end through the public C ABI (fft_exec_host) with HOST buffers:
    # pinned on the GPU's NUMA node (fft_host_alloc), H2D and D2H of every step
    # inside the timed region; compared with the host link measured here
    # (fft_link_probe: H2D and D2H at once, same buffers)
    e2e = None
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else min(args.steps, 5)
    del x
    torch.cuda.empty_cache()
    if e2e_steps > 0:
        h_in = bf.HostBuffer(batch, n, local)
        h_out = bf.HostBuffer(batch, n, local)
        h_in.a[:] = y.cpu().numpy()           # the bench input's transform: any data (data-oblivious path)
        del y
        torch.cuda.empty_cache()
        link = bf.link_probe(local, h_in, h_out, min(batch * 8 * n, 1 << 30), reps=3)
        bf.exec_host(h_in.a, n, bf.FFT_FORWARD, local, out=h_out.a)   # warm-up (cached pipeline)
        bd.barrier(dev)
        t0 = time.perf_counter()
        stats = None
        for _ in range(e2e_steps):
            stats = bf.exec_host(h_in.a, n, bf.FFT_FORWARD, local, out=h_out.a)
        el = bd.max_over_ranks(time.perf_counter() - t0, dev)
        each_way = batch * 8 * n * e2e_steps / el / 1e9
        e2e = {"value": recs_total * e2e_steps / el, "unit": "records/s",
               "h2d_bytes_per_step": int(batch * 8 * n), "d2h_bytes_per_step": int(batch * 8 * n),
               "steps": e2e_steps, "host_link_GBps_each_way": each_way,
               "host_link_roofline": {"h2d_GBps": link["both_h2d"], "d2h_GBps": link["both_d2h"],
                                      "h2d_alone_GBps": link["h2d"], "d2h_alone_GBps": link["d2h"],
                                      "how": "fft_link_probe: 1 GiB H2D and D2H at once, NUMA-local pinned"},
               "frac_of_host_link": each_way / min(link["both_h2d"], link["both_d2h"]),
               "numa_node": stats["numa_node"], "stream_stats_last_step": stats}
        h_in.close()
        h_out.close()
    else:
        del y

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, cores, sample = oracle_rate(n, seconds=args.cpu_seconds)
        cpu = {"value": v, "unit": "records/s", "cores": cores, "kind": "oracle", "sample": sample}

    if rank == 0:
        out = {
            "metric": "records_per_s", "value": value, "unit": "records/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded SplitMix64 counter stream, uniform [-1,1) complex64, generated in HBM)",
            "config": {"workload": cfg["name"], "n": n, "records_per_gpu": batch,
                       "direction": "forward", "variant": info["variant_name"],
                       "cluster": info["cluster"], "n1": info["n1"], "n2": info["n2"],
                       "l2": f"inputs {batch * 8 * n / 2**30:.1f} GiB per GPU >> L2 (126 MB); no flush needed",
                       "parallelism": f"dp{world} (independent record ranges, no collective)"},
            "alg_GBps": 16.0 * n * recs_total * args.steps / (max_ms * 1e-3) / 1e9,
            "file_GBps": 8.0 * n * recs_total * args.steps / (max_ms * 1e-3) / 1e9,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": kname, "alg_bytes_per_launch": alg_bytes,
                         "avg_launch_ms": avg_launch_s * 1e3, "peak_source": peak_src,
                         "traffic_source": traffic_src},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(args.steps * kernels_per_exec),
            "clocks": clk,
        }
        print(json.dumps(out), flush=True)
        print(f"[bench] {cfg['name']}: {value:.4g} records/s, {out['alg_GBps']:.1f} GB/s alg "
              f"({achieved / peak:.1%} of {peak:.0f}), {ms_per_step:.3f} ms/step, clocks {clk}", file=sys.stderr)
    plan.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
