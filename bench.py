#!/usr/bin/env python
"""Triangle-pair ST_3DDistance benchmark (BASELINE.json metric).

Workload (BASELINE.json configs[1]): synthetic terrain
(1024 x 512 cells, 1,048,576 CCW-up triangles, z ~ U(-20,20), seed 42)
against the reference ore body (make_ore_body, face target 1e6 ->
1,310,720 triangles), ST_3DDistance over every triangle pair, FP64.

A step is one pass of the hot path over one batch of terrain rows
(--batch-rows, default 65,536 rows x 1,310,720 ore faces = 8.6e10 pairs);
16 batches are the whole 1M x 1M job, so the default --steps 16 times the
full configuration. Under torchrun each rank takes its own batches (weak
scaling); per-step results are combined with an NCCL all_gather of 16 B per
rank (the lexicographic (distance, pair) min).

  value : pairs/s with both meshes resident in HBM (device events, max over
          ranks)
  e2e   : same metric through the one-shot C-ABI call with pinned host
          buffers (tdb_distance_host: H2D of the step's meshes, prep, filter,
          exact pass, D2H of the result inside the timed region)
  roofline : the filter kernel (the roofline kernel) against the FP64 peak
          measured in this run by a DFMA microbenchmark; algorithmic work
          W_d = 975 FP64 flops per pair.
  cpu_baseline : the reference's own primitives (oracle/_ref, the A17
          composition) on this host's cores on a row sample.

--impl reference times only that CPU reference (rank 0) on the same metric.
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

W_D = 975.0          # algorithmic FP64 flops per triangle pair
W_REF = 2838.0       # reference-composition flops per pair (op-counted)
FILTER_DP_INSTR = 318  # FP64-pipe instructions per pair in filter_kernel (cuobjdump -sass count)
FILTER_FLOPS = 492     # executed FP64 flops per pair (174 DFMA x 2 + 93 DMUL + 51 DADD)
METRIC = "triangle-pair tests/sec (3DDistance, 3DIntersects) at 1/2/4/8 B200 vs CPU ref"
UNIT = "pairs/s"
WORKLOAD = "C2: terrain 1,048,576 tris vs orebody 1,310,720 tris, ST_3DDistance (FP64, all pairs)"


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def make_meshes():
    import paper_1808_09571_b200 as T
    ter = T.terrain(1024, 512, 20.0, 42)
    ore = T.ore_body(1_000_000)
    return ter, ore


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
                power.append(float(f[3]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "power_w_max": max(power), "samples": len(sm)}


def cpu_reference_rate(ter, ore, rows, threads):
    """The reference's primitives (oracle/_ref) on `rows` strided terrain rows
    x all ore faces; falls back to the C restatement if _ref is absent."""
    import oracle as O
    n = len(ter)
    stride = max(1, n // rows)
    kind = "reference" if O.REF is not None else "port"
    t0 = time.perf_counter()
    if O.REF is not None:
        r = O.ref_mesh_mesh_distance(ter, ore, threads=threads, rows=(0, stride * rows, stride))
    else:
        r = O.mesh_mesh_distance(ter, ore, threads=threads, rows=(0, stride * rows, stride))
    dt = time.perf_counter() - t0
    return rows * len(ore) / dt, dt, kind, r


def run_reference(args, rank, world):
    """--impl reference: the reference CPU path on the host cores (rank 0)."""
    if rank != 0:
        return
    import oracle as O
    import paper_1808_09571_b200 as T
    ter = T.terrain(1024, 512, 20.0, 42)   # new generator (no reference terrain)
    ore = O.ref_ore_body(1_000_000) if O.REF is not None else T.ore_body(1_000_000)
    threads = os.cpu_count() or 1
    rows = max(1, args.ref_rows or threads)
    for _ in range(args.warmup):
        cpu_reference_rate(ter, ore, rows, threads)
    total_pairs, total_t, kind = 0, 0.0, "reference"
    for _ in range(args.steps):
        rate, dt, kind, _ = cpu_reference_rate(ter, ore, rows, threads)
        total_pairs += rows * len(ore)
        total_t += dt
    value = total_pairs / total_t
    sample = f"{rows} strided terrain rows x {len(ore)} ore faces per step"
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": WORKLOAD, "parallelism": f"cpu{threads}"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=16)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch-rows", type=int, default=65536)
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--cpu-rows", type=int, default=0, help="rows for cpu_baseline (0 = auto)")
    ap.add_argument("--ref-rows", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    assert args.warmup >= 0 and args.steps >= 1

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    import paper_1808_09571_b200 as T

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    T.init(local)
    stream = torch.cuda.current_stream()
    T.set_stream(stream.cuda_stream)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    from paper_1808_09571_b200 import shard

    def combine(d, p):
        """Lexicographic (distance, pair) min over ranks: NCCL all_gather."""
        return shard.combine_min(d, p, device="cuda")

    fp64_tf, _ = T.fp64_peak()
    ter, ore = make_meshes()
    NA, M = len(ter), len(ore)
    BR = min(args.batch_rows, NA)
    n_batches = (NA + BR - 1) // BR
    A, B = T.Mesh(ter), T.Mesh(ore)

    def batch_rows(s):
        b = (s * world + rank) % n_batches
        return b * BR, min(NA, (b + 1) * BR)

    results = []
    filt_ms, filt_pairs, kernels = [], [], 0

    def step(s, record=True):
        nonlocal kernels
        r0, r1 = batch_rows(s)
        r = T.mesh_mesh_distance(A, B, rows=(r0, r1))
        st = T.last_stats()
        d, p = combine(r.distance, r.pair_index if r.pair_index is not None else (1 << 64) - 1)
        if record:
            results.append((r0, r1, d, p))
            filt_ms.append(st["ms_filter"])
            filt_pairs.append(st["pairs"])
            kernels += st["kernels"]
        return (r1 - r0) * M

    for s in range(args.warmup):
        step(s, record=False)
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    pairs_rank = 0
    for s in range(args.steps):
        pairs_rank += step(args.warmup + s)
    e1.record(stream)
    barrier()
    clk = clocks.stop()
    ms = max_over_ranks(e0.elapsed_time(e1))
    pairs_total = pairs_rank * world
    value = pairs_total / (ms * 1e-3)

    # ---- e2e: one-shot C-ABI call from pinned host buffers -----------------
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else args.steps
    pin_a = torch.from_numpy(ter).pin_memory()
    pin_b = torch.from_numpy(ore).pin_memory()
    na_pin, nb_pin = pin_a.numpy(), pin_b.numpy()
    h2d = 0
    barrier()
    t0 = time.perf_counter()
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    e2e_pairs = 0
    for s in range(e2e_steps):
        r0, r1 = batch_rows(args.warmup + s)
        r = T.distance_host(na_pin[r0:r1], nb_pin)
        h2d += (r1 - r0 + M) * 72
        e2e_pairs += (r1 - r0) * M
    e3.record(stream)
    barrier()
    wall_e2e = time.perf_counter() - t0
    ms_e2e = max_over_ranks(max(e2.elapsed_time(e3), wall_e2e * 1e3))
    e2e_value = e2e_pairs * world / (ms_e2e * 1e-3)

    # ---- roofline of the filter kernel --------------------------------------
    f_ms = sum(filt_ms) / len(filt_ms)
    f_pairs = sum(filt_pairs) / len(filt_pairs)
    achieved_tf = W_D * f_pairs / (f_ms * 1e-3) / 1e12
    roofline = {
        "bound": "fp64", "achieved": achieved_tf, "peak": fp64_tf, "unit": "TFLOP/s",
        "frac": achieved_tf / fp64_tf, "traffic": None,
        "kernel": "filter_kernel (fast_pair.cuh)",
        "work_per_pair_flops": W_D,
        "peak_source": "measured in this run: DFMA issue-rate microbenchmark (tdb_fp64_peak); "
                       "spec 148 SM x 64 FMA x 2 x 1.965 GHz = 37.2",
        "fp64_pipe_frac": FILTER_DP_INSTR * f_pairs / (f_ms * 1e-3) / (fp64_tf * 1e12 / 2),
        "executed_fp64_tflops": FILTER_FLOPS * f_pairs / (f_ms * 1e-3) / 1e12,
        "filter_share_of_step": sum(filt_ms) / ms if world == 1 else None,
    }

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        rows = args.cpu_rows or 8 * threads
        rate, dt, kind, _ = cpu_reference_rate(ter, ore, rows, threads)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": kind,
               "sample": f"{rows} strided terrain rows x {M} ore faces ({rows * M:.3g} pairs, {dt:.1f} s)"}

    if rank == 0:
        best = min(((d, p) for (_, _, d, p) in results), default=(None, None))
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "batch_rows": BR, "pairs_per_step": BR * M * world,
                       "batches_per_job": n_batches, "parallelism": f"rows{world}",
                       "l2": "inputs larger than L2 (B store 377 MB of SoA planes)",
                       "op": "ST_3DDistance"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d // max(1, e2e_steps),
                    "d2h_bytes_per_step": 96, "steps": e2e_steps},
            "roofline": roofline, "cpu_baseline": cpu, "clocks": clk,
            "gpu_launches": kernels,
            "result": {"min_distance_seen": best[0], "pair": best[1]},
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
