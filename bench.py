#!/usr/bin/env python
"""Triangle-pair benchmark (BASELINE.json metric: triangle-pair tests/sec for
3DDistance / 3DIntersects at 1/2/4/8 B200 vs the CPU reference).

Default workload (BASELINE.json configs[1]): a synthetic
terrain (1024 x 512 cells, 1,048,576 CCW-up triangles, z ~ U(-20,20), seed 42)
against the reference ore body (make_ore_body, face target 1e6 -> 1,310,720
triangles); ST_3DDistance over every triangle pair, FP64.

A step is one pass of the hot path over one batch of A rows (default 65,536
terrain rows x 1,310,720 ore faces = 8.6e10 pairs); 16 batches are the whole
1M x 1M job, so the default --steps 16 times the full configuration. Under
torchrun each rank takes its own batches (weak scaling); per-step answers are
combined by NCCL MIN all-reduces (the distance, then the lowest pair among
the ranks holding it: the lexicographic (distance, pair) min).

  value        pairs/s with the meshes resident in HBM (CUDA events on the
               launch stream, max over ranks)
  e2e          same metric through the one-shot C-ABI calls from pinned host
               buffers (upload, prep, kernels, exact pass, D2H of the result
               inside the timed region)
  roofline     the roofline kernel (filter_kernel for distance, hit_kernel for
               intersects) against the FP64 peak measured in this run by a
               DFMA microbenchmark; algorithmic work W_d = 975 / W_i = 282
               FP64 flops per pair
  cpu_baseline the reference's own primitives (oracle/_ref: the A17
               composition over kernels.cpp) on this host's cores, on a sample

Other configurations (--config c1|c3|c4|c5) print the same
line for their workload. --impl reference times only the CPU reference
(rank 0) on the selected configuration.
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

METRIC = "triangle-pair tests/sec (3DDistance, 3DIntersects) at 1/2/4/8 B200 vs CPU ref"
UNIT = "pairs/s"
W_D = 975.0            # algorithmic FP64 flops per pair, distance
W_I = 282.0            # algorithmic FP64 flops per pair, intersects no-hit
# FULL-mode distance filter (scripts/sass_loops.py build/distance.o
# filter_kernelILb0 | vertex_kernel | edge_kernel): (FP64-pipe instructions,
# executed FP64 flops) per iteration. Per pair (one A face x one B face) the
# kernels run the face loop once, the vertex loop (B distinct vertices / B
# face) times, the vertex pair (A tile vertices / A face) times and the edge
# pair (A tile edges / A face) x (B block edges / B face) times.
FILTER_LOOP_FACE = (0, 0)      # filter_kernel<false> face loop (straddle test): skipped for every block whose
                               # bounding sphere lies beyond the A face's plane (~99% on C2); not counted
FILTER_LOOP_VERTEX = (13, 19)  # filter_kernel<false> vertex loop: a B vertex against the A face
FILTER_VERT_PAIR = (13, 19)    # vertex_kernel: an A tile vertex against a B face
FILTER_EDGE_PAIR = (31, 51)    # edge_kernel: an A tile edge against a B block edge
FILTER_EDGE_PAIR32 = (31, 48)  # edge32_kernel (FP32, the chunk a multiple of 1,024 faces), packed loop in
                               # scalar-equivalent ops per edge pair: 18 FFMA + 6 FMUL (one is the exact -fw) +
                               # 3 FADD + 3 FMUL.SAT + 1 FMNMX, + 1 MUFU.RCP (cuobjdump -sass; each FFMA2 /
                               # FMUL2 / FADD2 counts its two lanes; pinned by tests/test_sass_counts.py)
U64_MAX = (1 << 64) - 1
C3S_AXIS, C3S_ANGLE = (1.0, 2.0, 3.0), 0.37  # C3 stress variant rotation


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


# --------------------------------------------------------------------------
# mesh sources. The GPU arm builds its inputs with the product's generators;
# the reference arm (--impl reference) with the reference's own
# (oracle/_ref: dataset.cpp, rng.hpp) and never imports the product package.
# Both are pinned bit-for-bit to each other (tests/test_cpu_host.py).
# --------------------------------------------------------------------------
class ProductGen:
    def __init__(self):
        import paper_1808_09571_b200 as T
        self.unit_sphere, self.ore_body, self.terrain = T.unit_sphere, T.ore_body, T.terrain
        self.drills = lambda n, seed: T.drills(n, seed)


class ReferenceGen:
    def __init__(self):
        import oracle as O
        if O.REF is None:
            raise RuntimeError("oracle/_ref (the reference build) is missing")
        self.unit_sphere, self.ore_body, self.terrain = O.ref_unit_sphere, O.ref_ore_body, O.ref_terrain
        self.drills = lambda n, seed: O.ref_make_drills(seed, n, 0)


def translate(tris, dx=0.0, dy=0.0, dz=0.0):
    """Per-vertex translation (fixtures.cpp:37-46 translated)."""
    t = np.array(tris, dtype=np.float64, copy=True)
    t[:, 0::3] += dx
    t[:, 1::3] += dy
    t[:, 2::3] += dz
    return t


def rotate_scale(tris, axis, angle, scale):
    """scale * R(axis, angle) applied to every vertex (Rodrigues; C3's stress
    variant: '0.999 A rotated')."""
    k = np.asarray(axis, np.float64)
    k = k / np.linalg.norm(k)
    K = np.array([[0, -k[2], k[1]], [k[2], 0, -k[0]], [-k[1], k[0], 0]])
    R = np.eye(3) + np.sin(angle) * K + (1.0 - np.cos(angle)) * (K @ K)
    v = np.asarray(tris, np.float64).reshape(-1, 3) @ (scale * R).T
    return np.ascontiguousarray(v.reshape(-1, 9))


# --------------------------------------------------------------------------
# workloads
# --------------------------------------------------------------------------
class Workload:
    """Common step -> unit-range mapping. Units are A rows (mesh / query
    workloads) or records (table). A step is one batch of `batch_units`
    units. Weak scaling: rank r of W takes whole batch s*W + r. Strong
    scaling: every rank takes its slice of batch s (tile-aligned contiguous
    shards, shard.row_shards), so the job per step is fixed as W grows."""

    align = 128

    def span(self, s, rank=0, world=1, strong=False):
        if not strong:
            b = (s * world + rank) % self.n_batches
            return b * self.batch_units, min(self.n_units, (b + 1) * self.batch_units)
        b = s % self.n_batches
        lo, hi = b * self.batch_units, min(self.n_units, (b + 1) * self.batch_units)
        tiles = (hi - lo + self.align - 1) // self.align
        t0, t1 = (tiles * rank) // world, (tiles * (rank + 1)) // world
        return min(hi, lo + t0 * self.align), min(hi, lo + t1 * self.align)


class MeshWorkload(Workload):
    """A x B mesh workload; a step is a batch of A rows against all of B."""

    table = False

    def __init__(self, name, op, desc, make, batch_rows):
        self.name, self.op, self.desc, self._make, self.batch_rows = name, op, desc, make, batch_rows

    def build(self, gen):
        self.A, self.B = self._make(gen)
        self.NA, self.M = len(self.A), len(self.B)
        self.BR = min(self.batch_rows, self.NA)
        self.n_batches = (self.NA + self.BR - 1) // self.BR
        self.n_units, self.batch_units = self.NA, self.BR

    def pairs(self, r0, r1):
        return (r1 - r0) * self.M

    def upload(self, T):
        self.dA, self.dB = T.Mesh(self.A), T.Mesh(self.B)

    def run(self, T, r0, r1):
        if self.op == "distance":
            r = T.mesh_mesh_distance(self.dA, self.dB, rows=(r0, r1))
            return (r.distance, r.pair_index if r.pair_index is not None else U64_MAX)
        h = T.mesh_mesh_intersects(self.dA, self.dB, rows=(r0, r1))
        return (0.0 if h.hit else float("inf"), h.pair_index if h.hit else U64_MAX)

    def run_host(self, T, pinA, pinB, r0, r1):
        if self.op == "distance":
            r = T.distance_host(pinA[r0:r1], pinB)
            res = (r.distance, r.pair_index)
        else:
            h = T.intersects_host(pinA[r0:r1], pinB)
            res = (h.hit, h.pair_index)
        return res, (r1 - r0 + self.M) * 72, 96

    def cpu_rate(self, rows, threads):
        import oracle as O
        rows = min(rows, self.NA)
        stride = max(1, self.NA // rows)
        kind = "reference" if O.REF is not None else "port"
        t0 = time.perf_counter()
        if self.op == "distance":
            f = O.ref_mesh_mesh_distance if O.REF is not None else O.mesh_mesh_distance
        else:
            f = O.ref_mesh_mesh_intersects if O.REF is not None else O.mesh_mesh_intersects
        f(self.A, self.B, threads=threads, rows=(0, stride * rows, stride))
        dt = time.perf_counter() - t0
        return rows * self.M / dt, dt, kind, f"{rows} strided A rows x {self.M} B faces ({rows * self.M:.3g} pairs)"

    def cpu_default_rows(self, threads):
        per_row = self.M / (1.0e6 if self.op == "distance" else 6.0e6)  # s per row on one core
        # ~10-15 s of all-core work (R = 16 x nproc strided rows)
        return max(threads, int(20.0 * threads / max(per_row, 1e-6)))


class TableWorkload(Workload):
    """C4: a table of small objects (records) x one query mesh; a step is a
    batch of records, each record getting its own distance (run_batch)."""

    table = True
    align = 1

    def __init__(self, n_objects, batch_objects, op):
        self.name, self.op = "c4", op
        self.n_objects, self.batch_objects = n_objects, batch_objects
        self.desc = (f"C4: query orebody 81,920 tris vs table of {n_objects:,} objects x 1,280 tris "
                     f"(unit_sphere(1000) x U[2,10] + U(box)), per-record ST_3D{'Distance' if op == 'distance' else 'Intersects'}")

    def build(self, gen):
        self.Q = gen.ore_body(100_000)
        base = gen.unit_sphere(1000)
        rng = np.random.default_rng(42)
        scale = rng.uniform(2.0, 10.0, self.n_objects)
        ctr = np.stack([rng.uniform(0, 1000, self.n_objects), rng.uniform(0, 1000, self.n_objects),
                        rng.uniform(-400, 0, self.n_objects)], 1)
        self.nf = len(base)
        tab = np.empty((self.n_objects, self.nf, 9))
        for c in range(3):
            tab[:, :, c::3] = base[None, :, c::3] * scale[:, None, None] + ctr[:, None, c, None]
        self.tab = tab.reshape(-1, 9)
        self.M = len(self.Q)
        self.n_batches = (self.n_objects + self.batch_objects - 1) // self.batch_objects
        self.NA = len(self.tab)
        self.n_units, self.batch_units = self.n_objects, self.batch_objects

    def pairs(self, o0, o1):
        return (o1 - o0) * self.nf * self.M

    def upload(self, T):
        off = np.arange(self.n_objects + 1, dtype=np.uint64) * self.nf
        self.dT, self.dQ = T.Table(self.tab, off), T.Mesh(self.Q)

    def run(self, T, o0, o1):
        op = T.OP_DISTANCE if self.op == "distance" else T.OP_INTERSECTS
        v, p = T.table_eval(op, self.dT, self.dQ, objects=(o0, o1))
        return (float(np.min(v)) if self.op == "distance" else float(np.any(v)), int(p.min()) if len(p) else U64_MAX)

    def run_host(self, T, pinT, pinQ, o0, o1):
        off = np.arange(o1 - o0 + 1, dtype=np.uint64) * self.nf
        t = T.Table(pinT[o0 * self.nf:o1 * self.nf], off)
        q = T.Mesh(pinQ)
        op = T.OP_DISTANCE if self.op == "distance" else T.OP_INTERSECTS
        v, p = T.table_eval(op, t, q)
        t.free()
        q.free()
        return (v, p), ((o1 - o0) * self.nf + self.M) * 72, (o1 - o0) * 16

    def cpu_rate(self, rows, threads):
        import oracle as O
        kind = "reference" if O.REF is not None else "port"
        if self.op == "distance":
            f = O.ref_mesh_mesh_distance if O.REF is not None else O.mesh_mesh_distance
        else:
            f = O.ref_mesh_mesh_intersects if O.REF is not None else O.mesh_mesh_intersects
        objs = max(1, rows)
        t0 = time.perf_counter()
        for o in range(objs):
            f(self.tab[o * self.nf:(o + 1) * self.nf], self.Q, threads=threads)
        dt = time.perf_counter() - t0
        return objs * self.nf * self.M / dt, dt, kind, f"{objs} records x {self.nf} faces x {self.M} query faces"

    def cpu_default_rows(self, threads):
        return max(1, int(10.0 * threads * 1e6 / (self.nf * self.M)))


class QueryWorkload(Workload):
    """The paper's own workload: drill segments
    (make_drills, seed 42) x the ore body, per-segment distance_to_mesh /
    intersects_mesh. A step is one batch of drills against the whole ore."""

    align = 1

    table = False

    def __init__(self, n_drills, face_target, op, batch):
        self.name, self.op, self.n_drills, self.face_target, self.batch_rows = "paper", op, n_drills, face_target, batch
        self.desc = (f"paper: {n_drills:,} drill segments (make_drills) x ore body ({face_target}-face target), "
                     f"per-segment ST_3D{'Distance' if op == 'distance' else 'Intersects'} "
                     "(PAPER.md:352-361: 5M x 500 faces, 0.685 s on V100)")

    def build(self, gen):
        self.A = gen.drills(self.n_drills, 42)
        self.B = gen.ore_body(self.face_target)
        self.NA, self.M = len(self.A), len(self.B)
        self.BR = min(self.batch_rows, self.NA)
        self.n_batches = (self.NA + self.BR - 1) // self.BR
        self.n_units, self.batch_units = self.NA, self.BR

    def pairs(self, r0, r1):
        return (r1 - r0) * self.M

    def upload(self, T):
        self.dB = T.Mesh(self.B)
        self.dQ = {}

    def run(self, T, r0, r1):
        q = self.dQ.get((r0, r1))
        if q is None:  # query columns are resident like the meshes (uploaded on first use, untimed in warmup)
            q = self.dQ[(r0, r1)] = T.Queries(self.A[r0:r1])
        if self.op == "distance":
            d, f = T.queries_mesh_distance(q, self.dB)
            k = int(np.argmin(d))
            return float(d[k]), int(f[k])
        h, f = T.queries_mesh_intersects(q, self.dB)
        lowest = int(f.min())  # UINT64_MAX for the queries without a hit
        return (0.0, lowest) if lowest != U64_MAX else (float("inf"), U64_MAX)

    def run_host(self, T, pinA, pinB, r0, r1):
        m = T.Mesh(pinB)
        if self.op == "distance":
            res = T.segments_mesh_distance(pinA[r0:r1], m)
        else:
            res = T.segments_mesh_intersects(pinA[r0:r1], m)
        m.free()
        return res, (r1 - r0) * 48 + self.M * 72, (r1 - r0) * 16

    def cpu_rate(self, rows, threads):
        import oracle as O
        rows = min(rows, self.NA)
        kind = "reference" if O.REF is not None else "port"
        f = {("distance", True): O.ref_segments_mesh_distance, ("distance", False): O.segments_mesh_distance,
             ("intersects", True): O.ref_segments_mesh_intersects,
             ("intersects", False): O.segments_mesh_intersects}[(self.op, O.REF is not None)]
        t0 = time.perf_counter()
        f(self.A[:rows], self.B, threads=threads)
        dt = time.perf_counter() - t0
        return rows * self.M / dt, dt, kind, f"{rows} drills x {self.M} ore faces ({rows * self.M:.3g} pairs)"

    def cpu_default_rows(self, threads):
        per_row = self.M / (3.0e6 if self.op == "distance" else 2.0e7)
        return max(threads, int(10.0 * threads / max(per_row, 1e-9)))


def workload(name, op_override, objects):
    if name == "paper":
        return QueryWorkload(5_000_000, 500, op_override or "distance", 5_000_000)
    def c1(gen):
        a = gen.unit_sphere(10000)
        return a, translate(a, 2.5 if op_override != "intersects" else 0.5, 0, 0)

    def c2(gen):
        return gen.terrain(1024, 512, 20.0, 42), gen.ore_body(1_000_000)

    def c3(gen):
        a = gen.unit_sphere(1_000_000)
        return a, a * 0.9

    def c3s(gen):
        a = gen.unit_sphere(1_000_000)
        return a, rotate_scale(a, C3S_AXIS, C3S_ANGLE, 0.999)

    def c5(gen):
        a = gen.unit_sphere(10_000_000)
        return a, translate(a, 2.5, 0, 0)

    if name == "c1":
        op = op_override or "distance"
        return MeshWorkload("c1", op, f"C1: two 8,192-tri spheres ({'offset 2.5' if op == 'distance' else 'shift 0.5'}), "
                            f"ST_3D{'Distance' if op == 'distance' else 'Intersects'}", c1, 8192)
    if name == "c2":
        op = op_override or "distance"
        return MeshWorkload("c2", op, "C2: terrain 1,048,576 tris vs orebody 1,310,720 tris, "
                            f"ST_3D{'Distance' if op == 'distance' else 'Intersects'} (FP64, all pairs)", c2, 65536)
    if name == "c3":
        op = op_override or "intersects"
        return MeshWorkload("c3", op, "C3: 1,310,720-tri sphere vs 0.9x copy (overlapping AABBs, no hit: "
                            f"worst case), ST_3D{'Intersects' if op == 'intersects' else 'Distance'}", c3,
                            131072 if op == "intersects" else 65536)
    if name == "c3s":
        op = op_override or "intersects"
        return MeshWorkload("c3s", op, "C3 stress: 1,310,720-tri sphere vs 0.999x copy rotated 0.37 rad about (1,2,3) "
                            f"(surfaces 1e-3 apart, no hit), ST_3D{'Intersects' if op == 'intersects' else 'Distance'}",
                            c3s, 131072 if op == "intersects" else 65536)
    if name == "c4":
        return TableWorkload(objects, 1000, op_override or "distance")
    if name == "c5":
        op = op_override or "distance"
        return MeshWorkload("c5", op, "C5: 8,388,608-tri spheres offset 2.5, ST_3DDistance", c5, 65536)
    raise SystemExit(f"unknown config {name}")


# --------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.proc, self.lines = index, None, []

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


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def base_line(args, wl, world, value, ms):
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
    }


def config_of(args, wl, world):
    """The workload's config dict; both arms print exactly this."""
    return {"workload": wl.desc, "op": wl.op, "mode": args.mode,
            "pairs_per_step": wl.pairs(*wl.span(0)) * (1 if args.scaling == "strong" else world),
            "steps_per_job": wl.n_batches if args.scaling == "strong" else -(-wl.n_batches // world),
            "parallelism": f"rows{world}",
            "l2": "inputs larger than L2 (B / table stores of 288 B per face in HBM)"}


def run_reference(args, wl, rank, world):
    """--impl reference: the reference CPU path on the host cores (rank 0).
    Inputs come from the reference's own generators (oracle/_ref); this arm
    never imports paper_1808_09571_b200."""
    if rank != 0:
        return
    try:
        gen = ReferenceGen()
    except RuntimeError as e:
        print(json.dumps({"impl": "reference", "unavailable": str(e)}), flush=True)
        return
    wl.build(gen)
    threads = os.cpu_count() or 1
    # a whole number of rows per host thread (no idle threads in a step), ~3-4 s of CPU work per step
    rows = args.ref_rows or max(threads, (wl.cpu_default_rows(threads) // 2) // threads * threads)
    for _ in range(args.warmup):
        wl.cpu_rate(rows, threads)
    total_pairs, total_t, kind, sample, rates = 0.0, 0.0, "reference", "", []
    for _ in range(args.steps):
        rate, dt, kind, sample = wl.cpu_rate(rows, threads)
        total_pairs += rate * dt
        total_t += dt
        rates.append(rate)
    value = total_pairs / total_t
    out = base_line(args, wl, world, value, 1e3 * total_t)
    out.update({
        "impl": "reference",
        "config": config_of(args, wl, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": sample + " per step", "cpu_model": cpu_model(),
                         # the reference's own timing rule (bench.cpp:54-59,82): mean and sample stddev over repeats
                         "step_rate_mean": statistics.mean(rates),
                         "step_rate_stddev": statistics.stdev(rates) if len(rates) > 1 else 0.0},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    })
    print(json.dumps(out), flush=True)


def spawn_ranks(n):
    """--gpus N without a launcher: one process per GPU under
    torch.distributed.run (the same launch the driver uses), rendezvous on
    127.0.0.1; returns the launcher's exit code."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def plan_only(args, wl, rank, world):
    """Host-only check of the rank plan (tests/test_bench_contract.py): every
    rank reports the unit ranges it would evaluate in the timed steps; rank 0
    prints them with n_gpus. Builds the workload's inputs (the shapes fix the
    ranges) but touches no device."""
    import torch.distributed as dist
    from paper_1808_09571_b200 import shard
    if world > 1:
        dist.init_process_group(os.environ.get("TDB_BENCH_BACKEND", "gloo"))
    wl.build(ProductGen())
    strong = args.scaling == "strong"
    mine = [wl.span(args.warmup + s, rank, world, strong) for s in range(args.steps)]
    spans = [mine]
    if world > 1:
        spans = [None] * world
        dist.all_gather_object(spans, mine)
        # the answer every rank would hold after the step's reduction: here
        # the lexicographic min over ranks of each rank's (first unit, rank)
        d, p = shard.combine_min(float(mine[0][0]), rank)
    else:
        d, p = float(mine[0][0]), 0
    if rank == 0:
        print(json.dumps({"n_gpus": world, "scaling": args.scaling, "n_units": wl.n_units,
                          "batch_units": wl.batch_units, "spans": spans, "combined": [d, p]}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=16)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c3s", "c4", "c5", "paper"])
    ap.add_argument("--op", default=None, choices=[None, "distance", "intersects"])
    ap.add_argument("--batch-rows", type=int, default=0, help="A rows per step (0 = config default)")
    ap.add_argument("--objects", type=int, default=100_000, help="c4 table records")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--cpu-rows", type=int, default=0, help="cpu_baseline sample rows (0 = ~10 s)")
    ap.add_argument("--ref-rows", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--mode", default="full", choices=["full", "cull"])
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: each rank takes whole batches; strong: every step's batch is split over the ranks")
    ap.add_argument("--plan-only", action="store_true",
                    help="print the per-rank unit ranges of the timed steps and exit (no device work)")
    args = ap.parse_args()
    assert args.warmup >= 0 and args.steps >= 1 and args.gpus >= 1

    if "WORLD_SIZE" not in os.environ:
        if args.gpus > 1 and args.impl == "ours":
            return spawn_ranks(args.gpus)
        world_env = args.gpus  # reference arm: rank 0 only, reporting the job's GPU count
    else:
        world_env = env_int("WORLD_SIZE", 1)
        if world_env != args.gpus:
            raise SystemExit(f"bench.py: WORLD_SIZE={world_env} but --gpus {args.gpus}")

    wl = workload(args.config, args.op, args.objects)
    if args.batch_rows and not wl.table:
        wl.batch_rows = args.batch_rows
    rank, world, local = env_int("RANK", 0), world_env, env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, wl, rank, world)
    if args.plan_only:
        return plan_only(args, wl, rank, world)

    import torch
    import torch.distributed as dist

    import paper_1808_09571_b200 as T
    from paper_1808_09571_b200 import shard

    # one process per GPU; TDB_BENCH_BACKEND=gloo (with ranks sharing a GPU)
    # only exercises the multi-rank plumbing on a one-GPU box
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("TDB_BENCH_BACKEND", "nccl")
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator lines (nranks) stay in the log
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    T.init(local)
    T.set_mode(T.MODE_CULL if args.mode == "cull" else T.MODE_FULL)
    stream = torch.cuda.current_stream()
    T.set_stream(stream.cuda_stream)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def over_ranks(x, op):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=op)
        return float(t.item())

    def max_over_ranks(x):
        return over_ranks(x, dist.ReduceOp.MAX if world > 1 else None)

    def sum_over_ranks(x):
        return over_ranks(x, dist.ReduceOp.SUM if world > 1 else None)

    fp64_tf, _ = T.fp64_peak()
    wl.build(ProductGen())
    wl.upload(T)

    results, k_ms, k_pairs, kernels = [], [], [], 0

    strong = args.scaling == "strong"

    def step(s, record=True):
        nonlocal kernels
        lo, hi = wl.span(s, rank, world, strong)
        d, p = wl.run(T, lo, hi)
        st = T.last_stats()
        d, p = shard.combine_min(d, p, device="cuda")  # NCCL MIN all-reduce (distance, then pair)
        if record:
            results.append((d, p))
            k_ms.append(st["ms_filter"])
            k_pairs.append(st["pairs"])
            kernels += st["kernels"]
        return wl.pairs(lo, hi)

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
    pairs_total = sum_over_ranks(float(pairs_rank))  # units all ranks processed
    value = pairs_total / (ms * 1e-3)

    # ---- e2e: one-shot C-ABI calls from pinned host buffers -----------------
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else args.steps
    if wl.table:
        pinA, pinB = torch.from_numpy(wl.tab).pin_memory().numpy(), torch.from_numpy(wl.Q).pin_memory().numpy()
    else:
        pinA, pinB = torch.from_numpy(wl.A).pin_memory().numpy(), torch.from_numpy(wl.B).pin_memory().numpy()
    h2d = d2h = 0
    e2e_pairs = 0
    barrier()
    clocks_e2e = ClockSampler(local)
    clocks_e2e.start()
    t0 = time.perf_counter()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    for s in range(e2e_steps):
        lo, hi = wl.span(args.warmup + s, rank, world, strong)
        _, hb, db = wl.run_host(T, pinA, pinB, lo, hi)
        h2d += hb
        d2h += db
        e2e_pairs += wl.pairs(lo, hi)
    e3.record(stream)
    barrier()
    wall_e2e = time.perf_counter() - t0
    clk_e2e = clocks_e2e.stop()
    ms_e2e = max_over_ranks(max(e2.elapsed_time(e3), wall_e2e * 1e3))
    e2e_value = sum_over_ranks(float(e2e_pairs)) / (ms_e2e * 1e-3)

    # ---- roofline of the roofline kernel -------------------------------------
    f_ms = sum(k_ms) / len(k_ms)
    f_pairs = sum(k_pairs) / len(k_pairs)
    if wl.name == "paper":  # segment x triangle: SURVEY.md 8(a) A10 / A11 op counts
        w = 473.0 if wl.op == "distance" else 75.0
        kname = "q_filter_kernel" if wl.op == "distance" else "q_hit_kernel"
    else:
        w = W_D if wl.op == "distance" else W_I
        kname = "filter_kernel" if wl.op == "distance" else "hit_kernel"
    achieved_tf = w * f_pairs / (f_ms * 1e-3) / 1e12
    traffic = None
    try:  # DRAM bytes per pair from the committed ncu --set full capture, scaled to this launch
        tj = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))[kname]
        traffic = tj["dram_bytes_per_pair"] * f_pairs
    except (OSError, KeyError, ValueError):
        pass
    roofline = {
        "bound": "fp64", "achieved": achieved_tf, "peak": fp64_tf, "unit": "TFLOP/s",
        "frac": achieved_tf / fp64_tf, "traffic": traffic,
        "traffic_note": "dram__bytes_read+write per launch from profiles/traffic.json (ncu --set full; the "
                        "three filter-stage kernels summed for distance), scaled to this launch's pairs",
        "kernel": (kname if wl.op != "distance" or wl.name == "paper" else
                   "filter stage: edge_kernel (dominant, ~74% of it) + vertex_kernel + filter_kernel<false>, "
                   "timed together (events around the three launches)"),
        "work_per_pair_flops": w,
        "peak_source": "measured in this run: DFMA issue-rate microbenchmark (tdb_fp64_peak); "
                       "spec 148 SM x 64 FMA x 2 x 1.965 GHz = 37.2",
        "kernel_share_of_step": sum(k_ms) / ms if world == 1 else None,
    }
    if wl.op == "distance" and wl.name != "paper":
        fb = (wl.dQ if wl.table else wl.dB).feature_counts()
        fa = (wl.dT if wl.table else wl.dA).feature_counts()
        per_face_v = fb["vertices"] / fb["faces"]
        # the library's B-chunk choice (runtime.h pick_chunk): B's edges come
        # per 1,024 faces when the chunk is a multiple of that, else per block
        units = wl.batch_units if wl.table else wl.BR
        tiles = -(-units * (wl.nf if wl.table else 1) // 128)
        nb = len(wl.Q) if wl.table else wl.M
        chunk, target = 8192, torch.cuda.get_device_properties(local).multi_processor_count * 12
        while chunk > 64 and tiles * -(-nb // chunk) < target:
            chunk //= 2
        r_chunk_super = chunk % 1024 == 0
        per_face_e = (fb["super_edges"] if r_chunk_super else fb["edges"]) / fb["faces"]
        a_edges, a_verts = fa["tile_edges"] / fa["faces"], fa["tile_vertices"] / fa["faces"]
        ep = a_edges * per_face_e  # edge pairs per face pair
        instr = (FILTER_LOOP_FACE[0] + per_face_v * FILTER_LOOP_VERTEX[0] + a_verts * FILTER_VERT_PAIR[0]
                 + (0 if r_chunk_super else ep * FILTER_EDGE_PAIR[0]))
        flops = (FILTER_LOOP_FACE[1] + per_face_v * FILTER_LOOP_VERTEX[1] + a_verts * FILTER_VERT_PAIR[1]
                 + (0 if r_chunk_super else ep * FILTER_EDGE_PAIR[1]))
        instr32 = ep * FILTER_EDGE_PAIR32[0] if r_chunk_super else 0.0  # FP32 pipe (edge32_kernel)
        flops32 = ep * FILTER_EDGE_PAIR32[1] if r_chunk_super else 0.0
        roofline["features_per_face"] = {"b_vertices": per_face_v, "b_edges": per_face_e, "a_tile_edges": a_edges,
                                         "a_tile_vertices": a_verts}
        roofline["fp64_instr_per_pair"] = instr
        roofline["note"] = ("achieved/frac count W_d = 975 flops per pair (the per-pair algorithm, SURVEY.md 8(d)); "
                            "the kernels evaluate each distinct vertex / edge of a B block and each distinct edge of "
                            "an A tile once (DESIGN.md 4.1), so they execute executed_fp64_tflops and frac > 1 is "
                            "algorithmic; fp64_pipe_frac is the hardware fraction (FP64-pipe issue / peak)")
        roofline["fp64_pipe_frac"] = instr * f_pairs / (f_ms * 1e-3) / (fp64_tf * 1e12 / 2)
        roofline["executed_fp64_tflops"] = flops * f_pairs / (f_ms * 1e-3) / 1e12
        if r_chunk_super:  # the edge/edge candidates run on the FP32 pipe (128 lanes per SM per clock)
            sm_mhz = (clk or {}).get("sm_mhz") or 1965.0
            fp32_rate = torch.cuda.get_device_properties(local).multi_processor_count * 128 * sm_mhz * 1e6
            roofline["fp32_instr_per_pair"] = instr32
            roofline["fp32_pipe_frac"] = instr32 * f_pairs / (f_ms * 1e-3) / fp32_rate
            roofline["executed_fp32_tflops"] = flops32 * f_pairs / (f_ms * 1e-3) / 1e12
            roofline["pipe_busy_frac"] = roofline["fp64_pipe_frac"] + roofline["fp32_pipe_frac"]
            roofline["kernel"] = ("filter stage: edge32_kernel (FP32 edge/edge candidates) + vertex_kernel + "
                                  "filter_kernel<false> (FP64), timed together (events around the three launches)")
            roofline["note"] += ("; the edge/edge candidates run in FP32 (edge32_kernel, band widened by eta_f32), "
                                 "so fp64_pipe_frac + fp32_pipe_frac = pipe_busy_frac is the stage's hardware "
                                 "fraction (the kernels run one after another)")
    elif wl.op == "intersects":
        roofline["note"] = ("culled pairs skip the W_i work (conservative FP32/FP64 separating-plane test, "
                            "DESIGN.md 4.3): frac > 1 is algorithmic, not hardware")
    else:
        roofline["note"] = ("segment x triangle: W = 473 flops/pair is the reference composition's count "
                            "(SURVEY.md 8(a) A10); the FP64 filter needs fewer, so frac can exceed 1")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        rows = args.cpu_rows or max(threads, wl.cpu_default_rows(threads) // threads * threads)  # whole rows per thread
        rate, dt, kind, sample = wl.cpu_rate(rows, threads)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": kind, "sample": f"{sample}, {dt:.1f} s",
               "cpu_model": cpu_model()}
        # the single-core rate beside the all-core one (a one-thread sample of ~1-3 s)
        r1, dt1, _, sample1 = wl.cpu_rate(max(1, rows // threads // 4), 1)
        cpu["single_core"] = {"value": r1, "sample": f"{sample1}, {dt1:.1f} s"}

    if rank == 0:
        best = min(results) if results else (None, None)
        out = base_line(args, wl, world, value, ms)
        out.update({
            "config": config_of(args, wl, world),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d // max(1, e2e_steps),
                    "d2h_bytes_per_step": d2h // max(1, e2e_steps), "steps": e2e_steps},
            "roofline": roofline, "cpu_baseline": cpu, "clocks": clk, "clocks_e2e": clk_e2e,
            "gpu_launches": kernels,
            "result": {"best_value_seen": best[0], "pair": best[1]},
        })
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
