"""Multi-GPU plumbing for the triangle-pair path.

One process per GPU. Pairs are independent, so the A axis (rows of the
first mesh, or objects of a table) is split into contiguous shards and each
rank evaluates its shard against the replicated B with no data-path
collective. The only exchange is the final reduction of the per-rank answers:

* distance   : lexicographic min of (distance, pair index) — a MIN
               all-reduce of the distance (non-negative doubles order as their
               int64 bits), then a MIN all-reduce of the pair among the ranks
               holding that distance (NCCL over NVLink on B200s, gloo on CPU);
* intersects : one MIN all-reduce of the lowest hit pair index (the OR of the
               ranks' hits, keeping the reference's lowest-index winner);
* table      : each rank owns a slice of records; slices are gathered.

Pair indices are global (i * |B| + j) on every rank, so the reduced answer is
exactly the single-GPU answer (tests/test_gpu_parity.py shard tests,
tests/test_multirank_gloo.py).
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import numpy as np

U64_MAX = (1 << 64) - 1
TILE = 128  # A rows per CTA tile (tdb_internal.h kTile); shard cuts align to it


def row_shards(n_rows: int, world: int, align: int = TILE) -> List[Tuple[int, int]]:
    """Contiguous, tile-aligned [begin, end) row ranges, one per rank,
    covering [0, n_rows) with sizes differing by at most one tile."""
    tiles = (n_rows + align - 1) // align
    out = []
    for r in range(world):
        t0 = (tiles * r) // world
        t1 = (tiles * (r + 1)) // world
        out.append((min(n_rows, t0 * align), min(n_rows, t1 * align)))
    return out


def object_shards(face_offsets: Sequence[int], world: int) -> List[Tuple[int, int]]:
    """Contiguous object ranges with near-equal face counts (SURVEY.md 8(e):
    'shard rows by contiguous ranges with equal total face count')."""
    off = np.asarray(face_offsets, dtype=np.int64)
    n_obj = len(off) - 1
    total = int(off[-1])
    cuts = [0]
    for r in range(1, world):
        target = (total * r) // world
        cuts.append(int(np.searchsorted(off[:-1], target, side="left")))
    cuts.append(n_obj)
    cuts = [min(max(c, cuts[i - 1] if i else 0), n_obj) for i, c in enumerate(cuts)]
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def lexmin(pairs: Sequence[Tuple[float, int]]) -> Tuple[float, int]:
    """Lexicographic min of (distance, pair); unfound = (inf, UINT64_MAX)."""
    best = (float("inf"), U64_MAX)
    for d, p in pairs:
        if (d, p) < best:
            best = (d, p)
    return best


I64_MAX = (1 << 63) - 1  # "no pair" inside the int64 reductions


def _allreduce_min(value: int, group=None, device=None) -> int:
    import torch
    import torch.distributed as dist_

    t = torch.tensor([value], dtype=torch.int64, device=device or "cpu")
    dist_.all_reduce(t, op=dist_.ReduceOp.MIN, group=group)
    return int(t.item())


def combine_min(dist: float, pair: Optional[int], group=None, device=None) -> Tuple[float, int]:
    """All ranks get the lexicographic (distance, pair) min over ranks."""
    import torch.distributed as dist_

    none = pair is None or int(pair) == U64_MAX  # both spell "no pair" (callers pass either)
    p = U64_MAX if none else int(pair)
    if not dist_.is_initialized() or dist_.get_world_size(group) == 1:
        return float(dist), p
    dbits = int(np.float64(dist).view(np.int64))  # >= 0 (or +inf): orders as the double
    gbits = _allreduce_min(dbits, group, device)
    mine = p if (dbits == gbits and not none) else I64_MAX
    gp = _allreduce_min(mine, group, device)
    return float(np.int64(gbits).view(np.float64)), (U64_MAX if gp == I64_MAX else gp)


def combine_hit(pair: Optional[int], group=None, device=None) -> Optional[int]:
    """Lowest hit pair over ranks (None when no rank hit): one MIN all-reduce."""
    import torch.distributed as dist_

    if not dist_.is_initialized() or dist_.get_world_size(group) == 1:
        return pair
    none = pair is None or int(pair) == U64_MAX
    gp = _allreduce_min(I64_MAX if none else int(pair), group, device)
    return None if gp == I64_MAX else gp


def gather_slices(local: np.ndarray, counts: Sequence[int], group=None, device=None) -> np.ndarray:
    """Concatenate per-rank result slices (table path) in rank order."""
    import torch
    import torch.distributed as dist_

    if not dist_.is_initialized() or dist_.get_world_size(group) == 1:
        return local
    width = max(counts) if counts else 0
    raw = np.ascontiguousarray(local).view(np.uint8).reshape(len(local), -1)
    item = raw.shape[1] if len(local) else np.dtype(local.dtype).itemsize
    buf = np.zeros((width, item), np.uint8)
    buf[: len(local)] = raw
    t = torch.from_numpy(buf).to(device or "cpu")
    g = [torch.empty_like(t) for _ in range(dist_.get_world_size(group))]
    dist_.all_gather(g, t, group=group)
    parts = [x.cpu().numpy()[:c].reshape(-1).view(local.dtype) for x, c in zip(g, counts)]
    return np.concatenate(parts)


def mesh_mesh_distance_sharded(A, B, rank: int, world: int, group=None, device=None):
    """Rank-local rows of A against B on this rank's GPU, reduced over ranks."""
    from . import mesh_mesh_distance

    r0, r1 = row_shards(A.faces, world)[rank]
    r = mesh_mesh_distance(A, B, rows=(r0, r1))
    return combine_min(r.distance, r.pair_index, group, device)


def mesh_mesh_intersects_sharded(A, B, rank: int, world: int, group=None, device=None):
    from . import mesh_mesh_intersects

    r0, r1 = row_shards(A.faces, world)[rank]
    h = mesh_mesh_intersects(A, B, rows=(r0, r1))
    return combine_hit(h.pair_index, group, device)
