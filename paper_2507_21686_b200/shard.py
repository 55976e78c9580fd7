"""Multi-GPU partitioning of the scene evaluation.

Particles are sharded into contiguous ranges of the original index across the
ranks (one process per GPU); the mesh and cell grid are replicated; each
particle is reduced entirely on one GPU in a fixed order, so the gathered
result is bitwise independent of the rank count. The only collective is an
all-gather of the per-particle (value, grad_x, grad_y) records (NCCL over
NVLink on GPUs; gloo in the CPU tests).
"""
from __future__ import annotations

from typing import Callable, Optional

import numpy as np


def shard_ranges(n: int, world: int) -> list:
    """Equal-count contiguous ranges [begin, end) per rank."""
    base, extra = divmod(n, world)
    out, b = [], 0
    for r in range(world):
        e = b + base + (1 if r < extra else 0)
        out.append((b, e))
        b = e
    return out


def balanced_ranges(pair_counts: np.ndarray, world: int) -> list:
    """Contiguous ranges cut at equal cumulative pair counts (work balance)."""
    n = int(pair_counts.shape[0])
    csum = np.concatenate([[0], np.cumsum(pair_counts, dtype=np.int64)])
    total = int(csum[-1])
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(csum, total * r / world, side="left")))
    cuts.append(n)
    cuts = np.maximum.accumulate(np.clip(cuts, 0, n))
    return [(int(cuts[r]), int(cuts[r + 1])) for r in range(world)]


def shard_pairs(pairs, begin: int, end: int):
    """Explicit pair list restricted to particles [begin, end), renumbered."""
    pp, pt = pairs
    m = (pp >= begin) & (pp < end)
    return pp[m] - begin, pt[m]


def gather_per_particle(local: np.ndarray, ranges: list, rank: int, device=None, group=None) -> np.ndarray:
    """All-gather (n_local, 3) float64 records into the full (n, 3) array.
    Shards are padded to the largest one (all_gather needs equal sizes)."""
    import torch
    import torch.distributed as dist

    world = len(ranges)
    mx = max(e - b for b, e in ranges)
    buf = torch.zeros((mx, 3), dtype=torch.float64, device=device)
    buf[: local.shape[0]] = torch.from_numpy(np.ascontiguousarray(local)).to(buf.device)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    out = np.empty((ranges[-1][1], 3), dtype=np.float64)
    for r, (b, e) in enumerate(ranges):
        out[b:e] = parts[r][: e - b].cpu().numpy()
    return out


def evaluate_sharded(particles, h, triangles, table, rank: int, world: int, tri_values=None, pairs=None,
                     ranges: Optional[list] = None, device=None, group=None,
                     evaluator: Optional[Callable] = None):
    """Evaluate this rank's particle shard and all-gather the full result.
    evaluator(particles, h, triangles, table, tri_values, pairs) -> (v, g);
    defaults to the GPU path (sphbi.evaluate)."""
    if evaluator is None:
        from . import sphbi

        def evaluator(p, h_, t, tab, vals, pr):
            v, g, _ = sphbi.evaluate(p, h_, t, tab, tri_values=vals, pairs=pr)
            return v, g

    n = particles.shape[0]
    ranges = ranges or shard_ranges(n, world)
    b, e = ranges[rank]
    local_pairs = shard_pairs(pairs, b, e) if pairs is not None else None
    v, g = evaluator(particles[b:e], h, triangles, table, tri_values, local_pairs)
    local = np.concatenate([np.asarray(v).reshape(-1, 1), np.asarray(g).reshape(-1, 2)], axis=1)
    return gather_per_particle(local, ranges, rank, device=device, group=group)
