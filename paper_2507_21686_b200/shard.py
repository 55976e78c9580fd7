"""Multi-GPU partition of the scene evaluation (BASELINE.json
north_star: "Work is partitioned across the 8 B200s of one box by sharding
particles, with the triangle mesh and cell grid replicated; no collective is
needed beyond an NCCL all-gather of the per-particle results over NVLink").

The reference has no batch path or partition (it evaluates one pair per call;
SPEC.md:477 notes the pairs are embarrassingly parallel). Here, one process
per GPU:

* every rank holds the whole particle array, the mesh and (per call) the cell
  grid in its HBM -- replicated, 256 MB of positions and ~100 MB of mesh at
  cfg5;
* particles are cut into contiguous index ranges, one per rank: equal counts,
  or equal pair counts from the device count pass (`sphbi_pair_counts`, run
  sharded: each rank counts one equal block, the counts are all-gathered and
  every rank derives the same cuts);
* each rank evaluates its range with `sphbi_evaluate` on device pointers and
  writes value / gradient straight into its slice of the all-gather buffer
  (layout per rank: [value x m | grad x 2m], m = the largest shard);
* one in-place all-gather (NCCL over NVLink) assembles every rank's records;
  a device copy unpacks them into value (n,) and gradient (n, 2).

Each particle is reduced entirely on one rank in ascending triangle order and
the pair finder's results do not depend on which other particles share the
call, so the gathered result is bitwise identical for any rank count and cut
(tests/test_distributed.py, tests/test_gpu_sharded.py).

With the gloo backend (CPU tests; several ranks sharing one GPU in the GPU
test) CUDA tensors are staged through host memory for the collective -- NCCL
refuses two ranks on one device; on a real multi-GPU box the buffer stays in
HBM.
"""
from __future__ import annotations

import ctypes
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


def balanced_ranges(pair_counts, world: int) -> list:
    """Contiguous ranges cut at equal cumulative pair counts (work balance).
    Cut r is the first index whose prefix sum reaches r/world of the total."""
    pc = np.asarray(pair_counts, dtype=np.int64).reshape(-1)
    n = int(pc.shape[0])
    csum = np.concatenate([[0], np.cumsum(pc, dtype=np.int64)])
    total = int(csum[-1])
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(csum, (total * r + world - 1) // world, side="left")))
    cuts.append(n)
    cuts = np.maximum.accumulate(np.clip(cuts, 0, n))
    return [(int(cuts[r]), int(cuts[r + 1])) for r in range(world)]


def balanced_ranges_device(counts, world: int) -> list:
    """balanced_ranges on a device int64 tensor of per-particle pair counts:
    prefix sum and search on the GPU, only the world + 1 cuts reach the host.
    Bitwise the same cuts as balanced_ranges."""
    import torch

    n = int(counts.shape[0])
    csum = torch.cumsum(counts.to(torch.int64), 0)
    total = int(csum[-1].item()) if n else 0
    targets = torch.tensor([(total * r + world - 1) // world for r in range(1, world)], dtype=torch.int64,
                           device=counts.device)
    # csum here is inclusive; index j of the exclusive prefix = 1 + (first k with csum[k] >= target)
    inner = (torch.searchsorted(csum, targets, side="left") + 1).clamp(max=n) if n else targets * 0
    inner = torch.where(targets <= 0, torch.zeros_like(inner), inner)
    cuts = [0] + [int(x) for x in inner.tolist()] + [n]
    for i in range(1, len(cuts)):
        cuts[i] = max(cuts[i], cuts[i - 1])
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def shard_pairs(pairs, begin: int, end: int):
    """Explicit pair list restricted to particles [begin, end), renumbered."""
    pp, pt = pairs
    m = (pp >= begin) & (pp < end)
    return pp[m] - begin, pt[m]


def _all_gather_inplace(buf, local, group=None):
    """In-place all-gather of `local` (this rank's slice of the flat `buf`)."""
    import torch.distributed as dist

    if buf.is_cuda and dist.get_backend(group) != "nccl":
        hb = buf.cpu()
        world = dist.get_world_size(group)
        m = hb.numel() // world
        rank = dist.get_rank(group)
        dist.all_gather_into_tensor(hb, hb[rank * m:(rank + 1) * m].clone(), group=group)
        buf.copy_(hb.to(buf.device))
        return
    dist.all_gather_into_tensor(buf, local, group=group)


class ShardedScene:
    """This rank's part of a particle-sharded scene evaluation.

    particles (n, 2), triangles (T, 6) and tri_values ((T, 3) or None) are
    float64 tensors on this rank's device, replicated on every rank. table is
    a sphbi.KernelTermTable. balance: "count" (equal particle counts) or
    "pairs" (equal pair counts from the sharded device count pass).
    evaluator(p_begin, p_end, out_value_view, out_grad_view) overrides the
    device call (the CPU tests pass the oracle); with balance="pairs" it also
    needs evaluator.counts(p_begin, p_end) -> per-particle pair counts."""

    def __init__(self, particles, triangles, table, h: float, tri_values=None, ctx=None, group=None,
                 balance: str = "count", evaluator: Optional[Callable] = None):
        import torch
        import torch.distributed as dist

        self.group = group
        self.distributed = dist.is_available() and dist.is_initialized()
        self.rank = dist.get_rank(group) if self.distributed else 0
        self.world = dist.get_world_size(group) if self.distributed else 1
        self.particles, self.triangles, self.tri_values = particles, triangles, tri_values
        self.h = float(h)
        self.table = table
        self.n = int(particles.shape[0])
        self.device = particles.device
        self.evaluator = evaluator
        self.ctx = ctx
        if evaluator is None and ctx is None:
            from . import sphbi
            self.ctx = sphbi.default_context(self.device.index or 0)
        self.stats = None
        self.count_ms = 0.0
        if balance == "pairs":
            self.ranges = self._balanced_by_pairs()
        elif balance == "count":
            self.ranges = shard_ranges(self.n, self.world)
        else:
            raise ValueError(f"unknown balance {balance!r}")
        # shard slot length: a multiple of 64 records, so each rank's value and
        # gradient blocks start 512-B aligned (the reduction stores double2)
        self.m = -(-max(1, max(e - b for b, e in self.ranges)) // 64) * 64
        self.buf = torch.zeros(self.world * 3 * self.m, dtype=torch.float64, device=self.device)

    # ---- work balance -------------------------------------------------
    def _pair_counts(self, b: int, e: int):
        """Device count pass over particles [b, e) -> int64 tensor (e - b,)."""
        import torch

        from . import _native as N
        from .sphbi import _raise

        out = torch.zeros(max(e - b, 1), dtype=torch.int64, device=self.device)
        if e > b:
            self.ctx.set_stream(torch.cuda.current_stream(self.device).cuda_stream)  # ordered with `out`'s zeroing
            stats = N.Stats()
            lib = self.ctx.lib
            p = self.particles[b:e]
            _raise(lib.sphbi_pair_counts(self.ctx.handle, self.h, e - b, ctypes.c_void_p(p.data_ptr()),
                                         int(self.triangles.shape[0]), ctypes.c_void_p(self.triangles.data_ptr()),
                                         ctypes.c_void_p(out.data_ptr()), None, ctypes.byref(stats), N.MEM_DEVICE),
                   "pair_counts")
            self.count_ms += stats.ms_pairs
        return out[: e - b]

    def _balanced_by_pairs(self):
        import torch

        blocks = shard_ranges(self.n, self.world)
        mb = -(-max(1, max(e - b for b, e in blocks)) // 64) * 64
        cbuf = torch.zeros(self.world * mb, dtype=torch.int64, device=self.device)
        b, e = blocks[self.rank]
        local = cbuf[self.rank * mb:(self.rank + 1) * mb]
        if self.evaluator is None:
            local[: e - b] = self._pair_counts(b, e)
        else:
            local[: e - b] = torch.as_tensor(self.evaluator.counts(b, e), dtype=torch.int64, device=self.device)
        if self.world > 1:
            _all_gather_inplace(cbuf, local, self.group)
        counts = torch.cat([cbuf[r * mb: r * mb + (be[1] - be[0])] for r, be in enumerate(blocks)])
        return balanced_ranges_device(counts, self.world)

    # ---- evaluation ---------------------------------------------------
    def local_views(self):
        """(value view (m,), grad view (m, 2)) of this rank's all-gather slice."""
        m = self.m
        base = self.rank * 3 * m
        return self.buf[base: base + m], self.buf[base + m: base + 3 * m].view(m, 2)

    def evaluate_local(self):
        """Evaluate this rank's particle range into its all-gather slice."""
        b, e = self.ranges[self.rank]
        ov, og = self.local_views()
        if self.evaluator is not None:
            self.evaluator(b, e, ov[: e - b], og[: e - b])
            return
        from . import _native as N
        from .sphbi import _raise

        import torch

        # the inputs and the all-gather buffer are torch tensors: run on torch's
        # current stream so the call is ordered with whatever produced them
        self.ctx.set_stream(torch.cuda.current_stream(self.device).cuda_stream)
        stats = N.Stats()
        desc = self.table.desc()
        lib = self.ctx.lib
        vp = ctypes.c_void_p
        p = self.particles[b:e]
        tv = vp(self.tri_values.data_ptr()) if self.tri_values is not None else None
        _raise(lib.sphbi_evaluate(self.ctx.handle, ctypes.byref(desc), self.h, e - b, vp(p.data_ptr()),
                                  int(self.triangles.shape[0]), vp(self.triangles.data_ptr()), tv, -1, None, None,
                                  vp(ov.data_ptr()), vp(og.data_ptr()), None, None, ctypes.byref(stats),
                                  N.MEM_DEVICE), "evaluate (shard)")
        self.stats = stats

    def gather(self):
        """All-gather every rank's records; returns (value (n,), grad (n, 2))."""
        import torch

        if self.world > 1:
            m = self.m
            _all_gather_inplace(self.buf, self.buf[self.rank * 3 * m:(self.rank + 1) * 3 * m], self.group)
        m = self.m
        vals, grads = [], []
        for r, (b, e) in enumerate(self.ranges):
            base = r * 3 * m
            vals.append(self.buf[base: base + (e - b)])
            grads.append(self.buf[base + m: base + m + 2 * (e - b)].view(-1, 2))
        return torch.cat(vals), torch.cat(grads)

    def evaluate(self):
        self.evaluate_local()
        return self.gather()


def evaluate_sharded(particles, h, triangles, table, tri_values=None, balance: str = "count", ctx=None,
                     group=None, evaluator=None):
    """One call: shard, evaluate this rank's range on its GPU, all-gather.
    Tensors in, (value (n,), grad (n, 2)) device tensors out."""
    sc = ShardedScene(particles, triangles, table, h, tri_values=tri_values, ctx=ctx, group=group,
                      balance=balance, evaluator=evaluator)
    return sc.evaluate()
