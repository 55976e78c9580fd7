"""CPU tier: the multi-GPU host logic of paper_2507_21686_b200/shard.py
(particle shards, sharded count pass + equal-pair cuts, in-place all-gather of
the per-particle records) on world_size 2 with the gloo backend. The per-shard
evaluator is the CPU oracle standing in for the device call (the GPU variant
is tests/test_gpu_sharded.py). The gathered result must be BITWISE identical
to the single-process evaluation: each particle is reduced entirely on one
rank, in ascending triangle order."""
import os
import socket

import numpy as np
import pytest

import oracle_lib as OL


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleShardEvaluator:
    """Evaluates particles [b, e) of a scene with the CPU oracle over the exact
    pair list (the device path's cell list finds the same list)."""

    def __init__(self, sc):
        self.sc = sc
        self.O = OL.oracle()
        self.pairs = OL.cpu_pairs_grid(self.O, sc.particles, sc.triangles, sc.h)

    def counts(self, b, e):
        return np.bincount(self.pairs[:, 0], minlength=self.sc.particles.shape[0])[b:e]

    def __call__(self, b, e, ov, og):
        import torch
        sc = self.sc
        k = sc.kernels[0]
        m = (self.pairs[:, 0] >= b) & (self.pairs[:, 0] < e)
        pp, pt = self.pairs[m, 0] - b, self.pairs[m, 1]
        st, v, g = OL.oracle_scene_sums(self.O, sc.particles[b:e], sc.triangles, sc.values, k.coefficients,
                                        k.normalization, sc.h, pp, pt, threads=2)
        assert st == 0
        ov.copy_(torch.from_numpy(v))
        og.copy_(torch.from_numpy(g))


def _scene():
    from paper_2507_21686_b200 import scenes
    sc = scenes.cfg2(T=64, per_tri=16, linear_field=True)
    # cell-list pairing over a small cfg2 scene: ragged pair counts per particle
    sc.pairs = None
    return sc


def _worker(rank, world, port, q, balance):
    import torch
    import torch.distributed as dist
    from paper_2507_21686_b200 import shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc = _scene()
    ev = OracleShardEvaluator(sc)
    P = torch.from_numpy(sc.particles)
    T = torch.from_numpy(sc.triangles)
    s = shard.ShardedScene(P, T, None, sc.h, balance=balance, evaluator=ev)
    v, g = s.evaluate()
    if rank == 0:
        q.put((v.numpy().copy(), g.numpy().copy(), s.ranges))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("balance", ["count", "pairs"])
def test_sharded_gather_is_bitwise_identical(balance):
    import torch.multiprocessing as mp
    world = 2
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    port = _free_port()
    procs = [ctxm.Process(target=_worker, args=(r, world, port, q, balance)) for r in range(world)]
    for p in procs:
        p.start()
    v, g, ranges = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sc = _scene()
    ev = OracleShardEvaluator(sc)
    k = sc.kernels[0]
    st, v1, g1 = OL.oracle_scene_sums(ev.O, sc.particles, sc.triangles, sc.values, k.coefficients,
                                      k.normalization, sc.h, ev.pairs[:, 0], ev.pairs[:, 1], threads=2)
    assert np.array_equal(v, v1) and np.array_equal(g, g1)
    assert ranges[0][0] == 0 and ranges[-1][1] == sc.particles.shape[0] and ranges[0][1] == ranges[1][0]
    if balance == "pairs":
        counts = np.bincount(ev.pairs[:, 0], minlength=sc.particles.shape[0])
        from paper_2507_21686_b200 import shard
        assert ranges == shard.balanced_ranges(counts, world)
        work = [counts[b:e].sum() for b, e in ranges]
        assert abs(work[0] - work[1]) <= counts.max()


def test_ranges():
    import torch
    from paper_2507_21686_b200 import shard
    r = shard.shard_ranges(10, 3)
    assert r == [(0, 4), (4, 7), (7, 10)]
    counts = np.array([1, 1, 1, 1, 100, 1, 1, 1])
    b = shard.balanced_ranges(counts, 2)
    assert b[0][0] == 0 and b[-1][1] == 8 and b[0][1] == b[1][0]
    pp, pt = shard.shard_pairs((np.array([0, 1, 2, 3]), np.array([5, 6, 7, 8])), 1, 3)
    assert list(pp) == [0, 1] and list(pt) == [6, 7]
    rng = np.random.default_rng(3)
    for world in (1, 2, 3, 8):
        for n in (0, 1, 7, 1000):
            c = rng.integers(0, 50, n) * (rng.random(n) < 0.3)
            assert shard.balanced_ranges_device(torch.from_numpy(c), world) == shard.balanced_ranges(c, world)
