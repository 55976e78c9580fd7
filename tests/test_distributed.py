"""CPU tier: the multi-GPU host logic (particle sharding + all-gather of the
per-particle records) on world_size 2 with the gloo backend. The per-shard
evaluation is the CPU oracle standing in for the device kernel; the result
must be BITWISE identical to the single-process evaluation (each particle is
reduced entirely on one rank, in a fixed order)."""
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


def _oracle_evaluator(O, k):
    def ev(p, h, t, tab, vals, pairs):
        pp, pt = pairs
        st, v, g = OL.oracle_scene_sums(O, p, t, vals, k.coefficients, k.normalization, h, pp, pt, threads=2)
        assert st == 0
        return v, g
    return ev


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2507_21686_b200 import scenes, shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc = scenes.cfg2(T=64, per_tri=16, linear_field=True)
    O = OL.oracle()
    k = sc.kernels[0]
    counts = np.bincount(sc.pairs[0], minlength=sc.particles.shape[0])
    ranges = shard.balanced_ranges(counts, world)
    full = shard.evaluate_sharded(sc.particles, sc.h, sc.triangles, None, rank, world, tri_values=sc.values,
                                  pairs=sc.pairs, ranges=ranges, evaluator=_oracle_evaluator(O, k))
    if rank == 0:
        q.put(full)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_gather_is_bitwise_identical():
    import torch.multiprocessing as mp
    from paper_2507_21686_b200 import scenes
    world = 2
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    port = _free_port()
    procs = [ctxm.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    full = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sc = scenes.cfg2(T=64, per_tri=16, linear_field=True)
    k = sc.kernels[0]
    O = OL.oracle()
    st, v, g = OL.oracle_scene_sums(O, sc.particles, sc.triangles, sc.values, k.coefficients, k.normalization, sc.h,
                                    sc.pairs[0], sc.pairs[1], threads=2)
    single = np.concatenate([v[:, None], g], axis=1)
    assert np.array_equal(full, single)


def test_ranges():
    from paper_2507_21686_b200 import shard
    r = shard.shard_ranges(10, 3)
    assert r == [(0, 4), (4, 7), (7, 10)]
    counts = np.array([1, 1, 1, 1, 100, 1, 1, 1])
    b = shard.balanced_ranges(counts, 2)
    assert b[0][0] == 0 and b[-1][1] == 8 and b[0][1] == b[1][0]
    pp, pt = shard.shard_pairs((np.array([0, 1, 2, 3]), np.array([5, 6, 7, 8])), 1, 3)
    assert list(pp) == [0, 1] and list(pt) == [6, 7]
