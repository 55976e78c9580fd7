"""GPU tier: the particle-sharded multi-GPU path (paper_2507_21686_b200/shard.py)
with the product kernels. Two processes (world size 2) share the one B200 of
the test box: each runs the device count pass on its block, the equal-pair
cut, sphbi_evaluate on its particle range straight into its slice of the
all-gather buffer, and the all-gather. NCCL refuses two ranks on one device,
so the ranks talk over gloo here (the buffer is staged through host memory
for the collective only; on a multi-GPU box it is an in-place NCCL
all-gather). The gathered result must be BITWISE identical to one
single-process sphbi_evaluate over all particles, for both cut policies."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scene():
    from paper_2507_21686_b200 import scenes
    sc = scenes.cfg5(n_particles=200_000, n_discs=12, target_tris=40_000, domain=16.0)
    vals = np.random.default_rng(7).standard_normal((sc.triangles.shape[0], 3))
    return sc, vals


def _worker(rank, world, port, q, balance):
    import torch
    import torch.distributed as dist
    from paper_2507_21686_b200 import shard
    from paper_2507_21686_b200 import sphbi as S
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc, vals = _scene()
    k = sc.kernels[0]
    table = S.table1_terms(S.PolyKernel(list(k.coefficients), k.normalization))
    dev = torch.device("cuda", 0)
    P = torch.from_numpy(sc.particles).to(dev)
    T = torch.from_numpy(sc.triangles).to(dev)
    V = torch.from_numpy(vals).to(dev)
    s = shard.ShardedScene(P, T, table, sc.h, tri_values=V, balance=balance)
    v, g = s.evaluate()
    if rank == 0:
        q.put((v.cpu().numpy(), g.cpu().numpy(), s.ranges, int(s.stats.n_pairs)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("balance", ["pairs", "count"])
def test_two_ranks_on_one_gpu_bitwise_equal_single_process(balance):
    import torch.multiprocessing as mp
    from paper_2507_21686_b200 import sphbi as S
    world = 2
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    port = _free_port()
    procs = [ctxm.Process(target=_worker, args=(r, world, port, q, balance)) for r in range(world)]
    for p in procs:
        p.start()
    v, g, ranges, n0 = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    sc, vals = _scene()
    k = sc.kernels[0]
    table = S.table1_terms(S.PolyKernel(list(k.coefficients), k.normalization))
    v1, g1, st, plist = S.evaluate(sc.particles, sc.h, sc.triangles, table, tri_values=vals, return_pairs=True)
    assert np.array_equal(v, v1) and np.array_equal(g, g1)
    assert ranges[0][0] == 0 and ranges[1][1] == sc.particles.shape[0] and ranges[0][1] == ranges[1][0]
    b, e = ranges[0]
    assert n0 == int(((plist[:, 0] >= b) & (plist[:, 0] < e)).sum())
    if balance == "pairs":
        counts = np.bincount(plist[:, 0], minlength=sc.particles.shape[0])
        from paper_2507_21686_b200 import shard
        assert ranges == shard.balanced_ranges(counts, world)


def test_pair_counts_match_the_pair_list():
    """sphbi_pair_counts (the device count pass) equals the per-particle counts
    of the found pair list, on device and host memory."""
    import ctypes
    import torch
    from paper_2507_21686_b200 import _native as N
    from paper_2507_21686_b200 import sphbi as S
    sc, _ = _scene()
    k = sc.kernels[0]
    table = S.table1_terms(S.PolyKernel(list(k.coefficients), k.normalization))
    _, _, st, plist = S.evaluate(sc.particles, sc.h, sc.triangles, table, return_pairs=True)
    want = np.bincount(plist[:, 0], minlength=sc.particles.shape[0])
    ctx = S.Context(0)
    n, T = sc.particles.shape[0], sc.triangles.shape[0]
    host = np.zeros(n, dtype=np.int64)
    tot = ctypes.c_int64(0)
    S._raise(ctx.lib.sphbi_pair_counts(ctx.handle, sc.h, n, sc.particles.ctypes.data, T, sc.triangles.ctypes.data,
                                       host.ctypes.data, ctypes.byref(tot), None, N.MEM_HOST), "pair_counts")
    assert np.array_equal(host, want) and tot.value == plist.shape[0]
    dev = torch.device("cuda", 0)
    P = torch.from_numpy(sc.particles).to(dev)
    Tr = torch.from_numpy(sc.triangles).to(dev)
    out = torch.zeros(n, dtype=torch.int64, device=dev)
    S._raise(ctx.lib.sphbi_pair_counts(ctx.handle, sc.h, n, ctypes.c_void_p(P.data_ptr()), T,
                                       ctypes.c_void_p(Tr.data_ptr()), ctypes.c_void_p(out.data_ptr()), None, None,
                                       N.MEM_DEVICE), "pair_counts")
    assert np.array_equal(out.cpu().numpy(), want)
    ctx.close()
