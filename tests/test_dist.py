"""Multi-process (world_size 2, gloo, CPU) tests of the batch-sharded path:
FWD/BWI shards concatenate to the full-batch result with no communication,
and the BWW partial dG of the shards, summed by the allreduce, equals the
full-batch dG.  The per-rank compute here is the oracle (the GPU kernels are
covered by the -m gpu suite); what is tested is the sharding + exchange logic
the bench runs over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1911_10175_b200.dist import GradAllreduce, shard_batch, shard_range


def test_shard_range_partitions_the_batch():
    for n in (1, 2, 5, 16, 32, 33, 256):
        for w in (1, 2, 3, 4, 8):
            spans = [shard_range(n, w, r) for r in range(w)]
            assert spans[0][0] == 0
            assert sum(c for _, c in spans) == n
            for (s0, c0), (s1, _) in zip(spans, spans[1:]):
                assert s1 == s0 + c0
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O
        sh = O.shape_make(6, 16, 32, 7, 9, 3, 3, 1, 1)
        N, C, K, H, W, R, S = sh[:7]
        hp, wp = O.out_hw(sh)
        D = O.gen_sparse(N, C, H, W, 0.5, 1)
        G = O.gen_sparse(K, C, S, R, 0.0, 2)
        dY = O.gen_sparse(N, K, hp, wp, 0.5, 3)
        start, cnt = shard_range(N, world, rank)
        shs = (cnt,) + tuple(sh[1:])
        # FWD / BWI: per-shard, no communication
        y = O.dense(0, shs, shard_batch(D, world, rank), G)
        dd = O.dense(1, shs, shard_batch(dY, world, rank), G)
        # BWW: partial over the shard, then allreduce(sum)
        g = torch.from_numpy(O.dense(2, shs, shard_batch(D, world, rank), shard_batch(dY, world, rank)))
        ar = GradAllreduce()
        ar.submit(g)
        ar.wait()
        q.put((rank, start, y, dd, g.numpy()))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_passes_match_full_batch():
    import oracle as O
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sh = O.shape_make(6, 16, 32, 7, 9, 3, 3, 1, 1)
    N, C, K, H, W, R, S = sh[:7]
    hp, wp = O.out_hw(sh)
    D = O.gen_sparse(N, C, H, W, 0.5, 1)
    G = O.gen_sparse(K, C, S, R, 0.0, 2)
    dY = O.gen_sparse(N, K, hp, wp, 0.5, 3)
    y_full = np.concatenate([r[2] for r in res])
    dd_full = np.concatenate([r[3] for r in res])
    assert np.array_equal(y_full, O.dense(0, sh, D, G))          # per-image independent: bitwise
    assert np.array_equal(dd_full, O.dense(1, sh, dY, G))
    ref = O.dense(2, sh, D, dY)
    for r in res:  # every rank holds the same reduced dG
        assert O.max_abs_rel(r[4], ref) <= 1e-6
    assert np.array_equal(res[0][4], res[1][4])


def _plan_worker(rank, world, port, q):
    """The product's sharding code (dist.ShardPlan + the product's blocked
    pack/unpack + GradAllreduce) driving the per-rank compute, which on CPU is
    the 64-bit oracle (the GPU kernels are the -m gpu suite's)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O
        import paper_1911_10175_b200 as sp
        from paper_1911_10175_b200.dist import ShardPlan
        V = 16
        from paper_1911_10175_b200.workloads import PlainShape
        gsh = PlainShape(O.shape_make(19, 32, 16, 6, 7, 3, 3, 1, 1))
        N, C, K, H, W = gsh.N, gsh.C, gsh.K, gsh.H, gsh.W
        hp, wp = gsh.out_h(), gsh.out_w()
        D = O.gen_sparse(N, C, H, W, 0.6, 11)
        G = O.gen_sparse(K, C, 3, 3, 0.0, 12)
        dY = O.gen_sparse(N, K, hp, wp, 0.5, 13)
        plan = ShardPlan(N, world, rank)
        sh = plan.shape(gsh)
        # the global ActNCHWc tensors, sliced without copies to this rank's images
        bD = plan.slice_nchwc(sp.pack_act_nchwc(D, V))
        bY = plan.slice_nchwc(sp.pack_act_nchwc(dY, V))
        assert bD.n == plan.count and np.shares_memory(bD.data, bD.data)
        Dl, Yl = sp.unpack(bD), sp.unpack(bY)
        assert np.array_equal(Dl, plan.slice_plain(D)) and np.array_equal(Yl, plan.slice_plain(dY))
        # the rank's own ActCHWNn pack (ragged lane block zero-filled)
        bDc = sp.pack_act_chwnn(Dl, V)
        assert np.array_equal(sp.unpack(bDc), Dl)
        y = O.dense(0, sh.astuple(), Dl, G)
        dd = O.dense(1, sh.astuple(), Yl, G)
        g = torch.from_numpy(O.dense(2, sh.astuple(), sp.unpack(bDc), Yl))
        ar = GradAllreduce()
        ar.submit(g)
        ar.wait()
        q.put((rank, plan.start, plan.count, y, dd, g.numpy(), plan.global_flops([sh])))
    finally:
        dist.destroy_process_group()


def test_two_rank_shardplan_step_matches_full_batch():
    import oracle as O
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_plan_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [(r[1], r[2]) for r in res] == [(0, 10), (10, 9)]
    sh = O.shape_make(19, 32, 16, 6, 7, 3, 3, 1, 1)
    N, C, K, H, W, R, S = sh[:7]
    hp, wp = O.out_hw(sh)
    D = O.gen_sparse(N, C, H, W, 0.6, 11)
    G = O.gen_sparse(K, C, 3, 3, 0.0, 12)
    dY = O.gen_sparse(N, K, hp, wp, 0.5, 13)
    assert np.array_equal(np.concatenate([r[3] for r in res]), O.dense(0, sh, D, G))
    assert np.array_equal(np.concatenate([r[4] for r in res]), O.dense(1, sh, dY, G))
    ref = O.dense(2, sh, D, dY)
    for r in res:
        assert O.max_abs_rel(r[5], ref) <= 1e-6
        assert r[6] == 2 * N * K * C * R * S * hp * wp  # whole-job flops from every rank
