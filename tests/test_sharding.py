"""Multi-process (gloo, world_size 2, CPU) tests of the head-sharding host logic
(SURVEY.md §8e): partition coverage, shard/gather round trip, max-over-ranks
timing reduction, and the oracle computed per shard equals the oracle on the
whole tensor (heads are independent, tiled.cpp:146-147)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_01960_b200.sharding import gather_heads, head_range, max_over_ranks, shard_heads


def test_head_range_partitions_exactly():
    for H in (1, 2, 7, 8, 64):
        for world in (1, 2, 3, 4, 8):
            if world > H:
                continue
            covered = []
            for r in range(world):
                h0, h1 = head_range(H, world, r)
                assert h1 > h0
                covered.extend(range(h0, h1))
            assert covered == list(range(H))
    with pytest.raises(ValueError):
        head_range(8, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O
        B, H, S, D = 2, 4, 24, 8
        qf, kf, vf = (torch.from_numpy(x) for x in O.make_input((B, H, S, D), O.F32, 5))
        ql, kl, vl = (shard_heads(x, world, rank) for x in (qf, kf, vf))
        h0, h1 = head_range(H, world, rank)
        assert ql.shape == (B, h1 - h0, S, D) and ql.is_contiguous()
        # per-shard compute (oracle stands in for the kernel on CPU)
        ol = torch.from_numpy(O.sdpa_reference(ql.numpy(), kl.numpy(), vl.numpy())["o"])
        full = gather_heads(ol, world)
        want = O.sdpa_reference(qf.numpy(), kf.numpy(), vf.numpy())["o"]
        ok_gather = bool(np.array_equal(full.numpy(), want))
        t = max_over_ranks(1.0 + rank)
        q.put((rank, ok_gather, t))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_shard_compute_gather():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(world))
    assert all(ok for _, ok, _ in res)
    assert all(t == float(world) for _, _, t in res)  # max over ranks
