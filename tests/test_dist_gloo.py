"""world_size-2 gloo test of the request-parallel plumbing (CPU, two processes)."""

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2602_02579_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_requests, q):
    import numpy as np
    import torch.distributed as dist

    from oracle import pikv_oracle as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = D.shard_requests(n_requests, rank, world)
    # each rank scores its own requests with the oracle; no data-path collective
    cfg = O.Cfg(2, 2, 1, 4, 8, 16, 50)
    w = O.init_weights(cfg, 42)
    sels = {}
    for rid in mine:
        rng = np.random.default_rng(rid)
        units = [rng.integers(0, 50, 6).tolist() for _ in range(3)]
        cache = O.stitch([O.make_chunk(w, cfg, u) for u in units], cfg)
        _, fused = O.prophet_scores(w, cfg, cache, rng.integers(0, 50, 4).tolist())
        sels[rid] = O.select(fused, 0.3)[0]
    t = D.max_over_ranks(float(rank + 1))
    got = D.gather_results(sels)
    if rank == 0:
        q.put((t, got))
    dist.destroy_process_group()


def test_request_sharding_covers_every_request_once():
    for world in (1, 2, 3, 8):
        seen = sorted(i for r in range(world) for i in D.shard_requests(10, r, world))
        assert seen == list(range(10))
    with pytest.raises(ValueError):
        D.shard_requests(4, 2, 2)


def test_two_rank_gloo_request_parallel():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 5, q)) for r in range(2)]
    for p in procs:
        p.start()
    t, got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert t == 2.0  # max over ranks
    merged = {}
    for d in got:
        merged.update(d)
    assert sorted(merged) == list(range(5))
