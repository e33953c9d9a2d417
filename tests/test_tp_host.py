"""CPU tests of the head-sharded (tensor-parallel) host logic: shard geometry, the
NCCL unique-id exchange over a world-size-2 gloo group, and the exchange algebra
(per-token head-score partials summed before the f32 head mean; row-parallel o/down
partials summed into the replicated residual) restated on the oracle in numpy."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import pikv_oracle as O
from paper_2602_02579_b200 import ModelConfig
from paper_2602_02579_b200.errors import ConfigError
from paper_2602_02579_b200.model import shard_config


def test_shard_config_geometry():
    cfg = ModelConfig(32, 32, 8, 128, 4096, 14336, 128256, 500000.0)
    for w in (1, 2, 4, 8):
        sc = shard_config(cfg, w)
        assert (sc.n_heads, sc.n_kv_heads) == (32 // w, 8 // w)
        assert sc.hidden_dim == sc.n_heads * sc.head_dim
        assert sc.ffn_dim * w == 14336 and sc.ffn_dim % 128 == 0
    with pytest.raises(ConfigError):
        shard_config(cfg, 3)
    with pytest.raises(ConfigError):
        shard_config(ModelConfig(2, 4, 2, 64, 256, 384, 100), 2)  # 3 ffn blocks


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _uid_worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2602_02579_b200 import tp
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        uid = tp.exchange_unique_id()
    except Exception as e:  # libnccl absent on this host
        uid = repr(e).encode()
    q.put((rank, uid))
    dist.destroy_process_group()


def test_nccl_unique_id_exchange_over_gloo():
    import __graft_entry__
    __graft_entry__.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_uid_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got[0] == got[1] and len(got[0]) == 128


def test_exchange_algebra_on_the_oracle():
    """Sharded scoring + row-parallel projections == unsharded (f64 restatement)."""
    cfg = O.Cfg(1, 4, 2, 8, 32, 64, 50)
    w = O.init_weights(cfg, 3)
    lw = w.layers[0]
    rng = np.random.default_rng(0)
    m, s, W = 3, 20, 2
    x = rng.standard_normal((m, cfg.hidden_dim))
    h = rng.standard_normal((m, cfg.hidden_dim))
    H, Hkv, dk, G = cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.n_heads // cfg.n_kv_heads
    # per-head softmax rows P[h, i, t]; head mean over all H of the per-rank head sums
    P = rng.random((H, m, s))
    P /= P.sum(-1, keepdims=True)
    full = np.float32(P.sum(0) / H)
    hl = H // W
    parts = [P[r * hl:(r + 1) * hl].sum(0) for r in range(W)]
    assert np.array_equal(np.float32(sum(parts) / H), full)
    # o projection: rank r owns heads [r*hl, (r+1)*hl) -> rows of wo
    attn = rng.standard_normal((m, H * dk))
    want = h + attn @ lw.wo.astype(np.float64)
    outs = []
    for r in range(W):
        cols = slice(r * hl * dk, (r + 1) * hl * dk)
        part = attn[:, cols] @ lw.wo[cols].astype(np.float64)
        outs.append(h + part if r == 0 else part)  # rank 0 keeps the residual
    np.testing.assert_allclose(sum(outs), want, rtol=1e-12, atol=1e-12)
    # ffn: rank r owns ffn columns [r*F/W, (r+1)*F/W) of gate/up and rows of down
    F = cfg.ffn_dim
    fl = F // W
    act = O.silu(x @ lw.w_gate) * (x @ lw.w_up)
    want = h + act @ lw.w_down.astype(np.float64)
    outs = []
    for r in range(W):
        c = slice(r * fl, (r + 1) * fl)
        a = O.silu(x @ lw.w_gate[:, c]) * (x @ lw.w_up[:, c])
        part = a @ lw.w_down[c].astype(np.float64)
        outs.append(h + part if r == 0 else part)
    np.testing.assert_allclose(sum(outs), want, rtol=1e-10, atol=1e-10)
    # KV heads: rank r's q heads read only its own KV groups
    for r in range(W):
        for j in range(hl):
            assert (r * hl + j) // G in range(r * (Hkv // W), (r + 1) * (Hkv // W))


def test_token_parallel_row_partition():
    """pkv_recompute_rows' unit assignment (tp.rows_share): 128/G-row attention units,
    unit u on rank u mod W -- every selected row on exactly one rank, in ascending order
    per rank, balanced to one unit."""
    import numpy as np

    from paper_2602_02579_b200 import tp
    for k, group, world in [(6554, 4, 8), (6554, 4, 2), (410, 2, 4), (5, 2, 3), (0, 4, 2), (128, 1, 2)]:
        parts = [tp.rows_share(k, group, world, r) for r in range(world)]
        allr = np.sort(np.concatenate(parts)) if k else np.zeros(0)
        assert np.array_equal(allr, np.arange(k))
        for p in parts:
            assert np.all(np.diff(p) > 0)
        T = max(1, 128 // group)
        assert max(len(p) for p in parts) - min(len(p) for p in parts) <= T
