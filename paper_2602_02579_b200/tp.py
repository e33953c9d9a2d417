"""Head-sharded (tensor-parallel) prefill of one long request -- SURVEY §8(e), config C3.

Rank r of W owns KV heads [r*Hkv/W, (r+1)*Hkv/W) (with their query heads), the
matching slice of the chunk store and paged cache, and ffn blocks
[r*Fp/W, (r+1)*Fp/W).  Per layer the ranks exchange (in-place sums inside the C++
stage loops, include/pkv.h "Head-sharded prefill"):

* the per-(query row, context token) head-score partials of the scoring pass,
  before the f32 head mean of reference model.py:294, 303-307 -- so every rank
  fuses the same per-layer scores and selects the same tokens (the per-token score
  all-reduce before the global top-k);
* the row-parallel o / down projection outputs of the narrow passes ([m][D] fp32)
  and of Stage II ([k][D] fp32).

Alternative (``DeviceModel.rows``, include/pkv.h pkv_recompute_rows): token-parallel
Stage II -- every rank holds the full model and cache, the scoring pass is replicated,
and each rank repairs its attention units of the selected rows with one all-gather of
fresh cache entries per layer instead of the two [k][D] fp32 all-reduces.

Two communicator back ends: NCCL (one process per GPU, NVLink / NVSwitch; the
unique id travels over the torch.distributed process group) and an in-process
group of W threads sharing one GPU, which runs the sharded math end to end on a
single device (tests).
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from . import _lib
from .chunkstore import ChunkKV
from .model import DeviceModel, shard_config

__all__ = ["Comm", "local_group", "nccl_comm", "shard_chunks", "shard_config", "run_ranks", "rows_share"]


class Comm:
    """Owning wrapper of one rank's pkv_comm handle."""

    def __init__(self, handle: ctypes.c_void_p, rank: int, world: int):
        self.handle = handle
        self.rank, self.world = rank, world

    @property
    def as_parameter(self):
        return self.handle

    def allreduce_(self, tensor, stream=None) -> None:
        """In-place sum of a contiguous CUDA tensor (f32, f64 or bf16) over the ranks."""
        import torch
        dt = {torch.float32: _lib.PKV_DT_F32, torch.float64: _lib.PKV_DT_F64,
              torch.bfloat16: _lib.PKV_DT_BF16}[tensor.dtype]
        _lib.check(_lib.load().pkv_comm_allreduce(self.handle, tensor.data_ptr(), tensor.numel(), dt,
                                                  _lib.stream_ptr(torch, stream)))

    def close(self) -> None:
        if self.handle:
            _lib.load().pkv_comm_destroy(self.handle)
            self.handle = None


def local_group(world: int) -> list:
    """W rank communicators of one in-process group (all on the current device)."""
    arr = (ctypes.c_void_p * world)()
    _lib.check(_lib.load().pkv_comm_create_local(world, arr))
    return [Comm(ctypes.c_void_p(arr[r]), r, world) for r in range(world)]


def _nccl_lib_path() -> str | None:
    try:
        import nvidia.nccl
        for base in list(getattr(nvidia.nccl, "__path__", [])):
            p = Path(base) / "lib" / "libnccl.so.2"
            if p.exists():
                return str(p)
    except ImportError:
        pass
    return None


def nccl_unique_id() -> bytes:
    lib = _lib.load()
    path = os.environ.get("PKV_NCCL_LIB") or _nccl_lib_path()
    _lib.check(lib.pkv_nccl_load(path.encode() if path else None))
    buf = ctypes.create_string_buffer(128)
    _lib.check(lib.pkv_comm_unique_id(buf))
    return buf.raw


def exchange_unique_id(group=None) -> bytes:
    """Rank 0 creates the NCCL unique id; broadcast over the torch.distributed group."""
    import torch.distributed as dist
    obj = [nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    if not isinstance(obj[0], bytes) or len(obj[0]) != 128:
        raise RuntimeError("bad NCCL unique id from rank 0")
    return obj[0]


def nccl_comm(group=None) -> Comm:
    """NCCL communicator over the ranks of a torch.distributed group (one GPU per
    process, current device set)."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    uid = exchange_unique_id(group)
    lib = _lib.load()
    path = os.environ.get("PKV_NCCL_LIB") or _nccl_lib_path()
    _lib.check(lib.pkv_nccl_load(path.encode() if path else None))
    h = ctypes.c_void_p()
    _lib.check(lib.pkv_comm_create_nccl(uid, rank, world, ctypes.byref(h)))
    return Comm(h, rank, world)


def shard_chunks(chunks, rank: int, world: int) -> list:
    """Rank r's KV-head slice of device chunks ([L][t][Hkv][dkp] -> [L][t][Hkv/W][dkp])."""
    out = []
    for c in chunks:
        k, v = c._k_dev, c._v_dev
        hkv = k.shape[2]
        if hkv % world:
            raise ValueError(f"{hkv} KV heads do not split over {world} ranks")
        kl = hkv // world
        out.append(ChunkKV.from_device(c.chunk_id, c.config_fingerprint, c.token_ids,
                                       k[:, :, rank * kl:(rank + 1) * kl].contiguous(),
                                       v[:, :, rank * kl:(rank + 1) * kl].contiguous(), c._dk))
    return out


def rows_share(k: int, group: int, world: int, rank: int):
    """Global selection rows the rank repairs under token-parallel Stage II (include/pkv.h
    pkv_recompute_rows): attention units of T = 128 / group consecutive rows, unit u on rank
    u mod world."""
    import numpy as np
    T = max(1, 128 // max(1, group))
    units = range(rank, -(-k // T), world)
    return np.concatenate([np.arange(u * T, min(k, (u + 1) * T)) for u in units]) if len(units) else \
        np.zeros(0, dtype=np.int64)


def shard_model(dm: DeviceModel, comms: list) -> list:
    return [dm.shard(c.rank, c.world, c.handle) for c in comms]


def run_ranks(fns: list) -> list:
    """Run one callable per rank in its own host thread (in-process group); each
    thread gets its own CUDA stream.  Re-raises the first failure."""
    import torch
    results, errors = [None] * len(fns), [None] * len(fns)
    dev = torch.cuda.current_device()

    def body(r):
        try:
            torch.cuda.set_device(dev)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                results[r] = fns[r]()
            s.synchronize()
        except BaseException as e:  # noqa: BLE001 -- surfaced below
            errors[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(len(fns))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in errors:
        if e is not None:
            raise e
    return results
