"""Stage II repair and query finalisation on the GPU.

Drop-in for reference recompute.py (RecomputePlan 35-40, recompute_selected
43-82, FinalizeResult 98-102, finalize_query 105-125, selection_digest 153-155,
run_strategy 173-253).  Stage II runs through ``pkv_recompute``: per layer a
tcgen05 QKV GEMM whose epilogue rotates q/k and scatters the fresh K/V into the
paged cache, then the sparse-query tcgen05 attention over the updated layer,
then o / gate-up(SiLU) / down GEMMs with fp32 residual epilogues.
"""

from __future__ import annotations

import ctypes
import hashlib
import json
from dataclasses import dataclass

import numpy as np

from . import _lib
from .chunkstore import assemble, mark_finalized
from .errors import ArgumentError, ConfigError, InputError, NumericsError, StateError
from .model import FlopTally, KVCache, ModelConfig, bill_query_pass, bill_repair, resolve_device_model
from .selection import (STRATEGIES, SelectionResult, ValueScores, check_tokens, run_query_pass,
                        score_cacheblend_l1, score_epic, score_kvshare_l1, score_prophet, score_random, select_top_p,
                        workspace)


@dataclass
class RecomputePlan:
    selection: SelectionResult
    # the reference's stale-peer ablation (recompute.py:60-78) is not on the B200 path
    stale_peers: bool = False


def recompute_selected(weights, config: ModelConfig, cache, plan: RecomputePlan,
                       tally: FlopTally | None = None):
    """Repair the cache in place at the planned token set; returns the same object."""
    torch = _lib.require_cuda()
    if cache.finalized:
        raise StateError("cannot repair a finalized cache")
    if cache.recomputed.any():
        raise StateError("cache was already repaired once")
    if plan.stale_peers:
        raise ConfigError("stale_peers ablation is not implemented on the B200 path")
    sel = np.asarray(plan.selection.indices, dtype=np.int64)
    if sel.size == 0:
        return cache
    if not np.all(np.diff(sel) > 0):
        raise ArgumentError("selection indices must be strictly ascending")
    if sel[0] < 0 or sel[-1] >= cache.context_length:
        raise InputError("replacement index out of range")
    dm = resolve_device_model(weights, config)
    k = int(sel.size)
    d_sel = plan.selection._dev_idx
    if d_sel is None or int(d_sel.numel()) != k:
        d_sel = torch.from_numpy(sel.astype(np.int32)).to(cache.device)
    # the cache holds this rank's KV heads (all of them unless the model is head-sharded)
    L, Hkv, dk = config.n_layers, cache.config.n_kv_heads, config.head_dim
    tap_k = tap_v = None
    if cache.fp32_taps:
        tap_k = torch.empty((L, k, Hkv, dk), dtype=torch.float32, device=cache.device)
        tap_v = torch.empty_like(tap_k)
    lib = _lib.load()
    query = getattr(cache, "_pending_query", None)
    cache._pending_query = None
    if getattr(dm, "rows_comm", None) is not None:
        if tap_k is not None:
            raise ConfigError("fp32 taps are not available with the token-parallel Stage II")
        _recompute_rows(lib, dm, config, cache, d_sel, k, query if _fused_final() else None)
    elif query is not None and _fused_final():
        _recompute_with_query(lib, dm, config, cache, d_sel, k, query, tap_k, tap_v)
    else:
        _recompute(lib, dm, cache, d_sel, k, tap_k, tap_v, L)
    cache.recomputed[:, sel] = True
    if tap_k is not None:
        for li in range(L):
            cache.add_tap(li, sel, tap_k[li], tap_v[li])
    if cache.access_log is not None:
        for li in range(L):  # each layer writes its fresh K/V before its attention reads them
            cache.access_log.append(("write", li))
            cache.access_log.append(("read", li))
    bill_repair(tally, config, cache.context_length, k)
    return cache


def _fused_final() -> bool:
    """The query rows of finalize_query ride along Stage II (pkv_recompute_query) when the
    scoring pass left its query on the cache; PKV_FUSED_FINAL=0 keeps the separate
    fp32-faithful query pass."""
    import os
    return os.environ.get("PKV_FUSED_FINAL", "1") == "1"


def _recompute_with_query(lib, dm, config, cache, d_sel, k, query, tap_k, tap_v) -> None:
    """Stage II over the selection plus the m query rows at positions s..s+m-1: the query's
    first-token logits and fresh K/V are kept on the cache for finalize_query (reference
    recompute.py:105-125) of the same tokens, which then runs no pass of its own."""
    torch = _lib.require_cuda()
    m = int(query.shape[0])
    cache.ensure_query_room(m)
    L, Hkv, dk = config.n_layers, cache.config.n_kv_heads, config.head_dim
    fk = torch.empty((L, m, Hkv, dk), dtype=torch.float32, device=cache.device)
    fv = torch.empty_like(fk)
    logits = torch.empty(config.vocab_size, dtype=torch.float32, device=cache.device)
    d_q = torch.from_numpy(query).to(cache.device)
    ws = workspace(lib.pkv_recompute_query_workspace(dm.handle, k, m), "rc")
    cache._final_follow = None
    _lib.check(lib.pkv_recompute_query(dm.handle, ctypes.byref(cache.c_cache), d_sel.data_ptr(), k, d_q.data_ptr(), m,
                                       tap_k.data_ptr() if tap_k is not None else None,
                                       tap_v.data_ptr() if tap_v is not None else None, fk.data_ptr(), fv.data_ptr(),
                                       logits.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr(torch)))
    cache._fused_final = (query, logits, fk, fv)


def _recompute_rows(lib, dm, config, cache, d_sel, k, query) -> None:
    """Token-parallel Stage II (pkv_recompute_rows) on this rank's share of the selection,
    with the query rows riding along when finalize_query will follow (every rank)."""
    torch = _lib.require_cuda()
    comm = dm.rows_comm
    m = int(query.shape[0]) if query is not None else 0
    logits = d_q = None
    if m:
        cache.ensure_query_room(m)
        logits = torch.empty(config.vocab_size, dtype=torch.float32, device=cache.device)
        d_q = torch.from_numpy(query).to(cache.device)
    ws = workspace(lib.pkv_recompute_rows_workspace(dm.handle, k, m, comm.world), "rc")
    cache._final_follow = None
    _lib.check(lib.pkv_recompute_rows(dm.handle, ctypes.byref(cache.c_cache), d_sel.data_ptr(), k,
                                      d_q.data_ptr() if m else None, m, comm.handle,
                                      logits.data_ptr() if m else None, ws.data_ptr(), ws.numel(),
                                      _lib.stream_ptr(torch)))
    if m:
        # the query's fresh K/V for the KVCache views: read back from the pool (fp16 entries)
        s, L, Hkv, dk = cache.context_length, config.n_layers, cache.config.n_kv_heads, config.head_dim
        fk = (cache.k_pool[:, :, s:s + m, :dk].float() + cache.k2_pool[:, :, s:s + m, :dk].float()).permute(0, 2, 1, 3)
        fv = cache.v_pool[:, :, s:s + m, :dk].float().permute(0, 2, 1, 3)
        cache._fused_final = (query, logits, fk.contiguous(), fv.contiguous())


def _recompute(lib, dm, cache, d_sel, k, tap_k, tap_v, L) -> None:
    torch = _lib.require_cuda()
    ws = workspace(lib.pkv_recompute_workspace(dm.handle, k), "rc")
    c_rc = cache.c_cache
    if _final_overlap(dm):
        # finalize_query may follow Stage II layer by layer on its own stream: done[l] is
        # recorded once layer l's K/V are final (include/pkv.h layer_done)
        pre = torch.cuda.Event()
        pre.record()
        done = [torch.cuda.Event() for _ in range(L)]
        for e in done:
            e.record()  # creates the cudaEvent_t (torch creates it lazily)
        arr = (_lib.c_vp * L)(*[e.cuda_event for e in done])
        c_rc = _lib.Cache.from_buffer_copy(cache.c_cache)
        c_rc.layer_done = arr
        c_fin = _lib.Cache.from_buffer_copy(cache.c_cache)
        c_fin.layer_ready = arr
        cache._final_follow = (pre, done, arr, c_fin)
    _lib.check(lib.pkv_recompute(dm.handle, ctypes.byref(c_rc), d_sel.data_ptr(), k,
                                 tap_k.data_ptr() if tap_k is not None else None,
                                 tap_v.data_ptr() if tap_v is not None else None, ws.data_ptr(), ws.numel(),
                                 _lib.stream_ptr(torch)))


@dataclass
class FinalizeResult:
    cache: KVCache               # context + query, ready for decoding
    first_logits: np.ndarray     # [vocab] at the last query position
    rows: list | None


def _final_overlap(dm) -> bool:
    """finalize_query follows Stage II layer by layer on a side stream (unsharded models:
    collectives of two streams on one communicator could interleave differently per rank)."""
    import os
    return os.environ.get("PKV_FINAL_OVERLAP", "1") == "1" and getattr(dm, "tp_world", 1) == 1


def finalize_query(weights, config: ModelConfig, cache, query_tokens, capture_attn: bool = False,
                   tally: FlopTally | None = None) -> FinalizeResult:
    """Compute the query over the (repaired) cache and append its K/V entries.
    One-shot per cache (reference recompute.py:105-125).  With capture_attn the result
    carries the head-averaged attention rows [m, s+m] of every layer (model.py:386-398).
    Raises NumericsError for a non-finite value in the Stage-II repair or the logits."""
    torch = _lib.require_cuda()
    dm = resolve_device_model(weights, config)
    ids = check_tokens(query_tokens, config)
    if capture_attn and getattr(dm, "tp_world", 1) > 1:
        raise ConfigError("capture_attn is not supported on a head-sharded model")
    mark_finalized(cache)
    m = int(ids.shape[0])
    if cache.access_log is not None:
        cache.access_log.extend(("read", li) for li in range(config.n_layers))
    L, Hkv, dk = config.n_layers, cache.config.n_kv_heads, config.head_dim
    flags = _lib.PKV_QP_LOGITS | _lib.PKV_QP_APPEND_KV | _lib.PKV_QP_FROM_CHUNKS
    s = cache.context_length
    rows_dev = None
    if capture_attn:
        flags |= _lib.PKV_QP_ROWS
        rows_dev = torch.empty((L, m, s + m), dtype=torch.float32, device=cache.device)
    follow = getattr(cache, "_final_follow", None)
    cache._final_follow = None
    fused = getattr(cache, "_fused_final", None)
    cache._fused_final = None
    if fused is not None and not capture_attn and np.array_equal(fused[0], ids.astype(np.int32)):
        # the query rode along Stage II (pkv_recompute_query): logits and K/V are ready
        _, logits, fk, fv = fused
    elif follow is not None and cache.pool_tokens >= cache.context_length + m:
        # after the scoring pass (pre), layer l after Stage II's layer l (done[l]): the
        # narrow kernels of this pass run in the gaps of Stage II's big kernels
        pre, done, arr, c_fin = follow
        main = torch.cuda.current_stream()
        side = torch.cuda.Stream(device=cache.device)
        side.wait_event(pre)
        with torch.cuda.stream(side):
            fk = torch.empty((L, m, Hkv, dk), dtype=torch.float32, device=cache.device)
            fv = torch.empty_like(fk)
            logits = torch.empty(config.vocab_size, dtype=torch.float32, device=cache.device)
            run_query_pass(dm, cache, ids, flags, per_layer=rows_dev, fresh_k=fk, fresh_v=fv, logits=logits,
                           stream=side, c_cache=c_fin)
        main.wait_stream(side)
        for t in (fk, fv, logits) + ((rows_dev,) if rows_dev is not None else ()):
            t.record_stream(main)
    else:
        fk = torch.empty((L, m, Hkv, dk), dtype=torch.float32, device=cache.device)
        fv = torch.empty_like(fk)
        logits = torch.empty(config.vocab_size, dtype=torch.float32, device=cache.device)
        run_query_pass(dm, cache, ids, flags, per_layer=rows_dev, fresh_k=fk, fresh_v=fv, logits=logits)
    cache.query_kv = (fk, fv)
    bill_query_pass(tally, config, cache.context_length, m)
    first = logits.cpu().numpy()
    cache.check_finite()
    if not np.isfinite(first).all():
        raise NumericsError("non-finite values in the first-token logits")
    rows = None
    if rows_dev is not None:
        ra = rows_dev.cpu().numpy()
        rows = [np.ascontiguousarray(ra[li]) for li in range(L)]

    def keys():
        fkh = fk.cpu().numpy()
        return [np.concatenate([cache.keys_rebased[li], fkh[li]], axis=0) for li in range(L)]

    def values():
        fvh = fv.cpu().numpy()
        return [np.concatenate([cache.values[li], fvh[li]], axis=0) for li in range(L)]

    kv = KVCache(keys=keys, values=values, positions=np.arange(s + m, dtype=np.int64), last_logits=first)
    from .decode import DevicePools
    kv._device_pools = DevicePools.from_assembled(cache, s + m)  # decoding continues on the device
    return FinalizeResult(cache=kv, first_logits=first, rows=rows)


def selection_digest(indices) -> str:
    return hashlib.blake2b(np.asarray(sorted(indices), dtype=np.int64).tobytes(), digest_size=8).hexdigest()


@dataclass
class AnswerRecord:
    task_id: str
    strategy: str
    p: float
    answer_tokens: list
    answer_text: str
    exact_match: bool | None
    semantic_loss: float
    residual_loss: float
    flops_stage1: int
    flops_stage2: int
    selected_indices: list
    selection_digest: str

    def to_json_line(self) -> str:
        return json.dumps({"task_id": self.task_id, "strategy": self.strategy, "p": self.p,
                           "answer_text": self.answer_text, "exact_match": self.exact_match,
                           "semantic_loss": self.semantic_loss, "residual_loss": self.residual_loss,
                           "flops_stage1": self.flops_stage1, "flops_stage2": self.flops_stage2,
                           "selected_digest": self.selection_digest}, sort_keys=True)


@dataclass
class StrategyRun:
    """One (strategy, budget) cell: the TTFT slice plus greedy decoding on the device.
    The reference's unbilled measurement apparatus (full-prefill attention summaries and
    losses, recompute.py:194-206, 228-247) is outside the B200 hot path: those fields
    are None and the losses NaN."""
    record: AnswerRecord
    selection: SelectionResult
    scores: ValueScores
    full_summary: object
    naive_summary: object
    repaired_summary: object
    per_token_naive: object
    generated: object
    first_logits: np.ndarray


def run_strategy(weights, config: ModelConfig, chunks, query_tokens, strategy: str, p: float, *, seed: int = 0,
                 max_new_tokens: int = 16, stop_ids=(), gold_tokens=None, task_id: str = "",
                 tokenizer=None) -> StrategyRun:
    """assemble -> score -> select -> repair -> finalize (reference recompute.py:173-253)."""
    if strategy not in STRATEGIES and strategy != "naive":
        raise ArgumentError(f"unknown strategy {strategy!r}")
    if strategy == "naive" and p != 0.0:
        raise ConfigError("the naive baseline is only defined at p=0.0")
    cache = assemble(chunks, config)
    s = cache.context_length
    query = list(query_tokens)
    stage1 = FlopTally()
    if strategy == "prophet":
        scores = score_prophet(weights, config, cache, query, tally=stage1)
    elif strategy == "epic":
        scores = score_epic(cache, config.n_layers)
    elif strategy == "cacheblend_l1":
        scores = score_cacheblend_l1(weights, config, cache, tally=stage1)
    elif strategy == "kvshare_l1":
        scores = score_kvshare_l1(weights, config, cache, tally=stage1)
    elif strategy == "random":
        scores = score_random(s, seed, config.n_layers)
    else:
        scores = ValueScores.from_vector("naive", np.zeros(s, dtype=np.float32), config.n_layers)
    sel = select_top_p(scores, p)
    stage2 = FlopTally()
    recompute_selected(weights, config, cache, RecomputePlan(sel), tally=stage2)
    fin = finalize_query(weights, config, cache, query, tally=stage2)
    from .decode import greedy_generate
    gen = greedy_generate(weights, config, fin.cache, max_new_tokens, stop_ids=stop_ids)
    gold = list(gold_tokens) if gold_tokens is not None else None
    record = AnswerRecord(task_id=task_id, strategy=strategy, p=p, answer_tokens=gen.tokens,
                          answer_text=tokenizer.decode(gen.tokens) if tokenizer is not None else "",
                          exact_match=(gen.tokens == gold) if gold is not None else None,
                          semantic_loss=float("nan"), residual_loss=float("nan"),
                          flops_stage1=stage1.total.multiply_accumulate_count,
                          flops_stage2=stage2.total.multiply_accumulate_count, selected_indices=sel.indices,
                          selection_digest=selection_digest(sel.indices))
    return StrategyRun(record=record, selection=sel, scores=scores, full_summary=None, naive_summary=None,
                       repaired_summary=None, per_token_naive=None, generated=gen, first_logits=fin.first_logits)
