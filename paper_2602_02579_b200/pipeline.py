"""Sync-free device pipeline of one ProphetKV prefill (the bench's "step").

assemble -> narrow pass with scores -> fuse + top-k -> Stage II -> finalize,
as five stream-ordered C-ABI calls on preallocated buffers.  k = ceil(p*s) is
computed on the host before launch (reference tensor.py:136-140), so nothing in
the step waits for the device.  The public pikv-style functions run the same
calls but materialise numpy results (selection list, scores, logits) between
stages.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _lib
from .chunkstore import AssembledCache, ChunkKV, ctypes_ref
from .model import DeviceModel
from .tensor import ratio_budget


def _created_events(n: int) -> list:
    """torch creates the cudaEvent_t behind torch.cuda.Event on its first record(); the
    C side gets the raw handles (include/pkv.h layer_ready / layer_done), so record once."""
    torch = _lib.require_cuda()
    evs = [torch.cuda.Event() for _ in range(n)]
    for e in evs:
        e.record()
    return evs


class PrefillPipeline:
    def __init__(self, dm: DeviceModel, chunks: list, m: int, p: float, stage1_dm: DeviceModel | None = None):
        """stage1_dm: the scoring pass on a head-sharded model (DeviceModel.shard) over its
        head slice of this pipeline's full cache, with Stage II token-parallel on dm
        (DeviceModel.rows) -- both multi-GPU splits at once (include/pkv.h pool_heads)."""
        torch = _lib.require_cuda()
        self.dm = dm
        self.s1_dm = stage1_dm if stage1_dm is not None else dm
        cfg = dm.config
        self.cfg = cfg
        self.cache = AssembledCache(dm.cache_config, chunks, track_access=False, fp32_taps=False)
        self.cache.ensure_query_room(m)
        s = self.cache.context_length
        self.s, self.m, self.p = s, m, p
        self.k = ratio_budget(p, s)
        dev = self.cache.device
        lib = _lib.load()
        self.flags_score = _lib.PKV_QP_SCORES | _lib.PKV_QP_FROM_CHUNKS
        self.flags_final = _lib.PKV_QP_LOGITS | _lib.PKV_QP_APPEND_KV | _lib.PKV_QP_FROM_CHUNKS
        qp_bytes = max(lib.pkv_query_pass_workspace(self.s1_dm.handle, s, m, self.flags_score),
                       lib.pkv_query_pass_workspace(dm.handle, s, m, self.flags_final))
        self.ws_qp = torch.empty(qp_bytes, dtype=torch.uint8, device=dev)
        # finalize fused into Stage II (pkv_recompute_query): the query rows ride along the
        # repair, so no separate final pass runs after or interleaved with Stage II
        # (PKV_FUSED_FINAL=0: the separate fp32-faithful query pass)
        self.fused_final = os.environ.get("PKV_FUSED_FINAL", "1") == "1"
        self.rows_comm = getattr(dm, "rows_comm", None)  # token-parallel Stage II (DeviceModel.rows)
        if self.rows_comm is not None:
            rc_bytes = lib.pkv_recompute_rows_workspace(dm.handle, self.k, m if self.fused_final else 0,
                                                        self.rows_comm.world)
        else:
            rc_bytes = (lib.pkv_recompute_query_workspace(dm.handle, self.k, m) if self.fused_final
                        else lib.pkv_recompute_workspace(dm.handle, max(self.k, 1)))
        self.ws_rc = torch.empty(max(rc_bytes, 256), dtype=torch.uint8, device=dev)
        self.per_layer = torch.empty((cfg.n_layers, s), dtype=torch.float32, device=dev)
        self.fused = torch.empty(s, dtype=torch.float32, device=dev)
        self.idx = torch.empty(max(self.k, 1), dtype=torch.int32, device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.logits = torch.empty(cfg.vocab_size, dtype=torch.float32, device=dev)
        self.query = torch.zeros(m, dtype=torch.int32, device=dev)
        # layer-pipelined assembly: layer l is assembled on a side stream and the scoring
        # pass (and Stage II's scatter) wait on layer_ready[l] (include/pkv.h), so the
        # HBM-bound assembly of layers l+1.. overlaps the narrow pass over layer l
        self.side = torch.cuda.Stream(device=dev)
        # per-layer assembly on the side stream overlapping the scoring pass: measured
        # neutral for device-resident chunks (both phases compete for HBM), so opt-in
        self.pipelined_assembly = os.environ.get("PKV_ASM_PIPE", "0") == "1"
        self.layer_events = _created_events(cfg.n_layers)
        self.cache.layer_events = self.layer_events
        self.cache._c_cache = self.cache._make_c_cache()
        # final pass following Stage II layer by layer: pkv_recompute records done[l] once
        # layer l's K/V are final and the final query pass (on its own stream) waits on
        # done[l] before its layer-l attention, so its narrow kernels fill the gaps of
        # Stage II instead of running after it (PKV_FINAL_OVERLAP=0: serial)
        # (unsharded models only: two streams issuing collectives on one communicator
        # could be ordered differently on different ranks)
        self.final_overlap = os.environ.get("PKV_FINAL_OVERLAP", "1") == "1" and getattr(dm, "tp_world", 1) == 1
        self.fin = torch.cuda.Stream(device=dev)
        self.done_events = _created_events(cfg.n_layers)
        self._c_done = (_lib.c_vp * cfg.n_layers)(*[e.cuda_event for e in self.done_events])
        self._c_rc = _lib.Cache.from_buffer_copy(self.cache._c_cache)
        self._c_rc.layer_done = self._c_done
        self._c_fin = _lib.Cache.from_buffer_copy(self.cache._c_cache)
        self._c_fin.layer_ready = self._c_done

    def set_query(self, ids) -> None:
        torch = _lib.require_cuda()
        self.query.copy_(torch.as_tensor(np.asarray(ids, dtype=np.int32)), non_blocking=True)

    def full_prefill_step(self, stream=None) -> None:
        """The comparator of the north star's TTFT ratio: a full GPU prefill of the same
        request (reference model.py:332-359 over context + query) with the same kernels --
        Stage II with every context token selected (every cache entry recomputed, no chunk
        reuse), then the query pass for the first-token logits."""
        torch = _lib.require_cuda()
        lib = _lib.load()
        if not hasattr(self, "_all_idx"):
            self._all_idx = torch.arange(self.s, dtype=torch.int32, device=self.cache.device)
            self._ws_full = torch.empty(lib.pkv_recompute_workspace(self.dm.handle, self.s), dtype=torch.uint8,
                                        device=self.cache.device)
        st = _lib.stream_ptr(torch, stream)
        c = self.cache
        cc, ch = ctypes_ref(c.c_cache), ctypes_ref(c.c_chunks)
        _lib.check(lib.pkv_recompute(self.dm.handle, cc, self._all_idx.data_ptr(), self.s, None, None,
                                     self._ws_full.data_ptr(), self._ws_full.numel(), st))
        _lib.check(lib.pkv_query_pass(self.dm.handle, cc, ch, self.query.data_ptr(), self.m, self.flags_final, None,
                                      None, None, self.logits.data_ptr(), self.ws_qp.data_ptr(), self.ws_qp.numel(),
                                      st))

    def capture(self, fn=None):
        """Record one step (or `fn`, e.g. self.stage2) into a CUDA graph (call after a
        warm-up step so every kernel attribute is set); replay() then launches the ~1.5k
        kernels of a prefill with one host call.  Returns the graph."""
        torch = _lib.require_cuda()
        graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            with torch.cuda.graph(graph, stream=side):
                (fn or self.step)()
        torch.cuda.current_stream().wait_stream(side)
        # the events' last record was a capture node: waiting on them from eager work
        # (full_prefill_step, an eager step()) is an error until they are recorded again
        for e in self.layer_events + self.done_events:
            e.record()
        if fn is None:
            self.graph = graph
        return graph

    def replay(self) -> None:
        self.graph.replay()

    def score_select(self, stream=None) -> None:
        """assemble -> scoring pass -> fuse + top-k only (per_layer, fused, idx)."""
        torch = _lib.require_cuda()
        main = stream if stream is not None else torch.cuda.current_stream()
        self._stage1(_lib.load(), _lib.stream_ptr(torch, stream), main)
        main.wait_stream(self.side)

    def _stage1(self, lib, st, main) -> None:
        c = self.cache
        cc, ch = ctypes_ref(c.c_cache), ctypes_ref(c.c_chunks)
        self.side.wait_stream(main)
        if self.pipelined_assembly:
            for li in range(self.cfg.n_layers):
                _lib.check(lib.pkv_assemble_layers(ctypes_ref(c._cfg_c), ch, cc, li, li + 1, self.side.cuda_stream))
                self.layer_events[li].record(self.side)
        else:
            _lib.check(lib.pkv_assemble(ctypes_ref(c._cfg_c), ch, cc, self.side.cuda_stream))
            for ev in self.layer_events:
                ev.record(self.side)
        if self.s1_dm is not self.dm:  # this rank's head slice of the full cache
            w = self.s1_dm.tp_world
            hl = self.cfg.n_kv_heads // w
            sc = _lib.Cache.from_buffer_copy(c.c_cache)
            sc.pool_heads, sc.head0 = self.cfg.n_kv_heads, self.s1_dm.tp_rank * hl
            self._c_slice = sc
            cc = ctypes_ref(sc)
        _lib.check(lib.pkv_query_pass(self.s1_dm.handle, cc, ch, self.query.data_ptr(), self.m, self.flags_score,
                                      self.per_layer.data_ptr(), None, None, None, self.ws_qp.data_ptr(),
                                      self.ws_qp.numel(), st))
        _lib.check(lib.pkv_fuse_select(self.per_layer.data_ptr(), self.cfg.n_layers, self.s, self.k,
                                       self.fused.data_ptr(), self.idx.data_ptr(), self.status.data_ptr(), None, 0, st))

    def _plain_cache(self):
        """The cache view without per-layer readiness events (standalone phases: every layer
        is assembled before they run, and a graph capture may not wait on eager events)."""
        cc = _lib.Cache.from_buffer_copy(self.cache.c_cache)
        cc.layer_ready = None
        self._c_plain = cc
        return cc

    def stage2(self, stream=None) -> None:
        """Stage II alone (recompute of the current selection idx; with the fused finalize
        also the query rows and the first-token logits), serial order."""
        torch = _lib.require_cuda()
        self._recompute(_lib.load(), ctypes_ref(self._plain_cache()), _lib.stream_ptr(torch, stream))

    def _recompute(self, lib, cc, st) -> None:
        if self.rows_comm is not None:
            m = self.m if self.fused_final else 0
            _lib.check(lib.pkv_recompute_rows(self.dm.handle, cc, self.idx.data_ptr(), self.k,
                                              self.query.data_ptr() if m else None, m, self.rows_comm.handle,
                                              self.logits.data_ptr() if m else None, self.ws_rc.data_ptr(),
                                              self.ws_rc.numel(), st))
            if not m:
                _lib.check(lib.pkv_query_pass(self.dm.handle, cc, ctypes_ref(self.cache.c_chunks), self.query.data_ptr(),
                                              self.m, self.flags_final, None, None, None, self.logits.data_ptr(),
                                              self.ws_qp.data_ptr(), self.ws_qp.numel(), st))
        elif self.fused_final:
            _lib.check(lib.pkv_recompute_query(self.dm.handle, cc, self.idx.data_ptr(), self.k, self.query.data_ptr(),
                                               self.m, None, None, None, None, self.logits.data_ptr(),
                                               self.ws_rc.data_ptr(), self.ws_rc.numel(), st))
        else:
            _lib.check(lib.pkv_recompute(self.dm.handle, cc, self.idx.data_ptr(), self.k, None, None,
                                         self.ws_rc.data_ptr(), self.ws_rc.numel(), st))

    def final(self, stream=None) -> None:
        """The final query pass alone (first-token logits over the repaired cache)."""
        torch = _lib.require_cuda()
        c = self.cache
        _lib.check(_lib.load().pkv_query_pass(self.dm.handle, ctypes_ref(self._plain_cache()), ctypes_ref(c.c_chunks),
                                              self.query.data_ptr(), self.m, self.flags_final, None, None, None,
                                              self.logits.data_ptr(), self.ws_qp.data_ptr(), self.ws_qp.numel(),
                                              _lib.stream_ptr(torch, stream)))

    def step(self, stream=None) -> None:
        """One full prefill; results stay on the device (idx, logits, per_layer)."""
        torch = _lib.require_cuda()
        lib = _lib.load()
        st = _lib.stream_ptr(torch, stream)
        c = self.cache
        cc, ch = ctypes_ref(c.c_cache), ctypes_ref(c.c_chunks)
        main = stream if stream is not None else torch.cuda.current_stream()
        self._stage1(lib, st, main)
        if self.fused_final or self.rows_comm is not None:
            self._recompute(lib, cc, st)
            main.wait_stream(self.side)  # rejoin (required for graph capture)
            return
        if self.final_overlap:
            # after the scoring pass (it shares ws_qp) and the selection; layer l waits on done[l]
            self.fin.wait_stream(main)
        if self.final_overlap:
            self._c_rc.layer_ready = c.c_cache.layer_ready
            _lib.check(lib.pkv_recompute(self.dm.handle, ctypes_ref(self._c_rc), self.idx.data_ptr(), self.k, None,
                                         None, self.ws_rc.data_ptr(), self.ws_rc.numel(), st))
            _lib.check(lib.pkv_query_pass(self.dm.handle, ctypes_ref(self._c_fin), ch, self.query.data_ptr(), self.m,
                                          self.flags_final, None, None, None, self.logits.data_ptr(),
                                          self.ws_qp.data_ptr(), self.ws_qp.numel(), self.fin.cuda_stream))
            main.wait_stream(self.fin)
        else:
            _lib.check(lib.pkv_recompute(self.dm.handle, cc, self.idx.data_ptr(), self.k, None, None,
                                         self.ws_rc.data_ptr(), self.ws_rc.numel(), st))
            _lib.check(lib.pkv_query_pass(self.dm.handle, cc, ch, self.query.data_ptr(), self.m, self.flags_final,
                                          None, None, None, self.logits.data_ptr(), self.ws_qp.data_ptr(),
                                          self.ws_qp.numel(), st))
        main.wait_stream(self.side)  # rejoin (required for graph capture)


def random_device_chunks(cfg, n_chunks: int, chunk_len: int, seed: int = 0, fingerprint: str = "device-random"):
    """Synthetic chunk store: N(0,1) bf16 unrotated keys and values per chunk
    (layout [L][t][Hkv][dkp]) and uniform token ids -- for benchmarks only."""
    torch = _lib.require_cuda()
    lay = cfg.layout()
    g = torch.Generator(device="cuda").manual_seed(seed)
    rng = np.random.default_rng(seed)
    out = []
    for ci in range(n_chunks):
        shape = (cfg.n_layers, chunk_len, cfg.n_kv_heads, lay.dkp)
        k = torch.zeros(shape, dtype=torch.bfloat16, device="cuda")
        v = torch.zeros(shape, dtype=torch.bfloat16, device="cuda")
        k[..., :cfg.head_dim] = torch.randn(shape[:-1] + (cfg.head_dim,), generator=g, device="cuda")
        v[..., :cfg.head_dim] = torch.randn(shape[:-1] + (cfg.head_dim,), generator=g, device="cuda")
        ids = rng.integers(0, cfg.vocab_size, chunk_len)
        out.append(ChunkKV.from_device(ci, fingerprint, ids, k, v, cfg.head_dim))
    return out
