"""Position-independent chunk KV and the device-resident assembled cache.

Drop-in for reference chunkstore.py (ChunkKV 37-49, AssembledCache 65-96,
assemble 99-140, replace_entries 143-160, mark_finalized 232-236).  The cache
lives in HBM as one paged fp16 pool per (K, V) plus the keys' fp16 residual plane;
the reference's per-layer f32
arrays (``keys_rebased``/``values``) are exposed as lazily materialised views:
keys of entries that were never recomputed are re-derived bit-exactly from the
chunk store, recomputed entries come from the fp32 taps of Stage II.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ArgumentError, IncompatibleError, InputError, ShapeError, StateError
from .model import F32, F64, Layout, ModelConfig

PAGE = 128
QUERY_RESERVE = 256  # pool / rope headroom for query tokens appended at finalize


def chunk_content_id(fingerprint: str, token_ids) -> int:
    """64-bit content hash of (model fingerprint, token ids) (reference chunkstore.py:29-34)."""
    h = hashlib.blake2b(digest_size=8)
    h.update(fingerprint.encode())
    h.update(np.asarray(token_ids, dtype=np.int64).tobytes())
    return int.from_bytes(h.digest(), "little")


class ChunkKV:
    """Per-layer unrotated K and V of one chunk plus identity metadata.

    Host form (reference): ``keys_norope``/``values`` lists of f32 [t, Hkv, dk].
    Device form: one bf16 [L][t][Hkv][dkp] buffer each for K and V (the chunk
    store layout of include/pkv.h).  Either form is materialised on demand.
    """

    def __init__(self, chunk_id: int, config_fingerprint: str, token_ids, keys_norope=None, values=None,
                 device_k=None, device_v=None):
        self.chunk_id = chunk_id
        self.config_fingerprint = config_fingerprint
        self.token_ids = np.asarray(token_ids, dtype=np.int64)
        self._k_host = keys_norope
        self._v_host = values
        self._k_dev = device_k
        self._v_dev = device_v

    @property
    def n_tokens(self) -> int:
        return int(self.token_ids.shape[0])

    @property
    def keys_norope(self):
        if self._k_host is None:
            self._k_host = self._host_from_device(self._k_dev)
        return self._k_host

    @property
    def values(self):
        if self._v_host is None:
            self._v_host = self._host_from_device(self._v_dev)
        return self._v_host

    def _host_from_device(self, t):
        dk = self._dk
        a = t.float().cpu().numpy()
        return [np.ascontiguousarray(a[l, :, :, :dk]) for l in range(a.shape[0])]

    @property
    def pending_h2d(self) -> bool:
        """True while the device copy of a pinned-host chunk has not been scheduled."""
        return getattr(self, "_pinned", None) is not None

    def device_buffers(self, config: ModelConfig):
        """(K, V) bf16 device tensors [L][t][Hkv][dkp]; uploaded once from the host form.
        For pinned-host chunks the buffers are allocated here and filled layer by layer
        by assemble() (pipelined with the first query pass)."""
        if self._k_dev is None and self.pending_h2d:
            torch = _lib.require_cuda()
            kp, vp = self._pinned
            self._k_dev = torch.empty(kp.shape, dtype=kp.dtype, device="cuda")
            self._v_dev = torch.empty(vp.shape, dtype=vp.dtype, device="cuda")
        if self._k_dev is None:
            torch = _lib.require_cuda()
            lay = Layout.of(config)
            t, L, Hkv, dk = self.n_tokens, config.n_layers, config.n_kv_heads, config.head_dim
            if len(self._k_host) != L:
                raise IncompatibleError("chunk layer count does not match model config")
            dev = torch.device("cuda", torch.cuda.current_device())

            def pack(layers):
                a = np.stack([np.asarray(x, dtype=F32) for x in layers])
                if a.shape != (L, t, Hkv, dk):
                    raise ShapeError(f"chunk tensor shape {a.shape}, expected {(L, t, Hkv, dk)}")
                out = torch.zeros((L, t, Hkv, lay.dkp), dtype=torch.bfloat16, device=dev)
                out[..., :dk] = torch.from_numpy(a).to(dev).to(torch.bfloat16)
                return out

            self._k_dev = pack(self._k_host)
            self._v_dev = pack(self._v_host)
        self._dk = config.head_dim
        return self._k_dev, self._v_dev

    @classmethod
    def from_device(cls, chunk_id, fingerprint, token_ids, k_dev, v_dev, head_dim):
        c = cls(chunk_id, fingerprint, token_ids, device_k=k_dev, device_v=v_dev)
        c._dk = head_dim
        return c

    @classmethod
    def from_pinned(cls, chunk_id, fingerprint, token_ids, k_host, v_host, head_dim):
        """Chunk whose bf16 K/V ([L][t][Hkv][dkp]) live in pinned host memory (a host-tier
        chunk store); assemble() streams them to HBM layer by layer."""
        c = cls(chunk_id, fingerprint, token_ids)
        c._pinned = (k_host, v_host)
        c._dk = head_dim
        return c


def _rope_tables(theta: float, d: int, n: int):
    """float64 cos/sin [n][d/2] for positions 0..n-1 -- the reference's angle
    formula (tensor.py:104-107) evaluated by numpy, so device and reference use
    identical float64 factors."""
    inv = theta ** (-np.arange(0, d, 2, dtype=F64) / d)
    ang = np.arange(n, dtype=F64)[:, None] * inv[None, :]
    return np.cos(ang), np.sin(ang)


_ROPE_CACHE: dict = {}


def rope_device_tables(theta: float, d: int, n: int):
    torch = _lib.require_cuda()
    key = (float(theta), int(d), torch.cuda.current_device())
    hit = _ROPE_CACHE.get(key)
    if hit is None or hit[0] < n:
        n_alloc = max(n, 2 * (hit[0] if hit else 0))
        c, s = _rope_tables(theta, d, n_alloc)
        dev = torch.device("cuda", torch.cuda.current_device())
        cs32 = np.stack([c.astype(np.float32), s.astype(np.float32)], axis=-1)  # [n][d/2][2]
        hit = (n_alloc, torch.from_numpy(c).to(dev), torch.from_numpy(s).to(dev),
               torch.from_numpy(np.ascontiguousarray(cs32)).to(dev))
        _ROPE_CACHE[key] = hit
    return hit


class _LayerViews:
    """Sequence of per-layer f32 arrays [s, Hkv, dk] (keys_rebased / values)."""

    def __init__(self, cache: "AssembledCache", is_key: bool):
        self._c = cache
        self._k = is_key

    def __len__(self):
        return self._c.n_layers

    def __getitem__(self, layer):
        if isinstance(layer, slice):
            return [self[i] for i in range(*layer.indices(len(self)))]
        if layer < 0:
            layer += len(self)
        return self._c._layer_f32(layer, self._k)

    def __iter__(self):
        return (self[i] for i in range(len(self)))


class AssembledCache:
    """Device-resident assembled cache (reference chunkstore.py:65-96 surface)."""

    def __init__(self, config: ModelConfig, chunks, track_access: bool, fp32_taps):
        torch = _lib.require_cuda()
        self.config = config
        self.lay = Layout.of(config)
        fp = chunks[0].config_fingerprint
        self.config_fingerprint = fp
        self.token_ids = np.concatenate([c.token_ids for c in chunks]).astype(np.int64)
        s = int(self.token_ids.shape[0])
        self.positions = np.arange(s, dtype=np.int64)
        self.chunk_ids = [c.chunk_id for c in chunks]
        lens = [c.n_tokens for c in chunks]
        starts = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
        self.chunk_bounds = [(int(a), int(a + n)) for a, n in zip(starts, lens)]
        self.source_chunk = np.concatenate([np.full(n, i, dtype=np.int32) for i, n in enumerate(lens)])
        self.source_local = np.concatenate([np.arange(n, dtype=np.int32) for n in lens])
        self.recomputed = np.zeros((config.n_layers, s), dtype=bool)
        self.finalized = False
        self.access_log = [] if track_access else None
        dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        L, Hkv, dkp = config.n_layers, config.n_kv_heads, self.lay.dkp
        # device chunk view (keeps the chunk buffers alive)
        bufs = [c.device_buffers(config) for c in chunks]
        self._chunk_bufs = bufs
        self._d_kptr = torch.tensor([b[0].data_ptr() for b in bufs], dtype=torch.int64, device=dev)
        self._d_vptr = torch.tensor([b[1].data_ptr() for b in bufs], dtype=torch.int64, device=dev)
        self._d_len = torch.tensor(lens, dtype=torch.int32, device=dev)
        self._d_src_chunk = torch.from_numpy(self.source_chunk).to(dev)
        self._d_src_local = torch.from_numpy(self.source_local).to(dev)
        self._d_tokens = torch.from_numpy(self.token_ids.astype(np.int32)).to(dev)
        self._d_recomp = torch.zeros(s, dtype=torch.uint8, device=dev)
        # device check_finite of the Stage-II epilogues (include/pkv.h pkv_cache.nonfinite)
        self._d_nonfinite = torch.zeros(1, dtype=torch.int32, device=dev)
        self.pool_tokens = -(-(s + QUERY_RESERVE) // PAGE) * PAGE
        n_pages = self.pool_tokens // PAGE
        self._d_pages = torch.arange(n_pages, dtype=torch.int32, device=dev)
        shape = (L, Hkv, self.pool_tokens, dkp)
        self.k_pool = torch.empty(shape, dtype=torch.float16, device=dev)
        self.v_pool = torch.empty_like(self.k_pool)
        # residual plane of every f32 key (k_pool + k2 == f32 key to 2^-22), read by the
        # fp32-faithful narrow passes on the tensor cores
        self.k2_pool = torch.empty_like(self.k_pool)
        # slots [s, pool) are read by full-page tiles (masked, but P*V must stay finite):
        # assembly writes [0, s), so only the tail needs zeros
        for pool in (self.k_pool, self.v_pool, self.k2_pool):
            pool[:, :, s:].zero_()
        self.layer_events = None  # per-layer readiness when the chunk transfer is pipelined
        self._copy_stream = None
        self.rope_len, self._rcos, self._rsin, self._rcs32 = rope_device_tables(config.rope_theta, config.head_dim,
                                                                                self.pool_tokens)
        if fp32_taps == "auto":
            fp32_taps = 2 * L * s * Hkv * config.head_dim * 4 <= (1 << 30)
        self.fp32_taps = bool(fp32_taps)
        self._taps: dict = {}  # layer -> list of (idx np.int64, k f32 tensor, v f32 tensor)
        self._c_chunks = _lib.Chunks(self._d_kptr.data_ptr(), self._d_vptr.data_ptr(), self._d_len.data_ptr(),
                                     self._d_src_chunk.data_ptr(), self._d_src_local.data_ptr(), len(chunks))
        self._c_cache = self._make_c_cache()
        self._cfg_c = config.c_struct()
        self.query_kv = None  # set by finalize_query: (fresh_k, fresh_v) f32 device [L][m][Hkv][dk]

    # -- reference surface -------------------------------------------------------
    @property
    def context_length(self) -> int:
        return int(self.token_ids.shape[0])

    @property
    def n_layers(self) -> int:
        return self.config.n_layers

    @property
    def keys_rebased(self):
        return _LayerViews(self, True)

    @property
    def values(self):
        return _LayerViews(self, False)

    def layer_kv(self, layer: int):
        if self.access_log is not None:
            self.access_log.append(("read", layer))
        return self._layer_f32(layer, True), self._layer_f32(layer, False)

    def kv_layers(self):
        return [self.layer_kv(li) for li in range(self.n_layers)]

    # -- device plumbing ------------------------------------------------------------
    @property
    def c_cache(self):
        return self._c_cache

    @property
    def c_chunks(self):
        return self._c_chunks

    def _layer_f32(self, layer: int, is_key: bool) -> np.ndarray:
        torch = _lib.require_cuda()
        self.wait_ready()
        s, Hkv, dk = self.context_length, self.config.n_kv_heads, self.config.head_dim
        out = torch.empty((s, Hkv, dk), dtype=torch.float32, device=self.device)
        # never-recomputed entries: exact f32 from the chunk store; others: the cache
        use_chunks = not self.recomputed[layer].any() or self.fp32_taps
        _lib.check(_lib.load().pkv_cache_view(ctypes_ref(self._cfg_c), ctypes_ref(self._c_cache),
                                              ctypes_ref(self._c_chunks) if use_chunks else None, layer,
                                              1 if is_key else 0, out.data_ptr(),
                                              _lib.stream_ptr(torch)))
        if use_chunks and self.recomputed[layer].any():
            for idx, tk, tv in self._taps.get(layer, []):
                out[torch.from_numpy(idx).to(self.device)] = tk if is_key else tv
        return out.cpu().numpy()

    def add_tap(self, layer: int, idx: np.ndarray, k_f32, v_f32) -> None:
        self._taps.setdefault(layer, []).append((np.asarray(idx, dtype=np.int64), k_f32, v_f32))

    def ensure_query_room(self, m: int) -> None:
        """Grow pool / rope tables when a query longer than the reserve arrives."""
        need = self.context_length + m
        if need <= self.pool_tokens:
            return
        torch = _lib.require_cuda()
        self.wait_ready()
        new_tokens = -(-need // PAGE) * PAGE
        L, Hkv, dkp = self.k_pool.shape[0], self.k_pool.shape[1], self.k_pool.shape[3]
        self._final_follow = None  # the overlapped final pass would read the freed pools
        for name in ("k_pool", "v_pool", "k2_pool"):
            old = getattr(self, name)
            new = torch.zeros((L, Hkv, new_tokens, dkp), dtype=old.dtype, device=old.device)
            new[:, :, : self.pool_tokens] = old
            setattr(self, name, new)
        self.pool_tokens = new_tokens
        self._d_pages = torch.arange(new_tokens // PAGE, dtype=torch.int32, device=self.device)
        self.rope_len, self._rcos, self._rsin, self._rcs32 = rope_device_tables(
            self.config.rope_theta, self.config.head_dim, new_tokens)
        self._c_cache = self._make_c_cache()

    def _make_c_cache(self):
        ready = None
        if self.layer_events is not None:
            self._c_events = (_lib.c_vp * len(self.layer_events))(*[e.cuda_event for e in self.layer_events])
            ready = self._c_events
        return _lib.Cache(self.k_pool.data_ptr(), self.v_pool.data_ptr(), self.pool_tokens, self._d_pages.data_ptr(),
                          self.context_length, self._d_tokens.data_ptr(), self._rcos.data_ptr(),
                          self._rsin.data_ptr(), self.rope_len, self._d_recomp.data_ptr(), self.k2_pool.data_ptr(),
                          ready, self._rcs32.data_ptr(), nonfinite=self._d_nonfinite.data_ptr())

    def check_finite(self) -> None:
        """Raise NumericsError if a Stage-II epilogue wrote a non-finite (or fp16-overflowing)
        value -- the reference checks every kernel output (tensor.py:31-34); the device flag
        is read here, after a synchronisation (finalize_query calls it)."""
        from .errors import NumericsError
        if int(self._d_nonfinite.item()) != 0:
            raise NumericsError("non-finite values in the Stage-II repair")

    def wait_ready(self, stream=None) -> None:
        """Make `stream` (default: current) wait for a pipelined chunk transfer to finish."""
        if self._copy_stream is not None:
            torch = _lib.require_cuda()
            (stream or torch.cuda.current_stream()).wait_stream(self._copy_stream)


def _as_chunk(c) -> ChunkKV:
    """Accept reference pikv.ChunkKV objects (same field names); the device copy is
    cached on the object so a chunk shared by many requests uploads once."""
    if isinstance(c, ChunkKV):
        return c
    w = getattr(c, "__b200_chunk__", None)
    if w is None:
        w = ChunkKV(c.chunk_id, c.config_fingerprint, c.token_ids, c.keys_norope, c.values)
        try:
            c.__b200_chunk__ = w
        except AttributeError:
            pass
    return w


def ctypes_ref(x):
    import ctypes
    return ctypes.byref(x) if x is not None else None


def assemble(chunks, config: ModelConfig, track_access: bool = False, *, fp32_taps="auto",
             stream=None) -> AssembledCache:
    """Concatenate chunk KVs into the paged cache and rotate keys at their global
    positions (reference chunkstore.py:99-140), on the GPU (kernel K1)."""
    if not chunks:
        raise InputError("assemble needs at least one chunk")
    chunks = [_as_chunk(c) for c in chunks]
    fp = chunks[0].config_fingerprint
    for c in chunks:
        if c.config_fingerprint != fp:
            raise IncompatibleError(f"chunk {c.chunk_id:#x} was precomputed under fingerprint "
                                    f"{c.config_fingerprint}, expected {fp}")
        k = c._k_dev if c._k_dev is not None else c._k_host
        if k is not None and len(k) != config.n_layers:
            raise IncompatibleError("chunk layer count does not match model config")
    torch = _lib.require_cuda()
    pending = [c for c in chunks if c.pending_h2d]
    cache = AssembledCache(config, chunks, track_access, fp32_taps)
    lib = _lib.load()
    if not pending:
        _lib.check(lib.pkv_assemble(ctypes_ref(cache._cfg_c), ctypes_ref(cache._c_chunks),
                                    ctypes_ref(cache._c_cache), _lib.stream_ptr(torch, stream)))
        return cache
    # host-tier chunks: stream them layer by layer -- keys and values on two copy streams
    # (two DMA engines, never stalled behind a kernel) -- and assemble each layer on a
    # third stream as soon as both halves land; query passes / Stage II wait per layer
    main = stream or torch.cuda.current_stream()
    cs, ck, cv = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    for st_ in (cs, ck, cv):
        st_.wait_stream(main)  # pools and buffers were allocated / zeroed on `main`
    events = []
    for li in range(config.n_layers):
        ek, evv = torch.cuda.Event(), torch.cuda.Event()
        with torch.cuda.stream(ck):
            for c in pending:
                c._k_dev[li].copy_(c._pinned[0][li], non_blocking=True)
            ek.record(ck)
        with torch.cuda.stream(cv):
            for c in pending:
                c._v_dev[li].copy_(c._pinned[1][li], non_blocking=True)
            evv.record(cv)
        cs.wait_event(ek)
        cs.wait_event(evv)
        _lib.check(lib.pkv_assemble_layers(ctypes_ref(cache._cfg_c), ctypes_ref(cache._c_chunks),
                                           ctypes_ref(cache._c_cache), li, li + 1, cs.cuda_stream))
        ev = torch.cuda.Event()
        ev.record(cs)
        events.append(ev)
    cache._pinned_refs = [c._pinned for c in pending]  # host buffers stay alive until the DMA is done
    for c in pending:
        for st_ in (cs, ck, cv):
            c._k_dev.record_stream(st_)
            c._v_dev.record_stream(st_)
        c._pinned = None
    for t in (cache.k_pool, cache.v_pool, cache.k2_pool, cache._d_recomp):
        t.record_stream(cs)
    cache.layer_events = events
    cache._copy_stream = cs
    cache._c_cache = cache._make_c_cache()
    return cache


def replace_entries(cache: AssembledCache, layer: int, indices, new_keys, new_values) -> None:
    """Overwrite cache entries at one layer and mark them recomputed (reference
    chunkstore.py:143-160), scattering into the fp16 pool on the GPU."""
    if not 0 <= layer < cache.n_layers:
        raise ArgumentError(f"layer {layer} out of range for {cache.n_layers} layers")
    # a later finalize_query must see this write: no overlap with the preceding repair
    # (recompute.finalize_query only follows Stage II's per-layer events)
    cache._final_follow = None
    # ... nor reuse the query rows a fused repair computed before this write
    cache._fused_final = None
    idx = np.asarray(indices, dtype=np.int64)
    if idx.ndim != 1:
        raise ShapeError("indices must be 1-D")
    if idx.size and (idx.min() < 0 or idx.max() >= cache.context_length):
        raise InputError("replacement index out of range")
    want = (idx.shape[0], cache.config.n_kv_heads, cache.config.head_dim)
    nk, nv = np.asarray(new_keys), np.asarray(new_values)
    if nk.shape != want or nv.shape != want:
        raise ShapeError(f"replacement shape {nk.shape}/{nv.shape}, expected {want}")
    if cache.access_log is not None:
        cache.access_log.append(("write", layer))
    cache.wait_ready()
    if idx.size == 0:
        return
    torch = _lib.require_cuda()
    dev = cache.device
    d_idx = torch.from_numpy(idx.astype(np.int32)).to(dev)
    tk = torch.from_numpy(np.ascontiguousarray(nk, dtype=F32)).to(dev)
    tv = torch.from_numpy(np.ascontiguousarray(nv, dtype=F32)).to(dev)
    _lib.check(_lib.load().pkv_replace_entries(ctypes_ref(cache._cfg_c), ctypes_ref(cache._c_cache), layer,
                                               d_idx.data_ptr(), int(idx.size), tk.data_ptr(), tv.data_ptr(),
                                               _lib.stream_ptr(torch)))
    if cache.fp32_taps:
        cache.add_tap(layer, idx, tk, tv)
    cache.recomputed[layer, idx] = True


def mark_finalized(cache: AssembledCache) -> None:
    """One-shot finalisation flag (reference chunkstore.py:232-236)."""
    if cache.finalized:
        raise StateError("cache already finalized with query tokens")
    cache.finalized = True
