"""Model types of the drop-in and their B200 device image.

Host-side types keep the reference ``pikv.model`` surface (ModelConfig,
LayerWeights, ModelWeights, random_weights, FlopTally, KVCache -- reference
model.py:24-228) so caller code constructs them unchanged.  ``DeviceModel`` is the
B200 image: fp16 projection weights (pre-scaled by a power of two per matrix)
transposed to output-major rows, head dims padded to the kernel tile, bf16 embed /
lm_head (see include/pkv.h "Device layouts"), plus the C-ABI model handle.
"""

from __future__ import annotations

import ctypes
import hashlib
import json
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ConfigError, EngineError

F32 = np.float32
F64 = np.float64


@dataclass(frozen=True)
class ModelConfig:
    """Shape contract; validation mirrors reference model.py:36-50."""

    n_layers: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    hidden_dim: int
    ffn_dim: int
    vocab_size: int
    rope_theta: float = 10000.0
    norm_eps: float = 1e-5

    def __post_init__(self) -> None:
        dims = (self.n_layers, self.n_heads, self.n_kv_heads, self.head_dim, self.ffn_dim, self.vocab_size)
        if min(dims) <= 0:
            raise ConfigError("all model dimensions must be positive")
        if self.n_heads % self.n_kv_heads:
            raise ConfigError(f"n_heads={self.n_heads} not divisible by n_kv_heads={self.n_kv_heads}")
        if self.hidden_dim != self.n_heads * self.head_dim:
            raise ConfigError(f"hidden_dim={self.hidden_dim} != n_heads*head_dim={self.n_heads * self.head_dim}")
        if self.head_dim % 2:
            raise ConfigError(f"head_dim must be even for rotary pairs, got {self.head_dim}")
        if self.rope_theta <= 0 or self.norm_eps <= 0:
            raise ConfigError("rope_theta and norm_eps must be positive")

    @property
    def kv_dim(self) -> int:
        return self.n_kv_heads * self.head_dim

    def to_json_dict(self) -> dict:
        return {k: getattr(self, k) for k in ("n_layers", "n_heads", "n_kv_heads", "head_dim", "hidden_dim",
                                              "ffn_dim", "vocab_size", "rope_theta", "norm_eps")}

    def c_struct(self) -> _lib.Config:
        return _lib.Config(self.n_layers, self.n_heads, self.n_kv_heads, self.head_dim, self.hidden_dim,
                           self.ffn_dim, self.vocab_size, float(self.rope_theta), float(self.norm_eps))

    def layout(self) -> "Layout":
        return Layout.of(self)


@dataclass(frozen=True)
class Layout:
    """Padded device layout (pkv_layout): dkp, Dp, Fp, NQKV, HQ."""

    dkp: int
    Dp: int
    Fp: int
    NQKV: int
    HQ: int

    @staticmethod
    def of(cfg: ModelConfig) -> "Layout":
        if cfg.head_dim > 128:
            raise ConfigError("head_dim > 128 is not supported by the sm_100a kernels")
        dkp = 64 if cfg.head_dim <= 64 else 128
        Dp = -(-cfg.hidden_dim // 64) * 64
        Fp = -(-cfg.ffn_dim // 128) * 128
        return Layout(dkp, Dp, Fp, (cfg.n_heads + 2 * cfg.n_kv_heads) * dkp, cfg.n_heads * dkp)


@dataclass
class LayerWeights:
    attn_norm: np.ndarray   # [hidden]
    wq: np.ndarray          # [hidden, n_heads*head_dim]
    wk: np.ndarray          # [hidden, kv_dim]
    wv: np.ndarray          # [hidden, kv_dim]
    wo: np.ndarray          # [n_heads*head_dim, hidden]
    ffn_norm: np.ndarray    # [hidden]
    w_gate: np.ndarray      # [hidden, ffn]
    w_up: np.ndarray        # [hidden, ffn]
    w_down: np.ndarray      # [ffn, hidden]


@dataclass
class ModelWeights:
    """Host weights, input-major like the reference (model.py:79-160)."""

    embed: np.ndarray
    layers: list
    final_norm: np.ndarray
    lm_head: np.ndarray
    _fingerprint: str | None = field(default=None, repr=False, compare=False)
    _device: dict = field(default_factory=dict, repr=False, compare=False)

    def validate(self, config: ModelConfig) -> None:
        h, kv, hd = config.hidden_dim, config.kv_dim, config.n_heads * config.head_dim
        if self.embed.shape != (config.vocab_size, h):
            raise ConfigError(f"embed shape {self.embed.shape} does not match config")
        if len(self.layers) != config.n_layers:
            raise ConfigError(f"{len(self.layers)} layer weight sets for {config.n_layers} layers")
        want = {"attn_norm": (h,), "wq": (h, hd), "wk": (h, kv), "wv": (h, kv), "wo": (hd, h), "ffn_norm": (h,),
                "w_gate": (h, config.ffn_dim), "w_up": (h, config.ffn_dim), "w_down": (config.ffn_dim, h)}
        for i, lw in enumerate(self.layers):
            for name, shape in want.items():
                if getattr(lw, name).shape != shape:
                    raise ConfigError(f"layers.{i}.{name} shape {getattr(lw, name).shape}, expected {shape}")
        if self.final_norm.shape != (h,) or self.lm_head.shape != (h, config.vocab_size):
            raise ConfigError("final_norm / lm_head shape mismatch")

    def named_tensors(self) -> list:
        out = [("embed.weight", self.embed)]
        for i, lw in enumerate(self.layers):
            p = f"layers.{i}"
            out += [(f"{p}.attn_norm.gain", lw.attn_norm), (f"{p}.attn.wq", lw.wq), (f"{p}.attn.wk", lw.wk),
                    (f"{p}.attn.wv", lw.wv), (f"{p}.attn.wo", lw.wo), (f"{p}.ffn_norm.gain", lw.ffn_norm),
                    (f"{p}.ffn.w_gate", lw.w_gate), (f"{p}.ffn.w_up", lw.w_up), (f"{p}.ffn.w_down", lw.w_down)]
        return out + [("final_norm.gain", self.final_norm), ("lm_head.weight", self.lm_head)]

    @classmethod
    def from_named(cls, config: ModelConfig, tensors: dict) -> "ModelWeights":
        """Inverse of named_tensors (reference model.py:124-145): missing name -> ConfigError,
        tensors taken as contiguous f32, the result validated against the config."""
        def take(name):
            if name not in tensors:
                raise ConfigError(f"missing tensor {name!r}")
            return np.ascontiguousarray(tensors[name], dtype=F32)

        layers = []
        for i in range(config.n_layers):
            p = f"layers.{i}"
            layers.append(LayerWeights(
                attn_norm=take(f"{p}.attn_norm.gain"), wq=take(f"{p}.attn.wq"), wk=take(f"{p}.attn.wk"),
                wv=take(f"{p}.attn.wv"), wo=take(f"{p}.attn.wo"), ffn_norm=take(f"{p}.ffn_norm.gain"),
                w_gate=take(f"{p}.ffn.w_gate"), w_up=take(f"{p}.ffn.w_up"), w_down=take(f"{p}.ffn.w_down")))
        w = cls(embed=take("embed.weight"), layers=layers, final_norm=take("final_norm.gain"),
                lm_head=take("lm_head.weight"))
        w.validate(config)
        return w

    def fingerprint(self, config: ModelConfig) -> str:
        """blake2b-8 of config JSON + weight bytes (reference model.py:147-160)."""
        if self._fingerprint is None:
            h = hashlib.blake2b(digest_size=8)
            h.update(json.dumps(config.to_json_dict(), sort_keys=True).encode())
            for name, t in self.named_tensors():
                h.update(name.encode())
                h.update(np.ascontiguousarray(t, dtype=F32).tobytes())
            self._fingerprint = h.hexdigest()
        return self._fingerprint

    def device(self, config: ModelConfig) -> "DeviceModel":
        """The cached B200 image of these weights, uploaded once per (config, device): the
        same weights under another config (rope_theta, norm_eps, ...) get their own image."""
        import torch
        key = (config, torch.cuda.current_device())
        dm = self._device.get(key)
        if dm is None:
            dm = DeviceModel.from_host(self, config)
            self._device[key] = dm
        return dm


def random_weights(config: ModelConfig, seed: int) -> ModelWeights:
    """Seeded host weights; same PCG64 stream and scaling as reference model.py:163-185."""
    rng = np.random.default_rng(seed)

    def mat(rows, cols):
        return (rng.standard_normal((rows, cols)) / np.sqrt(rows)).astype(F32)

    h, hd, kv, f = config.hidden_dim, config.n_heads * config.head_dim, config.kv_dim, config.ffn_dim
    layers = []
    for _ in range(config.n_layers):
        wq, wk, wv, wo = mat(h, hd), mat(h, kv), mat(h, kv), mat(hd, h)
        wg, wu, wd = mat(h, f), mat(h, f), mat(f, h)
        layers.append(LayerWeights(np.ones(h, F32), wq, wk, wv, wo, np.ones(h, F32), wg, wu, wd))
    embed = rng.standard_normal((config.vocab_size, h)).astype(F32)
    return ModelWeights(embed=embed, layers=layers, final_norm=np.ones(h, F32), lm_head=mat(h, config.vocab_size))


@dataclass
class FlopCounter:
    """Monotonic multiply-accumulate counter (reference tensor.py:37-46)."""

    multiply_accumulate_count: int = 0

    def add(self, n: int) -> None:
        from .errors import ArgumentError
        if n < 0:
            raise ArgumentError(f"flop increment must be >= 0, got {n}")
        self.multiply_accumulate_count += n


@dataclass
class FlopTally:
    """MAC books (reference model.py:188-193), filled analytically by the device path."""

    total: FlopCounter = field(default_factory=FlopCounter)
    attn_scores: FlopCounter = field(default_factory=FlopCounter)


def bill_query_pass(tally, config: ModelConfig, s: int, m: int, with_logits: bool = True) -> None:
    """Books of one narrow pass of m tokens over s entries, as the reference's
    matmul-level counting produces them."""
    if tally is None:
        return
    H, dk, D, F, KV = config.n_heads, config.head_dim, config.hidden_dim, config.ffn_dim, config.kv_dim
    t = s + m
    per = m * D * (H * dk + 2 * KV) + 2 * H * m * dk * t + m * H * dk * D + 3 * m * D * F
    tally.total.add(config.n_layers * per + (m * D * config.vocab_size if with_logits else 0))
    tally.attn_scores.add(config.n_layers * H * m * dk * t)


def bill_repair(tally, config: ModelConfig, s: int, k: int) -> None:
    """Books of the Stage-II repair of k tokens (dense k x s attention billing)."""
    if tally is None or k == 0:
        return
    H, dk, D, F, KV = config.n_heads, config.head_dim, config.hidden_dim, config.ffn_dim, config.kv_dim
    per = k * D * (H * dk + 2 * KV) + 2 * H * k * dk * s + k * H * dk * D + 3 * k * D * F
    tally.total.add(config.n_layers * per)
    tally.attn_scores.add(config.n_layers * H * k * dk * s)


class KVCache:
    """Context + query K/V handed to decoding (reference model.py:208-228).

    Device-backed: ``keys``/``values`` materialise per-layer f32 arrays lazily.
    """

    def __init__(self, keys, values, positions, last_logits=None):
        self._keys = keys
        self._values = values
        self.positions = positions
        self.last_logits = last_logits

    @property
    def keys(self):
        return self._keys() if callable(self._keys) else self._keys

    @property
    def values(self):
        return self._values() if callable(self._values) else self._values

    @property
    def length(self) -> int:
        return int(self.positions.shape[0])

    @classmethod
    def from_prefill(cls, trace) -> "KVCache":
        """Reference KVCache.from_prefill (model.py:221-228): host copies of a prefill."""
        return cls(keys=[np.array(k, copy=True) for k in trace.keys],
                   values=[np.array(v, copy=True) for v in trace.values],
                   positions=np.array(trace.positions, copy=True), last_logits=np.array(trace.logits[-1], copy=True))


# ---------------------------------------------------------------------------- device


def _pad2(t, rows, cols):
    import torch
    out = torch.zeros((rows, cols), dtype=t.dtype, device=t.device)
    out[: t.shape[0], : t.shape[1]] = t
    return out


def fp16_scaled(w):
    """(fp16 tensor, scale) with w ~= fp16_tensor * scale: the matrix is multiplied by
    2^e, e chosen so that max|w| * 2^e <= 2^15, before rounding to fp16 -- every
    bf16-exact weight down to ~2^-24 * 2^-e is represented exactly, larger dynamic
    ranges keep 11 significant bits.  The kernels multiply accumulators by 2^-e."""
    import torch
    mx = float(w.abs().max()) if w.numel() else 0.0
    e = 0 if not (mx > 0 and math.isfinite(mx)) else max(-60, min(60, math.floor(math.log2(32768.0 / mx))))
    return (w.float() * (2.0 ** e)).to(torch.float16).contiguous(), 2.0 ** -e


class DeviceModel:
    """fp16 (pre-scaled) device weights in the kernel layout + the C-ABI model handle."""

    def __init__(self, config: ModelConfig, tensors: dict, fingerprint: str, tp_rank: int = 0, tp_world: int = 1,
                 comm=None):
        torch = _lib.require_cuda()
        self.config = config
        self.lay = Layout.of(config)
        self.tp_rank, self.tp_world, self.comm = tp_rank, tp_world, comm
        # config of this rank's cache / chunk store (its KV heads only when head-sharded)
        self.cache_config = config if tp_world == 1 else shard_config(config, tp_world)
        self.fingerprint = fingerprint
        self.t = tensors  # keeps device memory alive
        L = config.n_layers
        self._layers = (_lib.LayerWeights * L)()
        for i in range(L):
            lt = tensors["layers"][i]
            self._layers[i] = _lib.LayerWeights(lt["attn_norm"].data_ptr(), lt["ffn_norm"].data_ptr(),
                                                lt["wqkv"].data_ptr(), lt["wo"].data_ptr(), lt["wgu"].data_ptr(),
                                                lt["wd"].data_ptr(), (ctypes.c_float * 4)(*lt["wscale"]))
        self._w = _lib.Weights(tensors["embed"].data_ptr(), tensors["final_norm"].data_ptr(),
                               tensors["lm_head"].data_ptr(), self._layers)
        self._cfg = config.c_struct()
        h = ctypes.c_void_p()
        _lib.check(_lib.load().pkv_model_create_sharded(ctypes.byref(self._cfg), ctypes.byref(self._w), tp_rank,
                                                        tp_world, comm, ctypes.byref(h)))
        self.handle = h
        self.device = tensors["embed"].device
        del torch

    def __del__(self):
        try:
            if getattr(self, "handle", None) and not getattr(self, "_view_of", None):
                _lib.load().pkv_model_destroy(self.handle)
        except Exception:
            pass

    @property
    def cfg_ptr(self):
        return ctypes.byref(self._cfg)

    # -- construction ---------------------------------------------------------
    @classmethod
    def from_host(cls, weights: ModelWeights, config: ModelConfig, device=None) -> "DeviceModel":
        """Upload reference-layout f32 weights: projections as pre-scaled fp16 (exact for
        bf16-exact weights), embed / lm_head as bf16 (RNE)."""
        torch = _lib.require_cuda()
        weights.validate(config)
        dev = device or torch.device("cuda", torch.cuda.current_device())

        def up(a):
            return torch.from_numpy(np.ascontiguousarray(a, dtype=F32)).to(dev)

        names = ("attn_norm", "wq", "wk", "wv", "wo", "ffn_norm", "w_gate", "w_up", "w_down")
        layers = ({k: up(getattr(lw, k)) for k in names} for lw in weights.layers)
        return cls._build(config, layers, up(weights.embed), up(weights.lm_head), up(weights.final_norm),
                          weights.fingerprint(config), dev)

    @classmethod
    def _build(cls, config: ModelConfig, layers_ref, embed, lm_head, final_norm, fingerprint: str, dev):
        """Device layout from reference-layout device tensors (input-major [fan_in, fan_out]
        projections, one dict per layer; consumed one layer at a time)."""
        torch = _lib.require_cuda()
        lay = Layout.of(config)
        H, Hkv, dk = config.n_heads, config.n_kv_heads, config.head_dim
        bf = torch.bfloat16

        def heads_rows(w, n_h):  # [D, n_h*dk] -> [n_h*dkp, Dp] (transposed, padded per head)
            t = w.float().t().reshape(n_h, dk, -1)
            out = torch.zeros((n_h, lay.dkp, lay.Dp), dtype=torch.float32, device=dev)
            out[:, :dk, : config.hidden_dim] = t
            return out.reshape(n_h * lay.dkp, lay.Dp)

        def norm(g):
            out = torch.zeros(lay.Dp, dtype=torch.float32, device=dev)
            out[: config.hidden_dim] = g.float()
            return out

        layers = []
        for lw in layers_ref:
            wqkv, s_qkv = fp16_scaled(torch.cat([heads_rows(lw["wq"], H), heads_rows(lw["wk"], Hkv),
                                                 heads_rows(lw["wv"], Hkv)]))
            wo = lw["wo"].float().t().reshape(config.hidden_dim, H, dk)
            wo_p = torch.zeros((lay.Dp, H, lay.dkp), dtype=torch.float32, device=dev)
            wo_p[: config.hidden_dim, :, :dk] = wo
            wo16, s_o = fp16_scaled(wo_p.reshape(lay.Dp, lay.HQ))
            del wo_p, wo
            g = _pad2(lw["w_gate"].float().t(), lay.Fp, lay.Dp).reshape(lay.Fp // 128, 128, lay.Dp)
            u = _pad2(lw["w_up"].float().t(), lay.Fp, lay.Dp).reshape(lay.Fp // 128, 128, lay.Dp)
            wgu, s_gu = fp16_scaled(torch.stack([g, u], dim=1).reshape(2 * lay.Fp, lay.Dp))
            del g, u
            wd, s_d = fp16_scaled(_pad2(lw["w_down"].float().t(), lay.Dp, lay.Fp))
            layers.append({"attn_norm": norm(lw["attn_norm"]), "ffn_norm": norm(lw["ffn_norm"]), "wqkv": wqkv,
                           "wo": wo16, "wgu": wgu, "wd": wd, "wscale": (s_qkv, s_o, s_gu, s_d)})
            del lw
        tensors = {"layers": layers,
                   "embed": _pad2(embed.to(bf), config.vocab_size, lay.Dp).contiguous(),
                   "lm_head": _pad2(lm_head.to(bf).t(), config.vocab_size, lay.Dp).contiguous(),
                   "final_norm": norm(final_norm)}
        return cls(config, tensors, fingerprint)

    @classmethod
    def synthetic(cls, config: ModelConfig, seed: int = 0, device=None) -> "DeviceModel":
        """Random-init weights generated on the device by the SYN1 generator
        (paper_2602_02579_b200/synthetic.py): the reference's initialisation scale, bf16-exact
        values that the CPU oracle rebuilds bit for bit (oracle/synthetic_inputs.py)."""
        from . import synthetic as S
        torch = _lib.require_cuda()
        dev = device or torch.device("cuda", torch.cuda.current_device())
        ones = torch.ones(config.hidden_dim, dtype=torch.float32, device=dev)

        def layers():
            for li in range(config.n_layers):
                d = S.layer_weights(config, li, seed, dev)
                d["attn_norm"], d["ffn_norm"] = ones, ones
                yield d
        return cls._build(config, layers(), S.embed(config, seed, dev), S.lm_head(config, seed, dev), ones,
                          f"syn1-{seed}", dev)

    random = synthetic  # benchmark weights (round-1 name)

    def shard(self, rank: int, world: int, comm) -> "DeviceModel":
        """Rank `rank`'s tensor-parallel slice of this model (include/pkv.h, "Head-sharded
        prefill"): its q/k/v head rows, wo head columns, gate/up 128-row blocks and wd
        columns; embed / lm_head / norm gains are shared (same device tensors)."""
        torch = _lib.require_cuda()
        cfg, lay = self.config, self.lay
        H, Hkv, dkp = cfg.n_heads, cfg.n_kv_heads, lay.dkp
        check_shardable(cfg, world)
        hl, kl, fl = H // world, Hkv // world, lay.Fp // world
        layers = []
        for lt in self.t["layers"]:
            wqkv = lt["wqkv"]
            q = wqkv[rank * hl * dkp:(rank + 1) * hl * dkp]
            k = wqkv[(H + rank * kl) * dkp:(H + (rank + 1) * kl) * dkp]
            v = wqkv[(H + Hkv + rank * kl) * dkp:(H + Hkv + (rank + 1) * kl) * dkp]
            layers.append({"attn_norm": lt["attn_norm"], "ffn_norm": lt["ffn_norm"],
                           "wqkv": torch.cat([q, k, v]).contiguous(),
                           "wo": lt["wo"][:, rank * hl * dkp:(rank + 1) * hl * dkp].contiguous(),
                           "wgu": lt["wgu"][2 * rank * fl:2 * (rank + 1) * fl].contiguous(),
                           "wd": lt["wd"][:, rank * fl:(rank + 1) * fl].contiguous(), "wscale": lt["wscale"]})
        tensors = {"layers": layers, "embed": self.t["embed"], "lm_head": self.t["lm_head"],
                   "final_norm": self.t["final_norm"]}
        return DeviceModel(cfg, tensors, self.fingerprint, rank, world, comm)

    def rows(self, comm) -> "DeviceModel":
        """This (unsharded) model with a token-parallel Stage II over comm's ranks
        (pkv_recompute_rows): every rank holds the full weights and a full cache, the
        scoring pass is replicated, and the repair of the selected rows is split by
        attention unit with one all-gather of fresh cache entries per layer.  Shares the
        device tensors and the C model handle."""
        if self.tp_world != 1:
            raise ConfigError("token-parallel Stage II needs the unsharded model")
        view = object.__new__(DeviceModel)
        view.__dict__.update(self.__dict__)
        view._view_of = self  # keeps the owner (and its C handle) alive; the view never frees it
        view.rows_comm = comm
        return view

    def weight_bytes(self, include_head: bool = True) -> int:
        n = 0
        for lt in self.t["layers"]:
            n += sum(lt[k].numel() * lt[k].element_size() for k in ("wqkv", "wo", "wgu", "wd"))
        if include_head:
            n += self.t["lm_head"].numel() * 2
        return n


def check_shardable(cfg: ModelConfig, world: int) -> None:
    lay = Layout.of(cfg)
    if world < 1 or cfg.n_kv_heads % world or (lay.Fp // 128) % world:
        raise ConfigError(f"cannot head-shard {cfg.n_kv_heads} KV heads / {lay.Fp // 128} ffn blocks over {world} ranks")


def shard_config(cfg: ModelConfig, world: int) -> ModelConfig:
    """Config of one rank's cache and chunk store under head sharding: its H/W query
    heads and Hkv/W KV heads (hidden/ffn sizes are those of the local view)."""
    check_shardable(cfg, world)
    hl = cfg.n_heads // world
    return ModelConfig(cfg.n_layers, hl, cfg.n_kv_heads // world, cfg.head_dim, hl * cfg.head_dim,
                       Layout.of(cfg).Fp // world, cfg.vocab_size, cfg.rope_theta, cfg.norm_eps)


def resolve_device_model(weights, config: ModelConfig) -> DeviceModel:
    """Accept either host ModelWeights (uploaded once, cached) or a DeviceModel."""
    if isinstance(weights, DeviceModel):
        return weights
    if isinstance(weights, ModelWeights):
        return weights.device(config)
    # reference pikv.ModelWeights (duck-typed): same field names
    if hasattr(weights, "layers") and hasattr(weights, "embed"):
        import torch
        key = (config, torch.cuda.current_device())
        cache = getattr(weights, "__b200_device__", None)
        if cache is not None and getattr(cache, "_cache_key", None) != key:
            cache = None  # uploaded under another config / device
        if cache is None:
            mw = ModelWeights(embed=weights.embed, layers=[LayerWeights(**{k: getattr(lw, k) for k in (
                "attn_norm", "wq", "wk", "wv", "wo", "ffn_norm", "w_gate", "w_up", "w_down")})
                for lw in weights.layers], final_norm=weights.final_norm, lm_head=weights.lm_head)
            cache = DeviceModel.from_host(mw, config)
            cache.fingerprint = weights.fingerprint(config) if hasattr(weights, "fingerprint") else cache.fingerprint
            cache._cache_key = key
            try:
                weights.__b200_device__ = cache
            except AttributeError:
                pass
        return cache
    raise EngineError(f"unsupported weights object {type(weights)!r}")
