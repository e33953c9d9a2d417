"""The C-ABI library loads and exports every entry point include/pkv.h declares;
host-only calls (layout, validation, error mapping) work without a GPU."""

import ctypes
import re
from pathlib import Path

import pytest

import paper_2602_02579_b200 as P
from paper_2602_02579_b200 import _lib

HEADER = Path(__file__).resolve().parent.parent / "include" / "pkv.h"


def declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|void|const char\*|uint64_t)\s+(pkv_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__.build()
    return _lib.load()


def test_header_declares_the_api():
    names = declared()
    for n in ("pkv_assemble", "pkv_query_pass", "pkv_fuse_select", "pkv_topk", "pkv_recompute",
              "pkv_replace_entries", "pkv_cache_view", "pkv_model_create"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    for name in declared():
        assert hasattr(lib, name), name
    assert set(declared()) == set(_lib.EXPORTED_SYMBOLS)


def test_sm100a_code_in_library():
    import subprocess
    so = Path(_lib.LIB_PATH)
    if not so.exists():
        pytest.skip("library not built")
    out = subprocess.run(["cuobjdump", "-lelf", str(so)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_layout_and_config_validation(lib):
    cfg = P.ModelConfig(32, 32, 8, 128, 4096, 14336, 128256, 500000.0)
    out = (ctypes.c_int32 * 5)()
    _lib.check(lib.pkv_layout(ctypes.byref(cfg.c_struct()), out))
    assert list(out) == [128, 4096, 14336, 6144, 4096]
    assert P.model.Layout.of(cfg) == P.model.Layout(*list(out))
    tiny = P.ModelConfig(2, 2, 1, 4, 8, 16, 50)
    _lib.check(lib.pkv_layout(ctypes.byref(tiny.c_struct()), out))
    assert list(out) == [64, 64, 128, 256, 128]
    bad = _lib.Config(2, 3, 2, 4, 12, 16, 50, 1e4, 1e-5)
    with pytest.raises(P.ConfigError):
        _lib.check(lib.pkv_layout(ctypes.byref(bad), out))
    big = _lib.Config(1, 2, 2, 256, 512, 16, 50, 1e4, 1e-5)
    with pytest.raises(P.ConfigError, match="head_dim"):
        _lib.check(lib.pkv_layout(ctypes.byref(big), out))


def test_topk_rejects_bad_k_before_any_launch(lib):
    with pytest.raises(P.ArgumentError):
        _lib.check(lib.pkv_topk(None, 10, 11, None, None, None))
    with pytest.raises(P.ArgumentError):
        _lib.check(lib.pkv_fuse_select(None, 2, 10, -1, None, None, None, None, 0, None))


def test_product_path_fails_loudly_without_cuda(monkeypatch):
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    cfg = P.ModelConfig(2, 2, 1, 4, 8, 16, 50)
    w = P.random_weights(cfg, 0)
    with pytest.raises(P.EngineError):
        P.DeviceModel.from_host(w, cfg)
    with pytest.raises(P.EngineError):
        P.top_k_indices([1.0, 2.0], 1)
