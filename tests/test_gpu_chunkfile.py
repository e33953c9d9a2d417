"""Chunk files straight into pinned bf16 host buffers (chunkfile.load_chunk_pinned) give
exactly the scores of the same chunks uploaded from host f32 arrays."""

import numpy as np
import pytest

from test_gpu_parity import _device_inputs, _materialise, _setup

pytestmark = pytest.mark.gpu


def test_pinned_chunk_files_score_identically(built, tmp_path):
    import torch
    P = built
    cfg_o, seed, units, query, p = _materialise("c1")
    w, chunks = _setup(cfg_o, seed, units, query)
    cfg, mw, dch = _device_inputs(P, cfg_o, w, chunks)
    paths = []
    for i, c in enumerate(dch):
        paths.append(tmp_path / f"{i}.pkvc")
        P.store_chunk(c, paths[-1])
    runs = []
    for src in (dch, [P.load_chunk_pinned(pth, cfg) for pth in paths]):
        cache = P.assemble(src, cfg, fp32_taps=False)
        sc = P.score_prophet(mw, cfg, cache, query)
        torch.cuda.synchronize()
        runs.append((sc.per_layer, P.select_top_p(sc, p).indices))
    assert np.array_equal(runs[0][0], runs[1][0])
    assert runs[0][1] == runs[1][1]
