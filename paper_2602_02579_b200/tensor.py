"""Selection primitives of the drop-in (reference tensor.py:117-140).

``top_k_indices`` runs the device radix select (kernel K4); ``ratio_budget`` is
host arithmetic in Python double on purpose -- ``ceil(0.07*100) == 8`` is part
of the reference's contract and must never be recomputed on the device.
"""

from __future__ import annotations

import math

import numpy as np

from . import _lib
from .errors import ArgumentError, NumericsError, ShapeError
from .model import FlopCounter  # noqa: F401  (re-export, reference tensor.py:37-46)


def ratio_budget(p: float, n: int) -> int:
    """Selection budget k = ceil(p * n) for p in [0, 1] (reference tensor.py:136-140)."""
    if not 0.0 <= p <= 1.0:
        raise ArgumentError(f"recompute ratio must lie in [0, 1], got {p}")
    return math.ceil(p * n)


def device_topk(scores_dev, k: int, stream=None):
    """k largest of a device f32 vector, ties toward the smaller index, ascending.
    Returns (idx int32 device tensor [k], status int32 device tensor [1])."""
    torch = _lib.require_cuda()
    n = int(scores_dev.shape[0])
    idx = torch.empty(max(k, 1), dtype=torch.int32, device=scores_dev.device)
    status = torch.zeros(1, dtype=torch.int32, device=scores_dev.device)
    _lib.check(_lib.load().pkv_topk(scores_dev.data_ptr(), n, int(k), idx.data_ptr(), status.data_ptr(),
                                    _lib.stream_ptr(torch, stream)))
    return idx[:k], status


def top_k_indices(scores, k: int) -> list:
    """Indices of the k largest scores; ties break toward the smaller index; the
    result is sorted ascending (reference tensor.py:117-133)."""
    torch = _lib.require_cuda()
    if isinstance(scores, torch.Tensor):
        s = scores.detach().to(torch.float32)
        if s.dim() != 1:
            raise ShapeError(f"top_k_indices expects a 1-D score vector, got {tuple(s.shape)}")
        n = int(s.shape[0])
    else:
        a = np.asarray(scores, dtype=np.float32)
        if a.ndim != 1:
            raise ShapeError(f"top_k_indices expects a 1-D score vector, got {a.shape}")
        n = int(a.shape[0])
        s = None
    if k < 0:
        raise ArgumentError(f"k must be >= 0, got {k}")
    if k > n:
        raise ArgumentError(f"k={k} exceeds the {n} available scores")
    if n == 0:
        return []
    if s is None:
        s = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    s = s.contiguous().cuda()
    idx, status = device_topk(s, k)
    st = int(status.item())
    if st == 7:
        raise NumericsError("non-finite values in top-k scores")
    _lib.check(st)
    return [int(i) for i in idx.cpu().tolist()]
