"""SYN1 synthetic inputs: the device generator (paper_2602_02579_b200/synthetic.py, run
here on the CPU through the same torch code) and the oracle's numpy restatement
(oracle/synthetic_inputs.py) produce identical bytes; the values have the reference's
initialisation scale (model.py:163-185)."""

import math

import numpy as np
import pytest

from oracle import pikv_oracle as O
from oracle import synthetic_inputs as SO

torch = pytest.importorskip("torch")


@pytest.mark.parametrize("shape,tid,std", [((257, 33), 5, 1.0), ((4096, 64), 0x0FFFFFF0, 1 / 64),
                                           ((3, 2, 128), 0x10000803, 1.0)])
def test_device_and_host_generators_agree(shape, tid, std):
    from paper_2602_02579_b200 import synthetic as S
    for seed in (0, 1, 12345):
        dev = S.normal_bf16(shape, seed, tid, std, device="cpu", block=1000).float().numpy()
        host = SO.normal_f32(shape, seed, tid, std, block=777)
        assert np.array_equal(dev, host)
        assert np.array_equal(O.bf16_round(host), host)  # bf16-exact
    ids_d = S.token_ids(1000, 128256, 3, S.TID_QUERY, device="cpu").numpy()
    assert np.array_equal(ids_d, SO.token_ids(1000, 128256, 3, SO.TID_QUERY))
    assert ids_d.min() >= 0 and ids_d.max() < 128256


def test_scale_and_moments():
    x = SO.normal_f32((1 << 20,), 0, 1, 1.0).astype(np.float64)
    assert abs(x.mean()) < 3e-3 and abs(x.std() - 1.0) < 3e-3
    assert np.abs(x).max() <= 131070 / SO.IH4_SD * 1.01  # Irwin-Hall(4) is bounded at ~3.46 sd
    w = SO.normal_f32((4096, 512), 0, 2, 1 / math.sqrt(4096)).astype(np.float64)
    assert abs(w.std() * math.sqrt(4096) - 1.0) < 1e-2
    # distinct tensors / seeds are decorrelated
    a, b = SO.normal_f32((1 << 16,), 0, 1, 1.0), SO.normal_f32((1 << 16,), 0, 2, 1.0)
    c = SO.normal_f32((1 << 16,), 1, 1, 1.0)
    assert abs(np.corrcoef(a, b)[0, 1]) < 0.02 and abs(np.corrcoef(a, c)[0, 1]) < 0.02
