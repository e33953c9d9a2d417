"""PKVC chunk files: round trip, byte compatibility with the reference's
own store_chunk/load_chunk (when the reference is mounted), and the error taxonomy of
reference tests/test_chunkstore.py:82-124."""

import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2602_02579_b200 as P
from oracle import pikv_oracle as O

REF = Path("/root/reference/pkg/src")


@pytest.fixture(scope="module")
def chunk():
    cfg = O.Cfg(2, 4, 2, 8, 32, 64, 50)
    w = O.init_weights(cfg, 3)
    c = O.make_chunk(w, cfg, [3, 17, 42, 0, 9, 31, 7])
    return P.ChunkKV(c.chunk_id, c.fp, c.token_ids, c.k_nr, c.v)


def test_roundtrip_is_byte_stable(tmp_path, chunk):
    a = tmp_path / "a.pkvc"
    P.store_chunk(chunk, a)
    got = P.load_chunk(a)
    assert got.chunk_id == P.chunk_content_id(chunk.config_fingerprint, chunk.token_ids)
    assert got.config_fingerprint == chunk.config_fingerprint
    np.testing.assert_array_equal(got.token_ids, chunk.token_ids)
    for li in range(len(chunk.keys_norope)):
        np.testing.assert_array_equal(got.keys_norope[li], chunk.keys_norope[li])
        np.testing.assert_array_equal(got.values[li], chunk.values[li])
    b = tmp_path / "b.pkvc"
    P.store_chunk(got, b)
    assert a.read_bytes() == b.read_bytes()


@pytest.mark.skipif(not REF.exists(), reason="reference package not mounted")
def test_files_are_interchangeable_with_the_reference(tmp_path, chunk):
    sys.path.insert(0, str(REF))
    import pikv
    ours, theirs = tmp_path / "ours.pkvc", tmp_path / "theirs.pkvc"
    P.store_chunk(chunk, ours)
    ref_chunk = pikv.chunkstore.load_chunk(ours)
    pikv.chunkstore.store_chunk(ref_chunk, theirs)
    assert ours.read_bytes() == theirs.read_bytes()
    back = P.load_chunk(theirs)
    for li in range(len(chunk.keys_norope)):
        np.testing.assert_array_equal(back.keys_norope[li], ref_chunk.keys_norope[li])


def test_error_taxonomy(tmp_path, chunk):
    path = tmp_path / "c.pkvc"
    P.store_chunk(chunk, path)
    data = path.read_bytes()
    bad = tmp_path / "bad.pkvc"
    cases = [(b"NOPE" + data[4:], P.FormatError), (data[:6], P.TruncatedError), (data[:-8], P.TruncatedError),
             (data[:4] + b"\xff\xff" + data[6:], P.FormatError)]
    hlen = int.from_bytes(data[6:10], "little")
    cases.append((data[:10] + b"{" * hlen + data[10 + hlen:], P.FormatError))
    for blob, err in cases:
        bad.write_bytes(blob)
        with pytest.raises(err):
            P.load_chunk(bad)
    assert issubclass(P.TruncatedError, P.FormatError)


def test_content_addressed_name(chunk):
    from paper_2602_02579_b200.chunkfile import chunk_path
    assert chunk_path("/s", 0xab) == "/s/00000000000000ab.pkvc"
