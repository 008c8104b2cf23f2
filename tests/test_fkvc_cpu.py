"""FKVC record files (serialize_record / deserialize_record) on
the host: byte layout pinned against an independent numpy writer/reader of
the spec's layout, bit-exact round trips, and the FormatError kinds of
common.hpp:33 (bad magic, version mismatch, truncation, malformed)."""
import struct

import numpy as np
import pytest

from paper_2601_12904_b200 import fusion as F


def _spec_bytes(cid, variant, native, k, v):
    # magic "FKVC", version u32, chunk_id (16 bytes), variant u8,
    # native_start u32, layers u16, heads u16, head_dim u16, tokens u32, then
    # per-layer K then V, little-endian fp32
    L, n, H, dh = k.shape
    out = b"FKVC" + struct.pack("<I", 1) + bytes(cid.bytes) + struct.pack("<BIHHHI", variant, native, L, H, dh, n)
    for l in range(L):
        out += k[l].astype("<f4").tobytes() + v[l].astype("<f4").tobytes()
    return out


def _rec(seed=0, shape=(3, 5, 2, 8)):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(shape).astype(np.float32), rng.standard_normal(shape).astype(np.float32)


def test_fkvc_layout_matches_spec(tmp_path):
    k, v = _rec()
    cid = F.hash_tokens([1, 2, 3])
    p = tmp_path / "a.fkvc"
    F.fkvc_write(p, cid, k, v, native_start=9, variant=F.FUSED)
    assert p.read_bytes() == _spec_bytes(cid, 1, 9, k, v)
    h, k2, v2 = F.fkvc_read(p)
    assert h["id"] == cid and h["variant"] == F.FUSED and h["native_start"] == 9
    assert (h["layers"], h["tokens"], h["heads"], h["head_dim"]) == k.shape
    assert np.array_equal(k, k2) and np.array_equal(v, v2)


def test_fkvc_reads_spec_written_file(tmp_path):
    k, v = _rec(1, (2, 7, 1, 4))
    cid = F.hash_tokens([5])
    p = tmp_path / "b.fkvc"
    p.write_bytes(_spec_bytes(cid, 0, 1, k, v))
    h, k2, v2 = F.fkvc_read(p)
    assert h["id"] == cid and np.array_equal(k, k2) and np.array_equal(v, v2)


@pytest.mark.parametrize("mutate,kind", [
    (lambda b: b"FKVX" + b[4:], "BadMagic"),
    (lambda b: b[:4] + struct.pack("<I", 2) + b[8:], "BadVersion"),
    (lambda b: b[:20], "Truncated"),
    (lambda b: b[:-4], "Truncated"),
    (lambda b: b[:24] + bytes([7]) + b[25:], "Malformed"),
])
def test_fkvc_format_errors(tmp_path, mutate, kind):
    k, v = _rec(2)
    cid = F.hash_tokens([9, 9])
    good = _spec_bytes(cid, 0, 3, k, v)
    p = tmp_path / "bad.fkvc"
    p.write_bytes(mutate(good))
    with pytest.raises(F.FormatError) as ei:
        F.fkvc_read(p)
    assert ei.value.kind == kind


def test_fkvc_missing_file_is_io_error(tmp_path):
    with pytest.raises(F.FormatError) as ei:
        F.fkvc_read(tmp_path / "nope.fkvc")
    assert ei.value.kind == "Io"
