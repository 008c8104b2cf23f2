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


def _manifest(tmp_path, n=3, mutate=None):
    import json
    recs = []
    for i in range(n):
        k, v = _rec(10 + i, (2, 4 + i, 2, 8))
        toks = list(range(i, i + 4 + i))
        cid = F.hash_tokens(toks)
        name = f"{cid.hex()}.fkvc"
        F.fkvc_write(tmp_path / name, cid, k, v, native_start=3 + i, variant=i % 2)
        recs.append({"chunk_id": cid.hex(), "path": name, "variant": ["ISOLATED", "FUSED"][i % 2],
                     "native_start": 3 + i, "tokens": toks})
    doc = {"format": "FKVC-manifest", "version": 1, "records": recs}
    if mutate:
        doc = mutate(doc)
    p = tmp_path / "manifest.json"
    p.write_text(doc if isinstance(doc, str) else json.dumps(doc))
    return p


def test_manifest_written_independently_validates(tmp_path):
    """SPEC.md:322 manifest (chunk_id -> relative path + variant +
    native_start, plus the token ids FKVC omits), written here by Python's
    json module, is read by the library's parser and checked against every
    file header."""
    assert F.manifest_validate(_manifest(tmp_path)) == 3


@pytest.mark.parametrize("mutate,kind", [
    (lambda d: "{\"format\": \"FKVC-manifest\", \"version\": 1, \"records\": [", "Malformed"),
    (lambda d: {**d, "version": 2}, "BadVersion"),
    (lambda d: {**d, "format": "other"}, "Malformed"),
    (lambda d: {**d, "records": [{**d["records"][0], "chunk_id": d["records"][1]["chunk_id"]}]}, "Malformed"),
    (lambda d: {**d, "records": [{**d["records"][0], "native_start": 99}]}, "Malformed"),
    (lambda d: {**d, "records": [{**d["records"][0], "tokens": [1]}]}, "Malformed"),
    (lambda d: {**d, "records": [{**d["records"][0], "path": "missing.fkvc"}]}, "Io"),
])
def test_manifest_errors(tmp_path, mutate, kind):
    p = _manifest(tmp_path, mutate=mutate)
    with pytest.raises(F.FormatError) as ei:
        F.manifest_validate(p)
    assert ei.value.kind == kind


def test_cpp_wrapper_maps_format_error_kinds(tmp_path):
    """frag::check re-throws FRAG_E_FORMAT as FormatError with the library's
    kind (common.hpp:33), not a blanket Malformed."""
    import shutil
    import subprocess
    from pathlib import Path
    from paper_2601_12904_b200 import _lib as L
    gxx = shutil.which("g++")
    if not gxx:
        pytest.skip("no g++")
    root = Path(__file__).resolve().parent.parent
    src = tmp_path / "kinds.cpp"
    src.write_text('#include "frag/fusion.hpp"\n#include <cstdio>\n'
                   'int main(int argc, char** argv){ frag_fkvc_header h{};\n'
                   '  try { frag::check(frag_fkvc_read(argv[1], &h, nullptr, nullptr, 0)); return 9; }\n'
                   '  catch (const frag::FormatError& e) { std::printf("%d\\n", (int)e.kind()); return 0; } }\n')
    exe = tmp_path / "kinds"
    subprocess.run([gxx, "-std=c++20", f"-I{root / 'include'}", str(src), f"-L{L.LIB_PATH.parent}", "-lfrag",
                    f"-Wl,-rpath,{L.LIB_PATH.parent}", "-o", str(exe)], check=True, capture_output=True)
    k, v = _rec(3)
    good = _spec_bytes(F.hash_tokens([1]), 0, 1, k, v)
    cases = {"bad_magic": (b"XXXX" + good[4:], 0), "bad_version": (good[:4] + struct.pack("<I", 9) + good[8:], 1),
             "truncated": (good[:30], 2), "malformed": (good[:24] + bytes([5]) + good[25:], 3)}
    for name, (blob, want) in cases.items():
        p = tmp_path / f"{name}.fkvc"
        p.write_bytes(blob)
        r = subprocess.run([str(exe), str(p)], capture_output=True, text=True)
        assert r.returncode == 0 and int(r.stdout) == want, (name, r.stdout, r.stderr)
    r = subprocess.run([str(exe), str(tmp_path / "none.fkvc")], capture_output=True, text=True)
    assert int(r.stdout) == 4  # Io
