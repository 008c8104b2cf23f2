"""C-ABI boundary checks that need no GPU: libfrag.so loads, exports every
symbol include/frag/frag_c.h declares, reports errors with the reference's
taxonomy, and the C++ wrapper (frag/fusion.hpp, frag/core.hpp) compiles,
links and agrees with the library on hash_tokens."""
import ctypes as C
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2601_12904_b200 import _lib as L
from paper_2601_12904_b200 import fusion as F

ROOT = Path(__file__).resolve().parent.parent


def test_exports_every_declared_symbol():
    declared = L.declared_symbols()
    assert len(declared) >= 36
    out = subprocess.run(["nm", "-D", "--defined-only", str(L.LIB_PATH)], capture_output=True, text=True,
                         check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    assert set(L._SIGS) == set(declared)  # the ctypes binding covers the whole header


def test_oracle_presets_equal_library_presets():
    """bench.py's oracle legs read the shapes from oracle/presets.py (plain
    data, so the reference arm never maps libfrag.so); they must equal the
    library's frag_model_preset table."""
    from oracle import presets as OP
    for name, want in OP.PRESETS.items():
        assert F.preset(name).as_dict() == pytest.approx(want), name


def test_presets_match_survey_table():
    c = F.preset("llama3-8b")
    assert (c.layers, c.d_model, c.n_heads, c.n_kv_heads, c.head_dim, c.ffn_dim, c.vocab) == \
        (32, 4096, 32, 8, 128, 14336, 128256)
    t = F.preset("tiny")
    assert (t.layers, t.d_model, t.n_heads, t.head_dim, t.vocab) == (2, 256, 4, 64, 256)
    m = F.preset("mistral-7b")
    assert m.vocab == 32768 and m.rope_base == 1e6
    s = F.preset("llama3-70b")
    assert (s.layers, s.d_model, s.n_heads, s.n_kv_heads, s.ffn_dim) == (80, 8192, 64, 8, 28672)
    with pytest.raises(F.ContractError):
        F.preset("gpt-5")


def test_hash_tokens_semantics():
    a = F.hash_tokens([1, 2, 3])
    assert a == F.hash_tokens([1, 2, 3])
    assert a != F.hash_tokens([1, 2, 4]) and a != F.hash_tokens([3, 2, 1]) and a != F.hash_tokens([1, 2, 3], salt=1)
    assert F.hash_tokens([]) != F.hash_tokens([0])
    ids = {F.hash_tokens(list(np.random.default_rng(i).integers(0, 1000, 16))).hex() for i in range(2000)}
    assert len(ids) == 2000


def test_no_device_is_a_loud_cuda_error():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    with pytest.raises(F.CudaError, match="no CUDA device"):
        F.Engine("tiny")
    with pytest.raises(F.CudaError):
        F.ChunkKVStore(F.preset("tiny"))


def test_contract_errors_before_any_device_work():
    cfg = F.preset("tiny")
    cfg.head_dim = 48  # unsupported head_dim -> ContractError, not a silent fallback
    with pytest.raises(F.ContractError):
        F.Engine(cfg)
    cfg = F.preset("tiny")
    cfg.n_kv_heads = 3
    with pytest.raises(F.ContractError):
        F.Engine(cfg)


def test_shared_v_switch_is_process_wide_and_queryable():
    """frag_set_shared_v: -1 queries, 1 / 0 set and return the previous value
    (no device needed; the request path reads it)."""
    prev = F.set_shared_v(None)
    assert prev is True  # default on (FRAG_SHARED_V unset)
    assert F.set_shared_v(False) is True
    assert F.set_shared_v(None) is False
    assert F.set_shared_v(True) is False
    assert F.set_shared_v(None) is True


def _gxx():
    for c in ("/usr/bin/g++", shutil.which("g++")):
        if c and Path(c).exists():
            return c
    pytest.skip("no g++")


def test_cpp_wrapper_compiles_links_and_hash_agrees(tmp_path):
    exe = tmp_path / "reprocess_demo"
    subprocess.run([_gxx(), "-std=c++20", "-O1", f"-I{ROOT / 'include'}", str(ROOT / "examples" / "reprocess_demo.cpp"),
                    f"-L{L.LIB_PATH.parent}", "-lfrag", f"-Wl,-rpath,{L.LIB_PATH.parent}", "-o", str(exe)],
                   check=True, capture_output=True)
    r = subprocess.run([str(exe), "--hash", "5", "17", "255", "128000"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    lib_hex, hdr_hex = r.stdout.split()
    assert lib_hex == hdr_hex == F.hash_tokens([5, 17, 255, 128000]).hex()


def test_core_header_rng_matches_reference_goldens(tmp_path):
    import json
    gold = json.loads((ROOT / "tests" / "golden" / "rng_kat.json").read_text())["vectors"]["42"]
    src = tmp_path / "rng.cpp"
    src.write_text('#include "frag/core.hpp"\n#include <cstdio>\nint main(){frag::Rng r(42);'
                   'for(int i=0;i<16;++i)std::printf("%llu\\n",(unsigned long long)r.next_u64());'
                   'frag::Rng n(42);for(int i=0;i<16;++i)std::printf("%.17g\\n",n.normal());'
                   'frag::Rng b(42);for(int i=0;i<32;++i)std::printf("%llu\\n",(unsigned long long)b.below(256));}')
    exe = tmp_path / "rng"
    subprocess.run([_gxx(), "-std=c++20", "-O2", f"-I{ROOT / 'include'}", str(src), "-o", str(exe)], check=True)
    vals = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    assert vals[:16] == gold["next_u64"]
    assert [float(v) for v in vals[16:32]] == gold["normal"]
    assert [int(v) for v in vals[32:]] == gold["below_256"]
