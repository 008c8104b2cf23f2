"""End-to-end reprocessing on the GPU through the C ABI: store semantics,
endpoint reductions (r=0 = Full Reuse, r=1 = Full Attention)
and the invariants of SPEC.md:448 and SPEC.md:173."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tiny(cuda):
    from paper_2601_12904_b200 import fusion as F
    eng = F.Engine("tiny", seed=1234)
    store = F.ChunkKVStore(eng.cfg)
    rng = np.random.default_rng(5)
    system = rng.integers(0, eng.cfg.vocab, 8).tolist()
    chunks = [rng.integers(0, eng.cfg.vocab, 256).tolist() for _ in range(8)]
    ids = [eng.preprocess_isolated(store, c, system=system) for c in chunks]
    question = rng.integers(0, eng.cfg.vocab, 32).tolist()
    res = F.Result(eng, 8 + 8 * 256 + 32 + 64)
    return dict(F=F, eng=eng, store=store, system=system, chunks=chunks, ids=ids, question=question, res=res)


def test_store_semantics(tiny):
    F, store, ids, chunks = tiny["F"], tiny["store"], tiny["ids"], tiny["chunks"]
    assert len(store) == 8
    r = store.peek(ids[0])
    assert r.n_tok == 256 and r.native_start == 9 and r.variant == F.ISOLATED
    h0 = r.heat
    store.fetch(ids[0])
    store.fetch(ids[0])
    assert store.peek(ids[0]).heat == h0 + 2
    store.release(ids[0])
    store.release(ids[0])
    with pytest.raises(F.StoreError):  # duplicate without overwrite
        tiny["eng"].preprocess_isolated(store, chunks[0], system=tiny["system"])
    with pytest.raises(F.StoreError):
        store.fetch(F.hash_tokens([1, 2, 3]))


def test_reprocess_runs_and_selects(tiny):
    eng, store, res = tiny["eng"], tiny["store"], tiny["res"]
    eng.reprocess(store, tiny["question"], tiny["ids"], 0.15, res, system=tiny["system"], timing=True)
    lg = res.logits()
    assert lg.shape == (1, eng.cfg.vocab) and np.isfinite(lg).all()
    crit = res.crit()
    N = 8 * 256
    assert len(crit) == int(np.floor(0.15 * N + 0.5))
    assert np.all(np.diff(crit) > 0)
    assert crit.min() >= 9 and crit.max() <= 8 + N  # never system or question tokens
    t = res.timing()
    assert t["total_ms"] > 0


def test_concurrent_requests_on_one_engine(tiny):
    """Host threads issuing requests on their own streams and results: the
    engine serialises their device work (its persistent GEMMs assume they own
    the GPU), and every request gets the logits of a sequential run."""
    import threading

    import torch
    F, eng, store, ids, q = tiny["F"], tiny["eng"], tiny["store"], tiny["ids"], tiny["question"]
    sys_ = tiny["system"]
    want = {}
    for k, r in enumerate((0.05, 0.15, 0.3, 1.0)):
        eng.reprocess(store, q, ids[k:], r, tiny["res"], system=sys_)
        want[k] = tiny["res"].logits().copy()
    got, err = {}, []

    def worker(k, r):
        try:
            res = F.Result(eng, 8 + 8 * 256 + 32 + 64)
            st = torch.cuda.Stream()
            for _ in range(3):
                eng.reprocess(store, q, ids[k:], r, res, system=sys_, stream=st.cuda_stream)
            got[k] = res.logits().copy()
        except Exception as ex:  # surfaced below
            err.append(ex)

    ths = [threading.Thread(target=worker, args=(k, r)) for k, r in enumerate((0.05, 0.15, 0.3, 1.0))]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=300)
    assert not err, err
    for k in want:
        assert np.array_equal(got[k], want[k]), k


def test_store_immutable_during_reprocess(tiny):
    store, ids = tiny["store"], tiny["ids"]
    before = [store.read_kv(i) for i in ids[:2]]
    tiny["eng"].reprocess(store, tiny["question"], ids, 0.3, tiny["res"], system=tiny["system"])
    after = [store.read_kv(i) for i in ids[:2]]
    for (k0, v0), (k1, v1) in zip(before, after):
        assert np.array_equal(k0, k1) and np.array_equal(v0, v1)


def test_endpoint_r1_equals_full_attention(tiny):
    F, eng = tiny["F"], tiny["eng"]
    res = tiny["res"]
    eng.reprocess(tiny["store"], tiny["question"], tiny["ids"], 1.0, res, system=tiny["system"])
    lg1 = res.logits()
    k1, v1 = res.fused_kv()
    fa = F.Result(eng, res.max_tokens)
    tokens = [t for c in tiny["chunks"] for t in c] + tiny["question"]
    eng.full_prefill(tokens, fa, system=tiny["system"])
    lgf = fa.logits()
    kf, vf = fa.fused_kv()
    # identical kernels on identical rows: bit-identical
    assert np.array_equal(k1, kf) and np.array_equal(v1, vf)
    assert np.array_equal(lg1, lgf)


def test_single_chunk_native_offset_is_bit_copy(tiny):
    # one chunk at its native offset -> stitched KV bit-equal to the record
    eng, store = tiny["eng"], tiny["store"]
    res = tiny["res"]
    eng.reprocess(store, tiny["question"], tiny["ids"][:1], 0.0, res, system=tiny["system"])
    k, v = res.fused_kv()
    rk, rv = store.read_kv(tiny["ids"][0])
    L_ = eng.cfg.layers
    # rows S..S+n-1 hold the record untouched (r=0: nothing recomputed there)
    assert np.array_equal(k[:, 8:8 + 256], rk) and np.array_equal(v[:, 8:8 + 256], rv)


def test_graph_replay_matches_eager(tiny):
    """The request body is replayed from a CUDA graph from the second request of
    a shape on; replays must reproduce the eager (timing=True) run bit for bit,
    including when a same-shape request brings different chunks / RoPE deltas /
    question tokens (the graph reads them from the per-request staging)."""
    eng, store, res, ids = tiny["eng"], tiny["store"], tiny["res"], tiny["ids"]
    q2 = list(reversed(tiny["question"]))
    order_b = ids[4:] + ids[:4]  # same shape, different deltas per chunk
    outs = {}
    for name, q, order in (("a", tiny["question"], ids), ("b", q2, order_b)):
        eng.reprocess(store, q, order, 0.2, res, system=tiny["system"], timing=True)
        outs[name] = (res.logits().copy(), res.crit().copy())
    for rep in range(3):
        for name, q, order in (("a", tiny["question"], ids), ("b", q2, order_b)):
            eng.reprocess(store, q, order, 0.2, res, system=tiny["system"])
            lg, crit = res.logits(), res.crit()
            assert np.array_equal(crit, outs[name][1]), (rep, name)
            assert np.array_equal(lg, outs[name][0]), (rep, name)
    assert not np.array_equal(outs["a"][0], outs["b"][0])


def test_decode_r1_equals_full_attention_decode(tiny):
    """sparse_prefill_and_decode endpoint: with r=1 the greedy
    answer equals Full Attention greedy decoding, bit for bit (same kernels)."""
    F, eng = tiny["F"], tiny["eng"]
    T = 8 + 8 * 256 + 32
    n = 6
    ra = F.Result(eng, T + n)
    eng.reprocess(tiny["store"], tiny["question"], tiny["ids"], 1.0, ra, system=tiny["system"])
    ta = eng.decode(ra, n)
    fa = F.Result(eng, T + n)
    tokens = [t for c in tiny["chunks"] for t in c] + tiny["question"]
    eng.full_prefill(tokens, fa, system=tiny["system"])
    tb = eng.decode(fa, n)
    assert np.array_equal(ta, tb)
    assert np.array_equal(ra.logits(), fa.logits())
    ka, va = ra.fused_kv()
    kb, vb = fa.fused_kv()
    assert ka.shape[1] == T + n - 1
    assert np.array_equal(ka, kb) and np.array_equal(va, vb)


def test_decode_contract_and_records_untouched(tiny):
    F, eng, store, ids = tiny["F"], tiny["eng"], tiny["store"], tiny["ids"]
    T = 8 + 8 * 256 + 32
    r = F.Result(eng, T + 2)
    eng.reprocess(store, tiny["question"], ids, 0.15, r, system=tiny["system"])
    first = int(np.argmax(r.logits()[-1]))
    before = store.read_kv(ids[0])
    with pytest.raises(F.ContractError):  # capacity: T + 4 - 1 > T + 2
        eng.decode(r, 4)
    toks = eng.decode(r, 3)
    assert int(toks[0]) == first
    after = store.read_kv(ids[0])
    assert np.array_equal(before[0], after[0]) and np.array_equal(before[1], after[1])
    fresh = F.Result(eng, 64)
    with pytest.raises(F.ContractError):  # nothing to continue from
        eng.decode(fresh, 1)


def test_fkvc_store_round_trip_and_reprocess(tiny, tmp_path):
    """serialize_record -> deserialize_record through the GPU loader: bit-exact
    record, and a reprocess over loaded records equals the original request."""
    F, eng, store, ids, chunks = tiny["F"], tiny["eng"], tiny["store"], tiny["ids"], tiny["chunks"]
    res = tiny["res"]
    eng.reprocess(store, tiny["question"], ids, 0.15, res, system=tiny["system"])
    want = res.logits().copy()
    paths = []
    for i, cid in enumerate(ids):
        p = tmp_path / f"c{i}.fkvc"
        store.save_record(cid, p)
        paths.append(p)
        h, k, v = F.fkvc_read(p)
        kb, vb = store.read_kv(cid)
        assert h["id"] == cid and h["native_start"] == 9 and h["tokens"] == 256
        assert np.array_equal((k.view(np.uint32) >> 16).astype(np.uint16), kb)  # bf16 -> fp32 exact
    st2 = F.ChunkKVStore(eng.cfg)
    got = [st2.load_record(p, ch) for p, ch in zip(paths, chunks)]
    assert got == list(ids)
    for cid in ids:
        a, b = store.read_kv(cid), st2.read_kv(cid)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    eng.reprocess(st2, tiny["question"], ids, 0.15, res, system=tiny["system"])
    assert np.array_equal(res.logits(), want)
    with pytest.raises(F.StoreError):  # single copy per chunk id
        st2.load_record(paths[0], chunks[0])
    st2.load_record(paths[0], chunks[0], overwrite=True)
    with pytest.raises(F.ContractError):  # the file holds 256 tokens
        st2.load_record(paths[0], chunks[0][:10], overwrite=True)


def test_fkvc_loader_rejects_other_model(tiny, tmp_path):
    F = tiny["F"]
    p = tmp_path / "odd.fkvc"
    k = np.zeros((3, 4, 4, 64), np.float32)  # 3 layers: tiny has 2
    F.fkvc_write(p, F.hash_tokens([1]), k, k, native_start=1)
    with pytest.raises(F.FormatError) as ei:
        tiny["store"].load_record(p, [1, 2, 3, 4])
    assert ei.value.kind == "Malformed"


def test_fkvc_loader_thread_overlaps_requests(tiny, tmp_path):
    """A loader thread fills a second store on its own stream while requests
    keep running on the first: both sides' results are unaffected."""
    import threading
    import torch
    F, eng, store, ids, chunks = tiny["F"], tiny["eng"], tiny["store"], tiny["ids"], tiny["chunks"]
    paths = []
    for i, cid in enumerate(ids):
        p = tmp_path / f"t{i}.fkvc"
        store.save_record(cid, p)
        paths.append(p)
    st2 = F.ChunkKVStore(eng.cfg)
    side = torch.cuda.Stream()
    err = []

    def loader():
        try:
            for p, ch in zip(paths, chunks):
                st2.load_record(p, ch, stream=side)
        except Exception as e:  # pragma: no cover
            err.append(e)

    res = F.Result(eng, 8 + 8 * 256 + 32)
    eng.reprocess(store, tiny["question"], ids, 0.15, res, system=tiny["system"])
    want = res.logits().copy()
    th = threading.Thread(target=loader)
    th.start()
    for _ in range(3):
        eng.reprocess(store, tiny["question"], ids, 0.15, res, system=tiny["system"])
        assert np.array_equal(res.logits(), want)
    th.join()
    assert not err and len(st2) == 8


_OVERLAP_SNIPPET = r"""
import hashlib, sys, numpy as np
sys.path.insert(0, '.')
from paper_2601_12904_b200 import fusion as F
eng = F.Engine("tiny", seed=1234)
store = F.ChunkKVStore(eng.cfg)
rng = np.random.default_rng(5)
system = rng.integers(0, eng.cfg.vocab, 8).tolist()
chunks = [rng.integers(0, eng.cfg.vocab, 256).tolist() for _ in range(8)]
ids = [eng.preprocess_isolated(store, c, system=system) for c in chunks]
question = rng.integers(0, eng.cfg.vocab, 32).tolist()
res = F.Result(eng, 8 + 8 * 256 + 32 + 64)
h = hashlib.sha256()
for i in range(3):  # eager, capture, replay
    eng.reprocess(store, question, ids, 0.15, res, system=system)
    k, v = res.fused_kv()
    h.update(k.tobytes()); h.update(v.tobytes()); h.update(res.logits().tobytes()); h.update(res.crit().tobytes())
print(h.hexdigest())
"""


def test_stitch_overlap_is_bit_identical(cuda):
    """K1 per layer on a side stream under the question pass (FRAG_STITCH_OVERLAP=1)
    gives the same bits as the single-launch stitch, eager and graph-replayed."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    out = {}
    for ov in ("0", "1"):
        env = dict(os.environ, FRAG_STITCH_OVERLAP=ov)
        p = subprocess.run([sys.executable, "-c", _OVERLAP_SNIPPET], cwd=root, env=env, capture_output=True,
                           text=True, timeout=300)
        assert p.returncode == 0, p.stderr[-2000:]
        out[ov] = p.stdout.strip().splitlines()[-1]
    assert out["0"] == out["1"]


_NORM_SNIPPET = r"""
import sys, numpy as np
sys.path.insert(0, '.')
from paper_2601_12904_b200 import fusion as F
eng = F.Engine("tiny", seed=1234)
store = F.ChunkKVStore(eng.cfg)
rng = np.random.default_rng(6)
chunks = [rng.integers(0, eng.cfg.vocab, 256).tolist() for _ in range(8)]
ids = [eng.preprocess_isolated(store, c) for c in chunks]
question = rng.integers(0, eng.cfg.vocab, 32).tolist()
res = F.Result(eng, 8 * 256 + 32)
eng.reprocess(store, question, ids, 0.15, res)
k, v = res.fused_kv()
kf = (np.asarray(k).astype(np.uint32) << 16).view(np.float32)  # bf16 bits -> values
np.savez(sys.argv[1], logits=res.logits(), k=kf, crit=res.crit())
"""


def test_folded_norm_matches_standalone_rmsnorm(cuda, tmp_path):
    """The RMSNorm folded into the GEMM epilogues (default) against the
    standalone rmsnorm kernel (FRAG_FUSED_NORM=0): same math, different bf16
    rounding point (bf16(h)·W·rs vs bf16(h·rs)·W), so close, not bit-equal."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    out = {}
    for fn in ("1", "0"):
        path = tmp_path / f"n{fn}.npz"
        env = dict(os.environ, FRAG_FUSED_NORM=fn)
        p = subprocess.run([sys.executable, "-c", _NORM_SNIPPET, str(path)], cwd=root, env=env,
                           capture_output=True, text=True, timeout=300)
        assert p.returncode == 0, p.stderr[-2000:]
        out[fn] = np.load(path)
    a, b = out["1"], out["0"]
    rel = np.linalg.norm(a["logits"] - b["logits"]) / np.linalg.norm(b["logits"])
    assert rel < 1e-2, rel
    diff = set(a["crit"].tolist()) ^ set(b["crit"].tolist())
    assert len(diff) <= len(b["crit"]) // 10
    # fused K away from the rows only one side recomputed (row = position - 1)
    keep = np.ones(a["k"].shape[1], bool)
    for c in diff:
        keep[max(c - 1, 0):c + 1] = False
    ka, kb = a["k"][:, keep], b["k"][:, keep]
    relk = np.linalg.norm(ka - kb) / np.linalg.norm(kb)
    assert relk < 1e-2, relk


_CHAIN_SNIPPET = r"""
import hashlib, sys, numpy as np
sys.path.insert(0, '.')
from paper_2601_12904_b200 import fusion as F
h = hashlib.sha256()
big = F.preset("llama3-8b")
big.layers = 2
for preset in ("tiny", big):
    eng = F.Engine(preset, seed=1234)
    store = F.ChunkKVStore(eng.cfg)
    rng = np.random.default_rng(8)
    n = 256 if preset == "tiny" else 512
    ids = [eng.preprocess_isolated(store, rng.integers(0, eng.cfg.vocab, n).tolist()) for _ in range(4)]
    question = rng.integers(0, eng.cfg.vocab, 32).tolist()
    res = F.Result(eng, 4 * n + 32 + 8)
    for ratio in (0.0, 0.15):
        for i in range(2):  # eager, then captured graph
            eng.reprocess(store, question, ids, ratio, res)
            k, v = res.fused_kv()
            h.update(k.tobytes()); h.update(v.tobytes()); h.update(res.logits().tobytes())
    h.update(eng.decode(res, 4).tobytes())
    eng.reprocess(store, question[:7], ids, 0.15, res)  # 7-row question pass
    h.update(res.logits().tobytes())
    for nq in (50, 100):  # the 64- and 128-row A stages
        long_q = rng.integers(0, eng.cfg.vocab, nq).tolist()
        res2 = F.Result(eng, 4 * n + nq + 8)
        eng.reprocess(store, long_q, ids, 0.05, res2)
        h.update(res2.logits().tobytes())
print(h.hexdigest())
"""


def test_gemm_chain_is_bit_identical(cuda):
    """The <= 128-row projection chain (gemm_chain.cu: O -> gate/up -> down ->
    next QKV in one persistent launch) computes exactly what the four separate
    weight-streaming GEMMs compute (same tiles, splits and fixup order):
    question pass, r = 0 sparse pass and decode, tiny and 8B width."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    out = {}
    for ch in ("0", "1"):
        env = dict(os.environ, FRAG_GEMM_CHAIN=ch)
        p = subprocess.run([sys.executable, "-c", _CHAIN_SNIPPET], cwd=root, env=env, capture_output=True,
                           text=True, timeout=600)
        assert p.returncode == 0, p.stderr[-2000:]
        out[ch] = p.stdout.strip().splitlines()[-1]
    assert out["0"] == out["1"]


@pytest.mark.parametrize("preset,layers", [("tiny", 0), ("llama3-8b", 2)])
def test_r0_full_reuse_fast_path_bit_identical(cuda, preset, layers):
    """r = 0 (Full Reuse): one full pass over the question rows
    replaces the question pass + the sparse pass over the same rows. Its
    logits, fused K/V and q_final equal the two-pass path (forced here by an
    empty injected critical set) bit for bit, eager and graph-replayed."""
    from paper_2601_12904_b200 import fusion as F
    cfg = F.preset(preset)
    if layers:
        cfg.layers = layers
    eng = F.Engine(cfg, seed=21)
    store = F.ChunkKVStore(cfg)
    rng = np.random.default_rng(5)
    ids = [eng.preprocess_isolated(store, rng.integers(0, cfg.vocab, 200).tolist()) for _ in range(3)]
    T = 600 + 32
    a, b = F.Result(eng, T), F.Result(eng, T)
    for _ in range(3):  # eager, capture, replay
        q = rng.integers(0, cfg.vocab, 32).tolist()
        eng.reprocess(store, q, ids, 0.0, a)
        eng.reprocess(store, q, ids, 0.0, b, inject_crit=[])
        assert len(a.crit()) == 0 and len(b.crit()) == 0
        assert np.array_equal(a.logits(), b.logits())
        ka, va = a.fused_kv()
        kb, vb = b.fused_kv()
        assert np.array_equal(ka, kb) and np.array_equal(va, vb)
        assert np.array_equal(a.debug()["q_final"], b.debug()["q_final"])
    a.close()
    b.close()
    store.close()
    eng.close()


def test_manifest_round_trip(tiny, tmp_path):
    """save_manifest -> load_manifest into a fresh store: the
    same records (bytes, variant, native_start, tokens) and the same request."""
    F, eng = tiny["F"], tiny["eng"]
    store, ids = tiny["store"], tiny["ids"]
    n = store.save_manifest(tmp_path)
    assert n == len(store) and (tmp_path / "manifest.json").exists()
    assert F.manifest_validate(tmp_path / "manifest.json") == n
    fresh = F.ChunkKVStore(eng.cfg)
    assert fresh.load_manifest(tmp_path / "manifest.json") == n
    for cid in ids:
        a, b = store.peek(cid), fresh.peek(cid)
        assert (a.n_tok, a.native_start, a.variant) == (b.n_tok, b.native_start, b.variant)
        ka, va = store.read_kv(cid)
        kb, vb = fresh.read_kv(cid)
        assert np.array_equal(ka, kb) and np.array_equal(va, vb)
    with pytest.raises(F.StoreError):
        fresh.load_manifest(tmp_path / "manifest.json")  # duplicates without overwrite
    assert fresh.load_manifest(tmp_path / "manifest.json", overwrite=True) == n
    fresh.close()
