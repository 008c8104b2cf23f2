"""Shared V pages (SPEC.md:148-150 exclusive pages, SPEC.md:173
shared-cache immutability, SPEC.md:174 batch isolation, SPEC.md:480-482 shared
records listed once; §4.3).

With shared V a request never copies its chunks' V rows: the attention kernels
read them in place from the records (TMA from the record's pages, the rows of
other records / KV_S / fresh rows patched into the tile) and only the rows the
request computes live in its exclusive slots. The V tile the tensor pipe
consumes is byte-identical to the private fused cache's, so every output --
logits, selection, fused K, the fused V view, decoded tokens -- must be
bit-identical to the private layout (frag_set_shared_v(0)), on the same kernels.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def F(cuda):
    from paper_2601_12904_b200 import fusion as F
    prev = F.set_shared_v(True)
    yield F
    F.set_shared_v(prev)


@pytest.fixture(scope="module")
def tiny(F):
    eng = F.Engine("tiny", seed=4321)
    store = F.ChunkKVStore(eng.cfg)
    rng = np.random.default_rng(5)
    system = rng.integers(0, eng.cfg.vocab, 8).tolist()
    # lengths that put chunk boundaries inside 128-row tiles (static patches)
    lens = [256, 200, 333, 97, 256, 150]
    chunks = [rng.integers(0, eng.cfg.vocab, n).tolist() for n in lens]
    ids = [eng.preprocess_isolated(store, ch, system=system) for ch in chunks]
    return eng, store, system, ids, rng


def _run(F, eng, store, q, ids, r, system, shared, cap, decode=0, **kw):
    F.set_shared_v(shared)
    res = F.Result(eng, cap)
    eng.reprocess(store, q, ids, r, res, system=system, **kw)
    out = {"logits": res.logits().copy(), "crit": res.crit().copy(), "mem": res.memory()}
    out["k"], out["v"] = res.fused_kv()
    if decode:
        out["tok"] = np.asarray(eng.decode(res, decode))
        out["k_dec"], out["v_dec"] = res.fused_kv()
        out["logits_dec"] = res.logits().copy()
    res.close()
    return out


@pytest.mark.parametrize("ratio", [0.0, 0.05, 0.15, 0.5])
def test_shared_v_bit_identical_to_private(F, tiny, ratio):
    eng, store, system, ids, rng = tiny
    q = rng.integers(0, eng.cfg.vocab, 32).tolist()
    T = len(system) + sum(store.peek(i).n_tok for i in ids) + len(q)
    a = _run(F, eng, store, q, ids, ratio, system, True, T + 16, decode=8)
    b = _run(F, eng, store, q, ids, ratio, system, False, T + 16, decode=8)
    assert a["mem"][1] and not b["mem"][1]
    assert np.array_equal(a["crit"], b["crit"])
    assert np.array_equal(a["logits"], b["logits"])
    assert np.array_equal(a["k"], b["k"]) and np.array_equal(a["v"], b["v"])
    assert np.array_equal(a["tok"], b["tok"])
    Td = T + 7
    assert np.array_equal(a["k_dec"][:, :Td], b["k_dec"][:, :Td])
    assert np.array_equal(a["v_dec"][:, :Td], b["v_dec"][:, :Td])
    assert np.array_equal(a["logits_dec"], b["logits_dec"])


def test_shared_v_injected_plan(F, tiny):
    eng, store, system, ids, rng = tiny
    q = rng.integers(0, eng.cfg.vocab, 20).tolist()
    N = sum(store.peek(i).n_tok for i in ids)
    crit = np.sort(rng.choice(N, 150, replace=False)) + len(system) + 1
    T = len(system) + N + len(q)
    a = _run(F, eng, store, q, ids, 0.15, system, True, T, inject_crit=crit)
    b = _run(F, eng, store, q, ids, 0.15, system, False, T, inject_crit=crit)
    assert np.array_equal(a["logits"], b["logits"])
    assert np.array_equal(a["v"], b["v"]) and np.array_equal(a["k"], b["k"])


@pytest.mark.parametrize("ratio", [0.0, 0.15])
def test_records_untouched_and_memory(F, tiny, ratio):
    """The attention reads the records' pages in place; nothing writes them
    (SPEC.md:173). Without a V read-back the shared request holds no fused V:
    only its exclusive slots and, for a sparse pass, a two-layer staging window
    (which for this 2-layer model is as large as the whole V -- hence r = 0,
    whose single pass reads the records directly, for the accounting)."""
    eng, store, system, ids, rng = tiny
    before = [store.read_kv(i) for i in ids]
    q = rng.integers(0, eng.cfg.vocab, 32).tolist()
    T = len(system) + sum(store.peek(i).n_tok for i in ids) + len(q)
    F.set_shared_v(True)
    res = F.Result(eng, T)
    eng.reprocess(store, q, ids, ratio, res, system=system)
    mem_shared, sv = res.memory()
    assert sv
    for i, (k0, v0) in zip(ids, before):
        k1, v1 = store.read_kv(i)
        assert np.array_equal(k0, k1) and np.array_equal(v0, v1)
    F.set_shared_v(False)
    res2 = F.Result(eng, T)
    eng.reprocess(store, q, ids, ratio, res2, system=system)
    mem_private, sv2 = res2.memory()
    assert not sv2
    if ratio == 0:
        c = eng.cfg
        v_bytes = c.layers * T * c.n_kv_heads * c.head_dim * 2
        assert mem_private - mem_shared >= 0.8 * v_bytes, (mem_private, mem_shared, v_bytes)
    F.set_shared_v(True)


def test_batch_shares_records(F, tiny):
    """Requests of one batch reusing the same records read one set of pages;
    each request equals its own single-request run and the batch equals the
    private-V batch bit for bit (batch isolation)."""
    eng, store, system, ids, rng = tiny
    reqs = [
        (rng.integers(0, eng.cfg.vocab, 32).tolist(), ids[:4], 0.15, system),
        (rng.integers(0, eng.cfg.vocab, 16).tolist(), [ids[2], ids[0], ids[5]], 0.3, ()),
        (rng.integers(0, eng.cfg.vocab, 24).tolist(), ids[:4], 0.05, system),
    ]
    slot = 8 + 256 + 200 + 333 + 97 + 32
    outs = []
    for shared in (True, False):
        F.set_shared_v(shared)
        res = F.Result(eng, len(reqs) * slot)
        eng.reprocess_batch(store, reqs, res, slot)
        k, v = res.fused_kv()
        outs.append((res.logits().copy(), [res.batch_crit(b).copy() for b in range(len(reqs))], k, v, res.memory()))
        res.close()
    (la, ca, ka, va, ma), (lb, cb, kb, vb, mb) = outs
    assert ma[1] and not mb[1]
    assert np.array_equal(la, lb)
    assert all(np.array_equal(x, y) for x, y in zip(ca, cb))
    for b, rq in enumerate(reqs):
        T = len(rq[3]) + sum(store.peek(i).n_tok for i in rq[1]) + len(rq[0])
        sl = slice(b * slot, b * slot + T)
        assert np.array_equal(ka[:, sl], kb[:, sl]) and np.array_equal(va[:, sl], vb[:, sl]), b
    F.set_shared_v(True)


def test_graph_replay_shared_v(F, tiny):
    """Shared-V requests replay from the captured body: the plan is rebuilt on
    the device from each request's own selection."""
    eng, store, system, ids, rng = tiny
    T = len(system) + sum(store.peek(i).n_tok for i in ids) + 32
    F.set_shared_v(True)
    res = F.Result(eng, T)
    qs = [rng.integers(0, eng.cfg.vocab, 32).tolist() for _ in range(4)]
    got = []
    for q in qs:
        eng.reprocess(store, q, ids, 0.15, res, system=system)
        got.append((res.logits().copy(), res.crit().copy(), res.fused_kv()[1]))
    for q, (lg, cr, v) in zip(qs, got):
        ref = _run(F, eng, store, q, ids, 0.15, system, False, T)
        assert np.array_equal(cr, ref["crit"]) and np.array_equal(lg, ref["logits"])
        assert np.array_equal(v, ref["v"])
    F.set_shared_v(True)


@pytest.mark.parametrize("nq,ratio", [(32, 0.15), (50, 0.05), (32, 0.0)])
def test_shared_v_8b_width(F, nq, ratio):
    """Llama-3-8B width (GQA 32/8: one attention tile = 32 tokens), 2 layers,
    4 x 512 chunks: the sparse pass stages V through the window, the 32-row
    question pass patches record tiles in the kernel, a 50-row question pass
    uses the window too; decode patches. Bit-identical to the private layout."""
    cfg = F.preset("llama3-8b")
    cfg.layers = 2
    eng = F.Engine(cfg, seed=77)
    store = F.ChunkKVStore(eng.cfg)
    rng = np.random.default_rng(nq)
    ids = [eng.preprocess_isolated(store, rng.integers(0, eng.cfg.vocab, 512).tolist()) for _ in range(4)]
    q = rng.integers(0, eng.cfg.vocab, nq).tolist()
    T = 4 * 512 + nq
    a = _run(F, eng, store, q, ids, ratio, (), True, T + 8, decode=4)
    b = _run(F, eng, store, q, ids, ratio, (), False, T + 8, decode=4)
    assert a["mem"][1] and not b["mem"][1]
    assert np.array_equal(a["crit"], b["crit"])
    assert np.array_equal(a["logits"], b["logits"])
    assert np.array_equal(a["k"], b["k"]) and np.array_equal(a["v"], b["v"])
    assert np.array_equal(a["tok"], b["tok"]) and np.array_equal(a["logits_dec"], b["logits_dec"])
    F.set_shared_v(True)


def test_result_keeps_shared_pages_alive(F):
    """A result reading records in place keeps their pages alive: destroying
    the store (or overwriting its records) after the request leaves the
    result's V view and its decode intact."""
    eng = F.Engine("tiny", seed=99)
    rng = np.random.default_rng(3)
    chunks = [rng.integers(0, eng.cfg.vocab, 256).tolist() for _ in range(4)]
    q = rng.integers(0, eng.cfg.vocab, 16).tolist()
    T = 4 * 256 + 16
    F.set_shared_v(True)
    store = F.ChunkKVStore(eng.cfg)
    ids = [eng.preprocess_isolated(store, ch) for ch in chunks]
    ref = F.Result(eng, T + 8)
    eng.reprocess(store, q, ids, 0.15, ref)
    want_v = ref.fused_kv()[1]
    want_tok = np.asarray(eng.decode(ref, 6))
    res = F.Result(eng, T + 8)
    eng.reprocess(store, q, ids, 0.15, res)
    assert res.memory()[1]
    store.close()  # the records' pages are still referenced by res
    assert np.array_equal(res.fused_kv()[1], want_v)
    assert np.array_equal(np.asarray(eng.decode(res, 6)), want_tok)
    res.close()
    ref.close()


@pytest.mark.parametrize("seed", [11, 12, 13, 14])
def test_shared_v_random_layouts(F, seed):
    """Random chunk counts and lengths (boundaries anywhere inside key tiles),
    random system prompts, question lengths and ratios: shared V pages equal
    the private layout bit for bit (tiny model)."""
    rng = np.random.default_rng(seed)
    eng = F.Engine("tiny", seed=seed)
    store = F.ChunkKVStore(eng.cfg)
    n_sys = int(rng.integers(0, 20))
    system = rng.integers(0, eng.cfg.vocab, n_sys).tolist()
    lens = rng.integers(1, 400, int(rng.integers(1, 9))).tolist()
    ids = [eng.preprocess_isolated(store, rng.integers(0, eng.cfg.vocab, n).tolist(), system=system) for n in lens]
    q = rng.integers(0, eng.cfg.vocab, int(rng.integers(1, 70))).tolist()
    ratio = float(rng.choice([0.0, 0.02, 0.1, 0.25, 0.5]))
    T = n_sys + sum(lens) + len(q)
    a = _run(F, eng, store, q, ids, ratio, system, True, T + 4, decode=4)
    b = _run(F, eng, store, q, ids, ratio, system, False, T + 4, decode=4)
    assert np.array_equal(a["crit"], b["crit"]) and np.array_equal(a["logits"], b["logits"])
    assert np.array_equal(a["k"], b["k"]) and np.array_equal(a["v"], b["v"])
    assert np.array_equal(a["tok"], b["tok"])
    F.set_shared_v(True)
