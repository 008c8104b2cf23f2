"""Multi-request batching (frag_reprocess_batch): B
requests in one fused cache (request b at rows [b*slot, ...)), one question
pass and one sparse pass over all of them. Each request must match its own
single-request reprocess: the question pass is row-independent with the same
split-K plan (critical sets and stitched rows bit-exact), the sparse pass may
reorder the long-K tail split (tolerance below)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(a.astype(np.float64) - b) / max(np.linalg.norm(b.astype(np.float64)), 1e-30))


@pytest.fixture(scope="module")
def setup(cuda):
    from paper_2601_12904_b200 import fusion as F
    eng = F.Engine("tiny", seed=1234)
    store = F.ChunkKVStore(eng.cfg)
    rng = np.random.default_rng(77)
    system = rng.integers(0, eng.cfg.vocab, 8).tolist()
    pool = [rng.integers(0, eng.cfg.vocab, 256).tolist() for _ in range(6)]
    ids_sys = [eng.preprocess_isolated(store, c, system=system) for c in pool[:3]]
    ids = [eng.preprocess_isolated(store, c) for c in pool[3:]]
    reqs = [
        (rng.integers(0, eng.cfg.vocab, 32).tolist(), ids_sys, 0.15, system),
        (rng.integers(0, eng.cfg.vocab, 16).tolist(), ids[:2], 0.3, ()),
        (rng.integers(0, eng.cfg.vocab, 32).tolist(), ids, 0.0, ()),
        (rng.integers(0, eng.cfg.vocab, 8).tolist(), [ids[2], ids[0]], 1.0, ()),
    ]
    return F, eng, store, reqs


def _single(F, eng, store, rq, cap):
    res = F.Result(eng, cap)
    eng.reprocess(store, rq[0], rq[1], rq[2], res, system=rq[3])
    k, v = res.fused_kv()
    return res.logits()[0].copy(), res.crit().copy(), k, v


def test_batch_matches_single_requests(setup):
    F, eng, store, reqs = setup
    slot = 8 + 3 * 256 + 32
    res = F.Result(eng, len(reqs) * slot)
    eng.reprocess_batch(store, reqs, res, slot)
    lg = res.logits()
    assert lg.shape == (len(reqs), eng.cfg.vocab)
    kb, vb = res.fused_kv()
    for b, rq in enumerate(reqs):
        l1, c1, k1, v1 = _single(F, eng, store, rq, slot)
        T = len(rq[3]) + 256 * len(rq[1]) + len(rq[0])
        assert np.array_equal(res.batch_crit(b), c1), b  # identical question pass -> identical selection
        kseg, vseg = kb[:, b * slot:b * slot + T], vb[:, b * slot:b * slot + T]
        fresh = np.zeros(T, bool)
        fresh[c1 - 1] = True
        fresh[T - len(rq[0]):] = True
        assert np.array_equal(kseg[:, ~fresh], k1[:, ~fresh]) and np.array_equal(vseg[:, ~fresh], v1[:, ~fresh])
        from oracle import oracle as O
        gk, sk = O.bf16_bits_to_f32(kseg[:, fresh]), O.bf16_bits_to_f32(k1[:, fresh])
        assert _rel(gk, sk) <= 1e-2, b
        assert _rel(lg[b], l1) <= 1e-2, b
        top = np.sort(l1)[::-1]
        if top[0] - top[1] >= 1e-2:
            assert np.argmax(lg[b]) == np.argmax(l1)


def test_batch_of_one_is_bit_identical(setup):
    """Same kernels on the same rows: fused KV, selection and logits bit-identical
    (both run the last layer's attention / O / MLP on the logit row alone,
    DESIGN.md §3; the batch compacts it after the plan rows)."""
    F, eng, store, reqs = setup
    rq = reqs[0]
    slot = 8 + 3 * 256 + 32
    res = F.Result(eng, slot)
    eng.reprocess_batch(store, [rq], res, slot)
    l1, c1, k1, v1 = _single(F, eng, store, rq, slot)
    k, v = res.fused_kv()
    assert np.array_equal(res.batch_crit(0), c1)
    assert np.array_equal(k, k1) and np.array_equal(v, v1)
    assert np.array_equal(res.logits()[0], l1)


def test_batch_contracts(setup):
    F, eng, store, reqs = setup
    res = F.Result(eng, 2 * 600)
    with pytest.raises(F.ContractError):  # request longer than its slot
        eng.reprocess_batch(store, reqs[:2], res, 600)
    with pytest.raises(F.ContractError):  # batch larger than the result
        eng.reprocess_batch(store, reqs[1:3], res, 1000)
    with pytest.raises(F.ContractError):
        res.batch_crit(5)


def test_batch_graph_replay_is_bit_identical(setup):
    """The batched body is captured into a CUDA graph on the second batch of a
    shape and replayed afterwards: eager, captured and replayed batches agree."""
    F, eng, store, reqs = setup
    slot = 8 + 3 * 256 + 32
    res = F.Result(eng, len(reqs) * slot)
    outs = []
    for _ in range(4):
        eng.reprocess_batch(store, reqs, res, slot)
        k, v = res.fused_kv()
        outs.append((res.logits().copy(), [res.batch_crit(b).copy() for b in range(len(reqs))], k, v))
    for lg, cr, k, v in outs[1:]:
        assert np.array_equal(lg, outs[0][0]) and np.array_equal(k, outs[0][2]) and np.array_equal(v, outs[0][3])
        assert all(np.array_equal(a, b) for a, b in zip(cr, outs[0][1]))
