"""SURVEY.md §8(f) rows at the bench model's width (Llama-3-8B layers: d=4096,
GQA 32/8, dh=128, F=14336; reduced depth): CacheBlend's kv_deviation
(Eq. 7) against the oracle, multi-request batching against
single requests, and greedy decode against the oracle fed the same tokens.
The tiny-config versions of these tests (test_cacheblend_gpu.py,
test_batch_gpu.py, test_parity_gpu.py) cover the edge cases; these pin the
GQA / dh = 128 kernels the bench runs."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rel(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.fixture(scope="module")
def w8b(cuda):
    from oracle import oracle as O
    from paper_2601_12904_b200 import fusion as F
    cfg = F.preset("llama3-8b")
    cfg.layers = 3
    eng = F.Engine(cfg, seed=2024)
    store = F.ChunkKVStore(cfg)
    rng = np.random.default_rng(17)
    S = 8
    system = rng.integers(0, cfg.vocab, S).tolist()
    chunks = [rng.integers(0, cfg.vocab, 256).tolist() for _ in range(4)]
    ids = [eng.preprocess_isolated(store, c, system=system) for c in chunks]
    questions = [rng.integers(0, cfg.vocab, 32).tolist() for _ in range(3)]
    om = O.Model(cfg).load_from_engine(eng)
    return dict(F=F, O=O, cfg=cfg, eng=eng, store=store, S=S, system=system, chunks=chunks, ids=ids,
                questions=questions, om=om)


def _records(t):
    O = t["O"]
    recs = []
    for i, ch in zip(t["ids"], t["chunks"]):
        rk, rv = t["store"].read_kv(i)
        recs.append({"k": O.bf16_bits_to_f32(rk), "v": O.bf16_bits_to_f32(rv), "tokens": ch,
                     "native_start": t["S"] + 1})
    return recs


def test_kv_deviation_8b_width_matches_oracle(w8b):
    t = w8b
    F, O, eng, S = t["F"], t["O"], t["eng"], t["S"]
    N = 4 * 256
    res = F.Result(eng, S + N + 32)
    dev = eng.kv_deviation(t["store"], t["ids"], res, system=t["system"], n_layers=2)
    assert dev.shape == (N, 2, 2) and np.all(dev >= 0)
    k, v = res.fused_kv()
    sys_kv = (O.bf16_bits_to_f32(k[:, :S]), O.bf16_bits_to_f32(v[:, :S]))
    odev = t["om"].kv_deviation(sys_kv, _records(t), n_layers=2, emulate_bf16=True)
    for comp in (0, 1):  # layer 2, K and V
        assert _rel(dev[:, 1, comp], odev[:, 1, comp]) <= 5e-2, comp
    scale = dev[256:, 1, 0].mean()
    assert dev[:256, 1, :].max() <= 1e-3 * scale  # the first chunk sits at its native offset (Eq. 4)
    assert np.all(dev[256:, 1, 0] > 0)            # later chunks miss cross-attention
    # CacheBlend selection = exact top-k of the layer-2 K deviation it computed
    eng.reprocess(t["store"], t["questions"][0], t["ids"], 0.15, res, system=t["system"], selector="cacheblend")
    scores = res.debug()["scores"].astype(np.float64)
    k_sel = int(np.floor(0.15 * N + 0.5))
    order = np.argsort(-scores, kind="stable")
    assert np.array_equal(res.crit(), np.sort(order[:k_sel]) + S + 1)


def test_batch_8b_width_matches_single_requests(w8b):
    """Three requests (different questions and ratios) in one fused cache:
    each selection identical to its single-request reprocess, logits and the
    recomputed K rows within 1e-2 (the batched GEMMs tile differently)."""
    t = w8b
    F, eng, S = t["F"], t["eng"], t["S"]
    T = S + 4 * 256 + 32
    reqs = [(t["questions"][b], t["ids"], r, t["system"]) for b, r in enumerate((0.15, 0.3, 0.05))]
    rb = F.Result(eng, 3 * T)
    eng.reprocess_batch(t["store"], reqs, rb, T)
    lg = rb.logits().copy()
    kb, _ = rb.fused_kv()
    for b, rq in enumerate(reqs):
        r1 = F.Result(eng, T)
        eng.reprocess(t["store"], rq[0], rq[1], rq[2], r1, system=rq[3])
        c1 = r1.crit()
        assert np.array_equal(rb.batch_crit(b), c1), b
        assert _rel(lg[b], r1.logits()[0]) <= 1e-2, b
        k1, _ = r1.fused_kv()
        fresh = np.zeros(T, bool)
        fresh[c1 - 1] = True
        fresh[T - 32:] = True
        kseg = kb[:, b * T:(b + 1) * T]
        assert np.array_equal(kseg[:, ~fresh], k1[:, ~fresh]), b
        O = t["O"]
        assert _rel(O.bf16_bits_to_f32(kseg[:, fresh]), O.bf16_bits_to_f32(k1[:, fresh])) <= 1e-2, b


def test_decode_8b_width_teacher_forced(w8b):
    """Greedy decode after a 15 % reprocess vs the oracle fed the GPU's tokens
    over its own selection-injected, bf16-emulating fused cache: final logits
    within the reprocess tolerance, every greedy choice the oracle's argmax
    unless its top-2 gap < 1e-2."""
    t = w8b
    F, O, eng, S = t["F"], t["O"], t["eng"], t["S"]
    T = S + 4 * 256 + 32
    n = 4
    res = F.Result(eng, T + n)
    eng.reprocess(t["store"], t["questions"][1], t["ids"], 0.15, res, system=t["system"])
    crit = res.crit().copy()
    k0, v0 = res.fused_kv()
    first = res.logits()[0].copy()
    toks = eng.decode(res, n)
    last = res.logits()[0]
    sys_kv = (O.bf16_bits_to_f32(k0[:, :S]), O.bf16_bits_to_f32(v0[:, :S]))
    out = t["om"].reprocess(sys_kv, _records(t), t["questions"][1], 0.15, inject=crit, emulate_bf16=True,
                            cap=T + n)
    assert _rel(first, out["logits"]) <= 3e-2
    steps = t["om"].decode_forced(out["k_cache"], out["v_cache"], T, toks[:-1], emulate_bf16=True)
    prev = [out["logits"]] + list(steps[:-1])
    for i, lg in enumerate(prev):  # every greedy choice, unless the oracle's top-2 gap is tiny
        top = np.sort(lg)[::-1]
        if top[0] - top[1] >= 1e-2:
            assert int(toks[i]) == int(np.argmax(lg)), i
    assert _rel(last, steps[-1]) <= 3e-2
