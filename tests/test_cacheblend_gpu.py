"""CacheBlend selector on the GPU (Eq. 7-8):
kv_deviation between Full Attention and Full Reuse over cat(S, chunks) through
the first two layers, and select_cacheblend = argTopk of the layer-2 K
deviation, feeding the same sparse prefill as the query-guided selector."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cb(cuda):
    from oracle import oracle as O
    from paper_2601_12904_b200 import fusion as F
    eng = F.Engine("tiny", seed=1234)
    store = F.ChunkKVStore(eng.cfg)
    rng = np.random.default_rng(31)
    system = rng.integers(0, eng.cfg.vocab, 8).tolist()
    chunks = [rng.integers(0, eng.cfg.vocab, 256).tolist() for _ in range(4)]
    ids = [eng.preprocess_isolated(store, c, system=system) for c in chunks]
    question = rng.integers(0, eng.cfg.vocab, 32).tolist()
    res = F.Result(eng, 8 + 4 * 256 + 32)
    om = O.Model(eng.cfg).load_from_engine(eng)
    return dict(F=F, O=O, eng=eng, store=store, system=system, chunks=chunks, ids=ids, question=question, res=res,
                om=om)


def _oracle_inputs(t, res_k, res_v):
    O = t["O"]
    S = len(t["system"])
    recs = []
    for i, ch in zip(t["ids"], t["chunks"]):
        rk, rv = t["store"].read_kv(i)
        recs.append({"k": O.bf16_bits_to_f32(rk), "v": O.bf16_bits_to_f32(rv), "tokens": ch, "native_start": S + 1})
    sys_kv = (O.bf16_bits_to_f32(res_k[:, :S]), O.bf16_bits_to_f32(res_v[:, :S]))
    return sys_kv, recs


def test_kv_deviation_matches_oracle(cb):
    eng, res = cb["eng"], cb["res"]
    dev = eng.kv_deviation(cb["store"], cb["ids"], res, system=cb["system"], n_layers=2)
    N = 4 * 256
    assert dev.shape == (N, 2, 2) and np.all(dev >= 0)
    k, v = res.fused_kv()
    sys_kv, recs = _oracle_inputs(cb, k, v)
    odev = cb["om"].kv_deviation(sys_kv, recs, n_layers=2, emulate_bf16=True)
    for comp in (0, 1):
        g, o = dev[:, 1, comp].astype(np.float64), odev[:, 1, comp]
        rel = np.linalg.norm(g - o) / np.linalg.norm(o)
        assert rel <= 5e-2, (comp, rel)
    # the first chunk sits at its native offset: FR == FA there (Eq. 4)
    scale = dev[256:, 1, 0].mean()
    assert dev[:256, 1, :].max() <= 1e-3 * scale
    assert np.all(dev[256:, 1, 0] > 0)  # later chunks miss cross-attention
    # layer-1 V depends only on the token embedding; layer-1 K only on the RoPE shift rounding
    assert dev[:, 0, 1].max() <= 1e-3 * scale
    assert dev[:, 0, 0].max() <= 1e-2 * scale
    # the result holds the Full-Reuse stitched cache afterwards
    eng.reprocess(cb["store"], cb["question"], cb["ids"], 0.0, res, system=cb["system"])
    k0, v0 = res.fused_kv()
    T = 8 + N
    assert np.array_equal(k[:, :T], k0[:, :T]) and np.array_equal(v[:, :T], v0[:, :T])


def test_kv_deviation_single_chunk_is_zero(cb):
    dev = cb["eng"].kv_deviation(cb["store"], cb["ids"][:1], cb["res"], system=cb["system"], n_layers=2)
    assert np.max(dev) <= 1e-6 * max(1.0, float(np.abs(dev).max()))


def test_cacheblend_selection_is_exact_topk_of_its_deviation(cb):
    eng, res = cb["eng"], cb["res"]
    N = 4 * 256
    for ratio, comp in ((0.15, "k"), (0.3, "v"), (0.05, "kv")):
        eng.reprocess(cb["store"], cb["question"], cb["ids"], ratio, res, system=cb["system"], selector="cacheblend",
                      deviation_component=comp)
        scores = res.debug()["scores"]
        k = int(np.floor(ratio * N + 0.5))
        crit = res.crit()
        order = np.argsort(-scores.astype(np.float64), kind="stable")
        assert np.array_equal(crit, np.sort(order[:k]) + 9)  # positions are 1-based after S = 8
        dev = eng.kv_deviation(cb["store"], cb["ids"], cb["F"].Result(eng, res.max_tokens), system=cb["system"])
        ref = {"k": dev[:, 1, 0], "v": dev[:, 1, 1], "kv": dev[:, 1, 0] + dev[:, 1, 1]}[comp]
        assert np.array_equal(scores, ref.astype(np.float32))


def test_cacheblend_equals_injected_plan_and_oracle_overlap(cb):
    eng, res, F = cb["eng"], cb["res"], cb["F"]
    eng.reprocess(cb["store"], cb["question"], cb["ids"], 0.15, res, system=cb["system"], selector="cacheblend")
    crit = res.crit().copy()
    lg = res.logits().copy()
    k, v = res.fused_kv()
    inj = F.Result(eng, res.max_tokens)
    eng.reprocess(cb["store"], cb["question"], cb["ids"], 0.15, inj, system=cb["system"], inject_crit=crit)
    ki, vi = inj.fused_kv()
    # the FA pass's rows were restored: the sparse pass saw exactly the Full-Reuse cache
    assert np.array_equal(k, ki) and np.array_equal(v, vi)
    assert np.array_equal(lg, inj.logits())
    # selection vs the oracle's own deviation (bf16 noise may swap boundary tokens)
    sys_kv, recs = _oracle_inputs(cb, k, v)
    odev = cb["om"].kv_deviation(sys_kv, recs, n_layers=2, emulate_bf16=True)
    osel = cb["O"].select_cacheblend(odev, len(crit)) + 9
    overlap = len(np.intersect1d(osel, crit)) / len(crit)
    assert overlap >= 0.9, overlap


def test_cacheblend_endpoints_and_graph_replay(cb):
    eng, res, F = cb["eng"], cb["res"], cb["F"]
    tokens = [t for c in cb["chunks"] for t in c] + cb["question"]
    fa = F.Result(eng, res.max_tokens)
    eng.full_prefill(tokens, fa, system=cb["system"])
    eng.reprocess(cb["store"], cb["question"], cb["ids"], 1.0, res, system=cb["system"], selector="cacheblend")
    assert len(res.crit()) == 4 * 256
    assert np.array_equal(res.logits(), fa.logits())  # r = 1 == Full Attention
    qg = F.Result(eng, res.max_tokens)
    eng.reprocess(cb["store"], cb["question"], cb["ids"], 0.0, qg, system=cb["system"])
    eng.reprocess(cb["store"], cb["question"], cb["ids"], 0.0, res, system=cb["system"], selector="cacheblend")
    assert len(res.crit()) == 0 and np.array_equal(res.logits(), qg.logits())  # r = 0 == Full Reuse
    outs = []
    for _ in range(4):  # eager, capture, replay, replay
        eng.reprocess(cb["store"], cb["question"], cb["ids"], 0.15, res, system=cb["system"], selector="cacheblend")
        outs.append((res.crit().copy(), res.logits().copy()))
    for c, l in outs[1:]:
        assert np.array_equal(c, outs[0][0]) and np.array_equal(l, outs[0][1])
    with pytest.raises(F.ContractError):
        eng.reprocess(cb["store"], cb["question"], cb["ids"], 0.15, res, system=cb["system"], selector="cacheblend",
                      deviation_layer=3)
