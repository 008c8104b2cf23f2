"""Pins the CPU oracle (test infrastructure) before it is trusted:
  * Rng against golden vectors from the REFERENCE header (tests/golden/rng_kat.json,
    produced by oracle/_ref/rng_kat built from /root/reference, common.hpp:45-100)
    and the survey's KATs;
  * every SPEC.md worked example / property oracle on the reprocessing path.
No GPU needed."""
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O

GOLD = json.loads((Path(__file__).parent / "golden" / "rng_kat.json").read_text())["vectors"]


# ---------------------------------------------------------------- Rng (common.hpp:45-100)
@pytest.mark.parametrize("seed", sorted(GOLD, key=int))
def test_rng_matches_reference_header(seed):
    g = GOLD[seed]
    s = int(seed)
    assert [int(x) for x in g["next_u64"]] == [int(v) for v in O.rng(s, "next_u64", 16)]
    assert np.array_equal(np.array(g["normal"], np.float64), O.rng(s, "normal", 16))
    assert np.array_equal(np.array(g["normal_f_0.02"], np.float32), O.rng(s, "normal_f_0.02", 16))
    assert g["below_256"] == O.rng(s, "below", 32, 256).tolist()
    assert g["below_128256"] == O.rng(s, "below", 32, 128256).tolist()
    assert np.array_equal(np.array(g["next_float"], np.float32), O.rng(s, "next_float", 16))
    assert g["range_m5_5"] == O.rng(s, "range", 16, 5).tolist()


def test_rng_survey_kats():
    # SURVEY.md §8(c) table (probe values)
    assert O.rng(0, "next_u64", 3).tolist() == [16294208416658607535, 7960286522194355700, 487617019471545679]
    assert O.rng(42, "next_u64", 3).tolist() == [13679457532755275413, 2949826092126892291, 5139283748462763858]
    assert np.allclose(O.rng(42, "normal", 4), [0.41471975043153059, 0.65268122215194291, -0.89188621362775633,
                                                 1.3268335628141066], rtol=0, atol=1e-16)
    assert O.rng(42, "below", 8, 256).tolist() == [149, 3, 82, 148, 242, 6, 93, 164]
    assert np.allclose(O.rng(7, "next_float", 3), [0.389829755, 0.0167882945, 0.90076071], atol=1e-9)


@pytest.mark.parametrize("seed,n", [(1, 1), (2, 7), (123456789, 1000), (2**63 + 5, 4097)])
def test_counter_form_weight_stream_equals_sequential_rng(seed, n):
    # init_model draws: the parallel counter form (used on the GPU) == literal Rng.normal_f
    a = O.gen_normal(seed, n, 0.02, sequential=True, round_bf16=False)
    b = O.gen_normal(seed, n, 0.02, sequential=False, round_bf16=False)
    assert np.array_equal(a, b)


# ---------------------------------------------------------------- rope
def test_rope_identity_isometry_additivity():
    rng = np.random.default_rng(0)
    for dh in (16, 64, 128):
        k = rng.standard_normal(dh).astype(np.float32)
        assert np.array_equal(O.rope_apply(k, 0), k)
    # isometry per pair, 1000 random (k, s)
    for _ in range(1000):
        k = rng.standard_normal(64).astype(np.float32)
        s = int(rng.integers(0, 8192))
        r = O.rope_apply(k, s)
        n0 = np.hypot(k[0::2].astype(np.float64), k[1::2])
        n1 = np.hypot(r[0::2].astype(np.float64), r[1::2])
        assert np.max(np.abs(n0 - n1)) < 1e-5
    # additivity |RoPE(RoPE(k,s1),s2) - RoPE(k,s1+s2)|_inf <= 1e-6 (acceptance #1)
    worst = 0.0
    for _ in range(10000):
        dh = int(rng.choice([16, 64, 128]))
        k = rng.uniform(-1, 1, dh).astype(np.float32)
        s1, s2 = (int(x) for x in rng.integers(0, 8193, 2))
        a = O.rope_apply(O.rope_apply(k, s1), s2)
        b = O.rope_apply(k, s1 + s2)
        worst = max(worst, float(np.max(np.abs(a - b))))
    assert worst <= 1e-6, worst


def test_shift_rope_appendix_a_and_group_action():
    rng = np.random.default_rng(1)
    raw = rng.standard_normal((4, 64)).astype(np.float32)
    cached = np.stack([O.rope_apply(raw[i], p) for i, p in enumerate([2, 3, 4, 5])])
    shifted = np.stack([O.shift_rope(cached[i], p, p + 3) for i, p in enumerate([2, 3, 4, 5])])
    direct = np.stack([O.rope_apply(raw[i], p) for i, p in enumerate([5, 6, 7, 8])])
    assert np.max(np.abs(shifted - direct)) <= 1e-6
    x = rng.standard_normal(128).astype(np.float32)
    assert np.array_equal(O.shift_rope(x, 17, 17), x)
    for _ in range(200):
        a, b, c = (int(v) for v in rng.integers(0, 4097, 3))
        two = O.shift_rope(O.shift_rope(x, a, b), b, c)
        one = O.shift_rope(x, a, c)
        assert np.max(np.abs(two - one)) <= 1e-6  # SPEC.md:49 composition
    back = O.shift_rope(O.shift_rope(x, 10, 900), 900, 10)
    assert np.max(np.abs(back - x)) <= 1e-6  # inverse via negative delta


# ---------------------------------------------------------------- small model fixtures
SMALL = dict(layers=2, d_model=64, n_heads=4, n_kv_heads=2, head_dim=16, ffn_dim=128, vocab=64, rope_base=1e4,
             norm_eps=1e-5)


@pytest.fixture(scope="module")
def small():
    m = O.Model(SMALL).init_seed(99)
    # non-trivial gains so norms matter
    return m


def _prefill(m, tokens, start_pos=1, cache=None, slots=None, logit_rows=None, mask=None):
    n = len(tokens)
    if cache is None:
        cache = m.new_cache(start_pos - 1 + n)
    pos = np.arange(start_pos, start_pos + n, dtype=np.int32)
    sl = pos - 1 if slots is None else slots
    lg, _ = m.forward(tokens, pos, sl, *cache, mask=mask, logit_rows=logit_rows)
    return lg, cache


def test_prefill_equals_token_by_token_decode(small):
    rng = np.random.default_rng(2)
    for _ in range(10):
        n = int(rng.integers(2, 40))
        toks = rng.integers(0, 64, n)
        _, c_full = _prefill(small, toks)
        cache = small.new_cache(n)
        for i in range(n):
            small.forward([toks[i]], [i + 1], [i], *cache)
        assert np.max(np.abs(cache[0] - c_full[0])) <= 1e-5
        assert np.max(np.abs(cache[1] - c_full[1])) <= 1e-5


def test_prefix_reuse_eq4(small):
    rng = np.random.default_rng(3)
    for _ in range(10):
        L = int(rng.integers(4, 120))
        s = int(rng.integers(1, L))
        toks = rng.integers(0, 64, L)
        lg_full, _ = _prefill(small, toks, logit_rows=np.arange(L))
        cache = small.new_cache(L)
        _prefill(small, toks[:s], cache=cache)
        lg, _ = small.forward(toks[s:], np.arange(s + 1, L + 1), np.arange(s, L), *cache,
                              logit_rows=np.arange(L - s))
        assert np.max(np.abs(lg - lg_full[s:])) <= 1e-5  # SPEC.md:110, acceptance #2


def _isolated_records(m, sys_toks, chunks):
    S = len(sys_toks)
    recs = []
    for ch in chunks:
        cache = m.new_cache(S + len(ch))
        _prefill(m, np.concatenate([sys_toks, ch]), cache=cache)
        recs.append({"k": cache[0][:, S:].copy(), "v": cache[1][:, S:].copy(), "tokens": ch, "native_start": S + 1})
    sc = m.new_cache(S)
    if S:
        _prefill(m, sys_toks, cache=sc)
    return recs, (sc[0], sc[1]) if S else None


def test_full_reuse_equals_parallel_context_mask(small):
    # Fig. 4 / SPEC.md:406 / acceptance #3: FR question logits == dense attention under the
    # block-diagonal (parallel context windows) mask over cat(S, C1..Cn, Q)
    # The identity is exact when every window's chunk-to-prefix distances are
    # preserved: with S = 0 each window only attends to itself, so RoPE's
    # relative form makes the shifted cache equal the masked full forward.
    # (With a system prompt, an isolated record encodes the distance from its
    # native offset to S, which re-positioning does not change.)
    rng = np.random.default_rng(4)
    for _ in range(50):
        S = 0
        chunks = [rng.integers(0, 64, int(rng.integers(2, 12))) for _ in range(int(rng.integers(2, 5)))]
        q = rng.integers(0, 64, int(rng.integers(1, 5)))
        sys_toks = rng.integers(0, 64, S)
        recs, skv = _isolated_records(small, sys_toks, chunks)
        out = small.reprocess(skv, recs, q, 0.0, emulate_bf16=False)
        N = sum(len(c) for c in chunks)
        T = S + N + len(q)
        seg = np.concatenate([np.zeros(S, int)] + [np.full(len(c), i + 1) for i, c in enumerate(chunks)] +
                             [np.full(len(q), -1)])
        mask = np.zeros((T, T), np.uint8)
        for i in range(T):
            for j in range(i + 1):
                mask[i, j] = seg[i] == -1 or seg[j] == 0 or seg[j] == seg[i]
        toks = np.concatenate([sys_toks] + chunks + [q])
        cache = small.new_cache(T)
        lg, _ = small.forward(toks, np.arange(1, T + 1), np.arange(T), *cache, mask=mask, logit_rows=[T - 1])
        assert np.max(np.abs(lg[0] - out["logits"])) <= 1e-5


def test_endpoint_reduction(small):
    # SPEC.md:441-446 / acceptance #4: r=1 == Full Attention, r=0 == Full Reuse
    rng = np.random.default_rng(5)
    for _ in range(6):
        S = int(rng.integers(0, 4))
        chunks = [rng.integers(0, 64, int(rng.integers(2, 10))) for _ in range(3)]
        q = rng.integers(0, 64, 3)
        sys_toks = rng.integers(0, 64, S)
        recs, skv = _isolated_records(small, sys_toks, chunks)
        full = np.concatenate([sys_toks] + chunks + [q])
        lg_fa, _ = _prefill(small, full, logit_rows=[len(full) - 1])
        out1 = small.reprocess(skv, recs, q, 1.0, emulate_bf16=False)
        assert np.max(np.abs(out1["logits"] - lg_fa[0])) <= 1e-5
        assert np.argmax(out1["logits"]) == np.argmax(lg_fa[0])
        out0 = small.reprocess(skv, recs, q, 0.0, emulate_bf16=False)
        assert len(out0["crit"]) == 0


def test_selector_equals_brute_force():
    # SPEC.md:433, acceptance #6: exact equality with materialise + column-sum + sort
    rng = np.random.default_rng(6)
    for t in range(100):
        nq, Hkv, G, dh = int(rng.integers(1, 5)), int(rng.integers(1, 3)), int(rng.choice([1, 2, 4])), 16
        Hq = Hkv * G
        N = int(rng.integers(1, 200))
        k = int(rng.integers(0, N + 1))
        q = rng.standard_normal((nq, Hq, dh)).astype(np.float32)
        keys = rng.standard_normal((N, Hkv, dh)).astype(np.float32)
        raw = bool(t % 5 == 4)
        scores, sel = O.select(q, keys, k, raw=raw)
        kk = np.repeat(keys.astype(np.float64), G, axis=1)  # [N][Hq][dh]
        W = np.einsum("thd,nhd->thn", q.astype(np.float64), kk) / np.sqrt(dh)
        if not raw:
            W = np.exp(W - W.max(-1, keepdims=True))
            W /= W.sum(-1, keepdims=True)
        col = W.sum(axis=(0, 1))
        order = np.argsort(-col, kind="stable")
        assert np.allclose(scores, col, rtol=1e-12, atol=1e-12)
        assert np.array_equal(sel, np.sort(order[:k]))


def test_select_degenerate_cases():
    q = np.ones((1, 2, 16), np.float32)
    keys = np.ones((10, 1, 16), np.float32)  # all scores tie
    _, sel = O.select(q, keys, 4)
    assert sel.tolist() == [0, 1, 2, 3]  # ties -> lower index
    _, sel = O.select(q, keys, 10)
    assert sel.tolist() == list(range(10))  # r covering all tokens
    _, sel = O.select(q, keys, 0)
    assert sel.tolist() == []


# ---------------------------------------------------------------- sparse attention
def test_fig5_worked_example_mask():
    # S = X[1], chunks X[2:3], X[4:6], Q = X[7:8], critical {3, 5} -> q idx [3,5,7,8];
    # row X3 attends keys 1..3
    m = O.build_equivalent_mask([3, 5, 7, 8], [0, 0, 1, 1], 6)
    assert m.shape == (4, 8)
    assert m[0, :6].tolist() == [1, 1, 1, 0, 0, 0] and m[0, 6:].tolist() == [0, 0]
    assert m[1, :6].tolist() == [1, 1, 1, 1, 1, 0]
    assert m[3].tolist() == [1] * 8


def test_fig9_plan_masks_stale_originals():
    # chunk b tokens 6-10 cached, critical {6, 8}, user tokens {13,14,15} -> q_indices [6,8,13,14,15];
    # the stale originals at 6 and 8 are never read
    crit, user = [6, 8], [13, 14, 15]
    q_idx = sorted(crit + user)
    assert q_idx == [6, 8, 13, 14, 15]
    is_new = [0, 0, 1, 1, 1]
    rng = np.random.default_rng(7)
    H, dh, T = 2, 16, 12
    q = rng.standard_normal((5, H, dh)).astype(np.float32)
    sk, sv = rng.standard_normal((2, T, H, dh)).astype(np.float32)
    fk, fv = rng.standard_normal((2, 5, H, dh)).astype(np.float32)
    base = O.q_sparse_attn(q, sk, sv, fk, fv, q_idx, is_new)
    sk2, sv2 = sk.copy(), sv.copy()
    sk2[[5, 7]] += 100.0  # positions 6 and 8 (stale) perturbed
    sv2[[5, 7]] -= 50.0
    assert np.array_equal(O.q_sparse_attn(q, sk2, sv2, fk, fv, q_idx, is_new), base)
    sk3 = sk.copy()
    sk3[6] += 1.0  # position 7 (not critical) is read
    assert not np.array_equal(O.q_sparse_attn(q, sk3, sv, fk, fv, q_idx, is_new), base)


def test_q_sparse_attn_equals_dense_masked_200_plans():
    # SPEC.md:161/170, acceptance #5
    rng = np.random.default_rng(8)
    for t in range(200):
        T = int(rng.integers(4, 512))
        r = float(rng.choice([0.05, 0.15, 0.5, 1.0]))
        n_crit = max(0, min(T, int(np.floor(r * T + 0.5))))
        crit = np.sort(rng.choice(np.arange(1, T + 1), n_crit, replace=False))
        n_new = int(rng.integers(1, 6))
        new = np.arange(T + 1, T + 1 + n_new)
        q_idx = np.concatenate([crit, new]).astype(np.int32)
        is_new = np.concatenate([np.zeros(n_crit), np.ones(n_new)]).astype(np.uint8)
        H, dh = 2, 8
        nq = len(q_idx)
        q = rng.standard_normal((nq, H, dh)).astype(np.float32)
        sk, sv = rng.standard_normal((2, T, H, dh)).astype(np.float32)
        fk, fv = rng.standard_normal((2, nq, H, dh)).astype(np.float32)
        sk0, sv0 = sk.tobytes(), sv.tobytes()
        out = O.q_sparse_attn(q, sk, sv, fk, fv, q_idx, is_new)
        assert sk.tobytes() == sk0 and sv.tobytes() == sv0  # shared cache byte-identical
        # dense oracle over logical keys cat(shared with fresh at critical positions, new tokens)
        K = np.concatenate([sk, fk[is_new == 1]])
        V = np.concatenate([sv, fv[is_new == 1]])
        for i, p in enumerate(crit):
            K[p - 1], V[p - 1] = fk[i], fv[i]
        mask = O.build_equivalent_mask(q_idx, is_new, T)
        s = np.einsum("ihd,jhd->ihj", q.astype(np.float64), K.astype(np.float64)) / np.sqrt(dh)
        s = np.where(mask[:, None, :] == 1, s, -np.inf)
        w = np.exp(s - s.max(-1, keepdims=True))
        w /= w.sum(-1, keepdims=True)
        dense = np.einsum("ihj,jhd->ihd", w, V.astype(np.float64))
        assert np.max(np.abs(out - dense)) <= 1e-5


def test_invalid_plan_rejected():
    q = np.zeros((2, 1, 8), np.float32)
    with pytest.raises(ValueError):
        O.q_sparse_attn(q, np.zeros((4, 1, 8)), np.zeros((4, 1, 8)), q, q, [3, 2], [0, 0])


def test_reprocess_selection_never_touches_system_or_question(small):
    rng = np.random.default_rng(9)
    S = 3
    sys_toks = rng.integers(0, 64, S)
    chunks = [rng.integers(0, 64, 20) for _ in range(4)]
    q = rng.integers(0, 64, 5)
    recs, skv = _isolated_records(small, sys_toks, chunks)
    for r in (0.05, 0.15, 0.5, 1.0):
        out = small.reprocess(skv, recs, q, r)
        crit = out["crit"]
        assert len(crit) == int(np.floor(r * 80 + 0.5))
        assert np.all(crit >= S + 1) and np.all(crit <= S + 80)
        assert np.all(np.diff(crit) > 0)


def test_oracle_decode_equals_prefill_of_extended_prompt():
    """Prefill/decode equivalence: decoding tokens one by one over
    a prefilled cache gives the logits of a full prefill of the longer prompt."""
    from oracle import oracle as O
    cfg = dict(vocab=64, d_model=32, n_heads=4, n_kv_heads=2, head_dim=8, ffn_dim=64, layers=2,
               rope_base=1e4, norm_eps=1e-5)
    m = O.Model(cfg).init_seed(3)
    rng = np.random.default_rng(0)
    prompt = rng.integers(0, 64, 12).tolist()
    extra = rng.integers(0, 64, 4).tolist()
    T = len(prompt)
    k, v, pos = m.new_cache(T + len(extra))
    m.forward(prompt, list(range(1, T + 1)), list(range(T)), k, v, pos)
    step_logits = m.decode_forced(k, v, T, extra, emulate_bf16=False)
    full = prompt + extra
    k2, v2, pos2 = m.new_cache(len(full))
    ref, _ = m.forward(full, list(range(1, len(full) + 1)), list(range(len(full))), k2, v2, pos2,
                       logit_rows=list(range(T, len(full))))
    assert np.allclose(step_logits, ref, rtol=1e-4, atol=1e-5)
    assert np.allclose(k, k2, rtol=1e-5, atol=1e-6)
    # greedy decoding feeds back the argmax
    k3, v3, pos3 = m.new_cache(T + 4)
    lg, _ = m.forward(prompt, list(range(1, T + 1)), list(range(T)), k3, v3, pos3, logit_rows=[T - 1])
    toks = m.greedy_decode(k3, v3, T, lg[0], 4, emulate_bf16=False)
    assert toks[0] == int(np.argmax(lg[0])) and len(toks) == 4


# ---------------------------------------------------------------- CacheBlend
def test_kv_deviation_single_chunk_is_zero(small):
    # a single retrieved chunk -> Delta ~ 0 everywhere (FR == FA, Eq. 4)
    rng = np.random.default_rng(20)
    for S in (0, 3):
        sys_toks = rng.integers(0, 64, S)
        recs, skv = _isolated_records(small, sys_toks, [rng.integers(0, 64, 17)])
        dev = small.kv_deviation(skv, recs, n_layers=2, emulate_bf16=False)
        assert dev.shape == (17, 2, 2)
        assert np.max(dev) <= 1e-10


def test_kv_deviation_first_layer_zero_second_layer_positive(small):
    # layer-1 Delta = 0 (embeddings + positions only); SPEC.md:416:
    # chunk 2 after chunk 1 -> layer-2 Delta strictly positive on chunk-2 tokens,
    # while chunk 1 (at its native offset) has Delta = 0
    rng = np.random.default_rng(21)
    for S in (0, 2):
        sys_toks = rng.integers(0, 64, S)
        c1, c2 = rng.integers(0, 64, 9), rng.integers(0, 64, 11)
        recs, skv = _isolated_records(small, sys_toks, [c1, c2])
        dev = small.kv_deviation(skv, recs, n_layers=2, emulate_bf16=False)
        assert np.all(dev[:, 0, 1] == 0.0)  # V of layer 1: same row, same GEMM
        assert np.max(dev[:, 0, 0]) <= 1e-9  # K of layer 1: shift-rotation rounding only
        assert np.max(dev[:9, 1, :]) <= 1e-10
        assert np.all(dev[9:, 1, 0] > 1e-8) and np.all(dev[9:, 1, 1] > 1e-8)


def test_select_cacheblend_equals_brute_force_sort():
    # SPEC.md:421-425, acceptance #6: exact argTopk of the deviation column, lower index on ties
    rng = np.random.default_rng(22)
    for t in range(100):
        N, L = int(rng.integers(1, 300)), int(rng.integers(2, 4))
        dev = rng.random((N, L, 2))
        if t % 4 == 0:
            dev = np.round(dev, 1)  # many ties
        k = int(rng.integers(0, N + 1))
        layer, comp = int(rng.integers(1, L + 1)), int(rng.integers(0, 3))
        sel = O.select_cacheblend(dev, k, layer, comp)
        col = dev[:, layer - 1, 0] + dev[:, layer - 1, 1] if comp == 2 else dev[:, layer - 1, comp]
        assert np.array_equal(sel, np.sort(np.argsort(-col, kind="stable")[:k]))
    dev = np.ones((10, 2, 2))
    assert O.select_cacheblend(dev, 0).tolist() == []  # r = 0 -> empty
    assert O.select_cacheblend(dev, 10).tolist() == list(range(10))  # r = 1 -> all chunk tokens
    assert O.select_cacheblend(dev, 3).tolist() == [0, 1, 2]


# ---------------------------------------------------------------- alternative_path_match
def test_alt_path_paper_query3():
    # Query1 caches b under S, Query2 caches a under S; Query3 context [b, a]:
    # b via PREFIX, a via ALT_PATH (path "system prompt + Chunk a")
    cached = {("S", ("b",)), ("S", ("a",))}
    got = O.alt_path_match(cached, {"a", "b"}, ["b", "a"], "S")
    assert got == [("b", "PREFIX", 0, 0), ("a", "ALT_PATH", 1, 1)]
    assert O.alt_path_match(cached, {"a", "b"}, ["x", "y"], "S") == []  # uncached context -> empty


def test_alt_path_permutations_and_completeness():
    import itertools
    # every chunk cached under "S + chunk": every permutation of any subset matches all
    for N in range(1, 6):
        chunks = [f"c{i}" for i in range(N)]
        cached = {("S", (c,)) for c in chunks}
        for r in range(1, N + 1):
            for sub in itertools.permutations(chunks, r):
                got = O.alt_path_match(cached, set(chunks), list(sub), "S")
                assert [g[0] for g in got] == list(sub)
    # completeness: a record cached under a longer path still matches anywhere
    cached = {("S", ("a", "c"))}
    got = O.alt_path_match(cached, {"a", "c"}, ["b", "c"], "S")
    assert got == [("c", "ALT_PATH", 1, 1)]
    assert O.alt_path_match(cached, {"a", "c"}, ["a", "c"], "S")[1] == ("c", "PREFIX", 1, 0)


def test_alt_path_hit_rate_dominates_plain_prefix():
    # alt-path hits >= plain prefix-cache hits on any workload
    rng = np.random.default_rng(7)
    chunks = [f"k{i}" for i in range(12)]
    cached, records = set(), set()
    alt = plain = 0
    for _ in range(300):
        ctx = list(rng.choice(chunks, int(rng.integers(1, 6)), replace=False))
        got = O.alt_path_match(cached, records, ctx, "S")
        alt += len(got)
        plain += sum(1 for g in got if g[1] == "PREFIX")
        for i, c in enumerate(ctx):  # the query caches its chunks under its own context
            records.add(c)
            cached.add(("S", tuple(ctx[:i + 1])))
    assert alt >= plain and alt > 0
