"""GPU (libfrag.so, sm_100a) vs CPU oracle parity on identical inputs.

Tolerances:
  * weights: bf16 weights generated on the GPU equal the oracle's Rng restatement
    (device fp64 log/sin/cos may differ in the last ulp: <= 1e-5 of elements may
    differ by one bf16 ulp);
  * K1 stitched rows that are not recomputed: bit-exact;
  * selection (K9+K10) on identical final-layer queries/keys: bit-exact set except
    indices whose oracle score lies within eps = 1e-4 * mean score of the k-th score;
  * recomputed fused K/V and logits ("selection-injection" mode, both sides use
    the GPU's critical set): relative L2 <= 2e-2, cosine >= 0.999 vs the
    bf16-emulating oracle; first-token argmax equal unless the top-2 gap < 1e-2.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rel_l2(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _cos(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return float(a @ b / max(np.linalg.norm(a) * np.linalg.norm(b), 1e-30))


def _setup(preset_or_cfg, n_chunks, chunk_len, S, nq, seed=1234, data_seed=7):
    from paper_2601_12904_b200 import fusion as F
    from oracle import oracle as O
    eng = F.Engine(preset_or_cfg, seed=seed)
    c = eng.cfg
    store = F.ChunkKVStore(c)
    rng = np.random.default_rng(data_seed)
    system = rng.integers(0, c.vocab, S).tolist()
    chunks = [rng.integers(0, c.vocab, chunk_len).tolist() for _ in range(n_chunks)]
    ids = [eng.preprocess_isolated(store, ch, system=system) for ch in chunks]
    question = rng.integers(0, c.vocab, nq).tolist()
    res = F.Result(eng, S + n_chunks * chunk_len + nq)
    om = O.Model(c).load_from_engine(eng)
    recs = []
    for i, ch in zip(ids, chunks):
        k, v = store.read_kv(i)
        recs.append({"k": O.bf16_bits_to_f32(k), "v": O.bf16_bits_to_f32(v), "tokens": ch,
                     "native_start": S + 1})
    return dict(F=F, O=O, eng=eng, store=store, system=system, chunks=chunks, ids=ids, question=question,
                res=res, om=om, recs=recs, S=S)


@pytest.fixture(scope="module")
def tiny(cuda):
    return _setup("tiny", 8, 256, 8, 32)


def test_weights_match_rng_restatement(tiny):
    eng, O = tiny["eng"], tiny["O"]
    c = eng.cfg
    checks = [("emb", 0, 0), ("lm_head", 0, 1), ("wq", 0, 16), ("wk", 1, 25), ("w_up", 1, 29), ("w_down", 0, 22)]
    for name, layer, tid in checks:
        gpu = eng.weight(name, layer).ravel()
        ref = O.gen_normal(O.weight_seed(eng.seed, tid), gpu.size, 0.02)
        mism = np.count_nonzero(gpu != ref)
        assert mism <= max(1, gpu.size // 100000), (name, mism)
        if mism:
            d = np.abs(gpu - ref)[gpu != ref]
            assert np.all(d <= np.abs(ref[gpu != ref]) * 2 ** -7)


def _gpu_run(t, ratio, **kw):
    t["eng"].reprocess(t["store"], t["question"], t["ids"], ratio, t["res"], system=t["system"], **kw)
    k, v = t["res"].fused_kv()
    return {"k": k, "v": v, "logits": t["res"].logits()[0], "crit": t["res"].crit(), "debug": t["res"].debug()}


def test_stitch_rows_bit_exact(tiny):
    O, S = tiny["O"], tiny["S"]
    g = _gpu_run(tiny, 0.0)
    sys_k, sys_v = g["k"][:, :S], g["v"][:, :S]
    chunks = [(O.bf16_bits_to_f32(sys_k), O.bf16_bits_to_f32(sys_v), 1, 0)]
    row = S
    for r in tiny["recs"]:
        chunks.append((r["k"], r["v"], r["native_start"], row))
        row += len(r["tokens"])
    ko, vo = O.stitch(tiny["eng"].cfg, chunks, row)
    # r = 0: only question rows were recomputed, every stitched row is K1 output
    assert np.array_equal(g["k"][:, :row], O.f32_to_bf16_bits(ko))
    assert np.array_equal(g["v"][:, :row], O.f32_to_bf16_bits(vo))


def test_selection_bit_exact_on_identical_inputs(tiny):
    O, S = tiny["O"], tiny["S"]
    for ratio in (0.05, 0.15, 0.3):
        g = _gpu_run(tiny, ratio)
        c = tiny["eng"].cfg
        N = 8 * 256
        qf = g["debug"]["q_final"]
        # selection reads the STITCHED final-layer keys (before the sparse pass
        # overwrites the critical rows): the oracle stitch of the same records,
        # bit-exact with K1 (test_stitch_rows_bit_exact)
        chunks = [(r["k"], r["v"], r["native_start"], S + i * 256) for i, r in enumerate(tiny["recs"])]
        ko, _ = O.stitch(c, chunks, S + N)
        keys = ko[c.layers - 1, S:S + N]
        k = int(np.floor(ratio * N + 0.5))
        scores, sel = O.select(qf, keys, k)
        gpu_sel = g["crit"] - S - 1
        assert len(gpu_sel) == k
        # GPU scores track the fp64 oracle scores to fp32 rounding
        assert np.allclose(g["debug"]["scores"], scores, rtol=1e-4, atol=1e-7)
        tau = np.sort(scores)[::-1][k - 1]
        eps = 1e-4 * scores.mean()
        diff = set(gpu_sel.tolist()) ^ set(sel.tolist())
        assert all(abs(scores[j] - tau) <= eps for j in diff), [(j, scores[j] - tau) for j in diff]


def test_reprocess_selection_injection_parity(tiny):
    O, S = tiny["O"], tiny["S"]
    for ratio in (0.0, 0.15, 1.0):
        g = _gpu_run(tiny, ratio)
        sys_kv = (O.bf16_bits_to_f32(g["k"][:, :S]), O.bf16_bits_to_f32(g["v"][:, :S]))
        out = tiny["om"].reprocess(sys_kv, tiny["recs"], tiny["question"], ratio, inject=g["crit"],
                                   emulate_bf16=True)
        ok = O.f32_to_bf16_bits(out["k"])
        ov = O.f32_to_bf16_bits(out["v"])
        T = out["T"]
        recomputed = np.zeros(T, bool)
        recomputed[g["crit"] - 1] = True
        recomputed[T - len(tiny["question"]):] = True
        # untouched stitched rows: bit-exact
        assert np.array_equal(g["k"][:, ~recomputed], ok[:, ~recomputed])
        assert np.array_equal(g["v"][:, ~recomputed], ov[:, ~recomputed])
        gk = O.bf16_bits_to_f32(g["k"][:, recomputed])
        rk = O.bf16_bits_to_f32(ok[:, recomputed])
        gv = O.bf16_bits_to_f32(g["v"][:, recomputed])
        rv = O.bf16_bits_to_f32(ov[:, recomputed])
        assert _rel_l2(gk, rk) <= 2e-2 and _cos(gk, rk) >= 0.999
        assert _rel_l2(gv, rv) <= 2e-2 and _cos(gv, rv) >= 0.999
        assert _rel_l2(g["logits"], out["logits"]) <= 2e-2 and _cos(g["logits"], out["logits"]) >= 0.999
        top = np.sort(out["logits"])[::-1]
        if top[0] - top[1] >= 1e-2:
            assert np.argmax(g["logits"]) == np.argmax(out["logits"])


def test_end_to_end_selection_window(tiny):
    """Full pipeline, each side runs its own question pass and selector. With
    delta = max_j |score_gpu[j] - score_oracle[j]| (the score perturbation the
    bf16 drift of q_final induces), every index in the symmetric difference of
    the two critical sets lies within 2*delta of the oracle's k-th score: the
    GPU's top-k is exact on its own scores, so a swap needs both scores within
    delta of the boundary. q_final itself: rel L2 <= 1e-2 vs the oracle's."""
    O, S = tiny["O"], tiny["S"]
    g = _gpu_run(tiny, 0.15)
    sys_kv = (O.bf16_bits_to_f32(g["k"][:, :S]), O.bf16_bits_to_f32(g["v"][:, :S]))
    out = tiny["om"].reprocess(sys_kv, tiny["recs"], tiny["question"], 0.15, emulate_bf16=True)
    assert _rel_l2(g["debug"]["q_final"], out["q_final"]) <= 1e-2
    a, b = g["crit"] - S - 1, out["crit"] - S - 1
    assert len(a) == len(b)
    so = out["scores"]
    delta = float(np.abs(g["debug"]["scores"].astype(np.float64) - so).max())
    tau = np.sort(so)[::-1][len(b) - 1]
    win = 2.0 * delta + 1e-6 * abs(tau)
    diff = set(a.tolist()) ^ set(b.tolist())
    print(f"tiny e2e selection: score delta {delta:.3e} (mean {so.mean():.3e}), {len(diff) // 2} swaps "
          f"of {len(a)}, window {win:.3e}")
    assert delta <= 5e-2 * so.mean(), (delta, so.mean())
    assert all(abs(so[j] - tau) <= win for j in diff), [(j, so[j] - tau) for j in diff if abs(so[j] - tau) > win]


@pytest.mark.slow
@pytest.mark.parametrize("preset,layers,n_chunks", [("llama3-8b", 2, 4), ("mistral-7b", 2, 4), ("llama3-70b", 1, 2)])
def test_large_width_reduced_depth_parity(cuda, preset, layers, n_chunks):
    """Full-width layers of the bench presets at reduced depth: Llama-3-8B (d=4096,
    GQA 32/8, F=14336, V=128256), Mistral-7B (V=32768, RoPE base 1e6) and
    Llama-3-70B (d=8192, GQA 64/8 -> 8 heads per KV group, F=28672)."""
    from paper_2601_12904_b200 import fusion as F
    cfg = F.preset(preset)
    cfg.layers = layers
    t = _setup(cfg, n_chunks, 256, 0, 32)
    O = t["O"]
    g = _gpu_run(t, 0.15)
    out = t["om"].reprocess(None, t["recs"], t["question"], 0.15, inject=g["crit"], emulate_bf16=True)
    assert _rel_l2(g["logits"], out["logits"]) <= 3e-2 and _cos(g["logits"], out["logits"]) >= 0.999
    rk = O.bf16_bits_to_f32(O.f32_to_bf16_bits(out["k"]))
    gk = O.bf16_bits_to_f32(g["k"])
    assert _rel_l2(gk, rk) <= 3e-2
    # selection on identical inputs (stitched keys, before the sparse pass)
    N = n_chunks * 256
    chunks = [(r["k"], r["v"], r["native_start"], i * 256) for i, r in enumerate(t["recs"])]
    ko, _ = O.stitch(cfg, chunks, N)
    keys = ko[cfg.layers - 1]
    scores, sel = O.select(g["debug"]["q_final"], keys, len(g["crit"]))
    tau = np.sort(scores)[::-1][len(sel) - 1]
    diff = set((g["crit"] - 1).tolist()) ^ set(sel.tolist())
    assert all(abs(scores[j] - tau) <= 1e-4 * scores.mean() for j in diff)


def test_decode_parity_teacher_forced(tiny):
    """Greedy decode after a 15% reprocess vs the oracle fed the same tokens
    over its own (selection-injected, bf16-emulating) fused cache: decoded K/V
    rows and final logits within the reprocess tolerances, and every greedy
    choice equal to the oracle's argmax unless its top-2 gap < 1e-2."""
    F, O, S, eng = tiny["F"], tiny["O"], tiny["S"], tiny["eng"]
    T = S + 8 * 256 + 32
    n = 6
    res = F.Result(eng, T + n)
    eng.reprocess(tiny["store"], tiny["question"], tiny["ids"], 0.15, res, system=tiny["system"])
    crit = res.crit()
    k0, v0 = res.fused_kv()
    toks = eng.decode(res, n)
    kd, vd = res.fused_kv()
    last = res.logits()[0]
    sys_kv = (O.bf16_bits_to_f32(k0[:, :S]), O.bf16_bits_to_f32(v0[:, :S]))
    out = tiny["om"].reprocess(sys_kv, tiny["recs"], tiny["question"], 0.15, inject=crit, emulate_bf16=True,
                               cap=T + n)
    steps = tiny["om"].decode_forced(out["k_cache"], out["v_cache"], T, toks[:-1], emulate_bf16=True)
    prev = [out["logits"]] + list(steps[:-1])
    for i, lg in enumerate(prev):
        top = np.sort(lg)[::-1]
        if top[0] - top[1] >= 1e-2:
            assert int(toks[i]) == int(np.argmax(lg)), i
    assert _rel_l2(last, steps[-1]) <= 2e-2 and _cos(last, steps[-1]) >= 0.999
    gk = O.bf16_bits_to_f32(kd[:, T:T + n - 1])
    rk = O.bf16_bits_to_f32(O.f32_to_bf16_bits(out["k_cache"][:, T:T + n - 1]))
    assert _rel_l2(gk, rk) <= 2e-2 and _cos(gk, rk) >= 0.999


def test_preprocess_fused(cuda):
    """Eq. 10: FUSED records. top_n = 0 -> the ISOLATED
    record exactly; C2 fused against its real predecessor C1 reproduces the
    Full-Attention KV of C2 in cat(S, C1, C2) (strictly closer than the
    ISOLATED record, the §3.1 deviation claim) and matches the oracle's
    prefill over the stitched context; budget truncation; missing neighbour."""
    t = _setup("tiny", 3, 256, 8, 32)
    F, O, eng, store, S = t["F"], t["O"], t["eng"], t["store"], t["S"]
    c1, c2, c3 = t["chunks"]
    i1, i2, i3 = t["ids"]
    out = F.ChunkKVStore(eng.cfg)
    f0 = eng.preprocess_fused(store, c2, [], system=t["system"], dst=out)
    r0 = out.peek(f0)
    assert f0 == i2 and r0.variant == F.FUSED and r0.native_start == S + 1
    a, b = out.read_kv(f0), store.read_kv(i2)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    # C2 fused against C1 (then C3, truncated by the 256-token budget)
    f2 = eng.preprocess_fused(store, c2, [i1, i3], system=t["system"], dst=out, budget=256, overwrite=True)
    r2 = out.peek(f2)
    assert r2.variant == F.FUSED and r2.native_start == S + 256 + 1
    kf, vf = out.read_kv(f2)
    # Full Attention of cat(S, C1, C2): rows of C2
    fa = F.Result(eng, S + 512)
    eng.full_prefill(c1 + c2, fa, system=t["system"])
    kfa, vfa = fa.fused_kv()
    k_fa = O.bf16_bits_to_f32(kfa[:, S + 256:S + 512])
    k_fu = O.bf16_bits_to_f32(kf)
    rec2 = t["recs"][1]  # the ISOLATED record of C2 re-positioned to S+257.. (Full Reuse)
    k_iso = O.stitch(eng.cfg, [(rec2["k"], rec2["v"], rec2["native_start"], S + 256)], S + 512)[0][:, S + 256:]
    dev_fu = float(np.sum((k_fu[1] - k_fa[1]) ** 2))
    dev_iso = float(np.sum((k_iso[1] - k_fa[1]) ** 2))
    assert _rel_l2(k_fu, k_fa) <= 1e-2 and dev_fu < 0.1 * dev_iso, (dev_fu, dev_iso)
    # oracle: prefill C2 at positions S+257.. over the stitched (S + C1) cache
    sys_kv = (O.bf16_bits_to_f32(kfa[:, :S]), O.bf16_bits_to_f32(vfa[:, :S]))
    rec1 = t["recs"][0]
    ck, cv = O.stitch(eng.cfg, [(sys_kv[0], sys_kv[1], 1, 0), (rec1["k"], rec1["v"], rec1["native_start"], S)],
                      S + 512)
    pos = np.zeros(S + 512, np.int32)
    pos[:S + 256] = np.arange(1, S + 257)
    t["om"].forward(c2, list(range(S + 257, S + 513)), list(range(S + 256, S + 512)), ck, cv, pos,
                    emulate_bf16=True)
    ko = O.bf16_bits_to_f32(O.f32_to_bf16_bits(ck[:, S + 256:S + 512]))
    assert _rel_l2(k_fu, ko) <= 2e-2 and _cos(k_fu, ko) >= 0.999
    with pytest.raises(F.StoreError, match="missing neighbour"):
        eng.preprocess_fused(store, c3, [F.hash_tokens([1, 2, 3])], dst=out)


@pytest.mark.parametrize("lens,S,nq,ratio", [((37, 256, 1, 129), 3, 1, 0.15), ((300, 5), 0, 7, 0.5),
                                             ((1,), 1, 2, 1.0), ((64, 64, 64), 8, 32, 0.0)])
def test_ragged_chunks_parity(cuda, lens, S, nq, ratio):
    """Ragged inputs (chunks of 1..300 tokens, 0-8 system tokens, 1-32 question
    tokens, r from 0 to 1): stitched rows bit-exact, selection invariants, and
    logits / recomputed rows vs the bf16-emulating oracle (injection mode)."""
    from paper_2601_12904_b200 import fusion as F
    from oracle import oracle as O
    eng = F.Engine("tiny", seed=99)
    c = eng.cfg
    store = F.ChunkKVStore(c)
    rng = np.random.default_rng(sum(lens) + S)
    system = rng.integers(0, c.vocab, S).tolist()
    chunks = [rng.integers(0, c.vocab, n).tolist() for n in lens]
    ids = [eng.preprocess_isolated(store, ch, system=system) for ch in chunks]
    question = rng.integers(0, c.vocab, nq).tolist()
    N = sum(lens)
    T = S + N + nq
    res = F.Result(eng, T)
    eng.reprocess(store, question, ids, ratio, res, system=system)
    k, v = res.fused_kv()
    crit = res.crit()
    assert len(crit) == int(np.floor(ratio * N + 0.5))
    assert np.all(np.diff(crit) > 0) and (len(crit) == 0 or (crit.min() > S and crit.max() <= S + N))
    om = O.Model(c).load_from_engine(eng)
    recs = []
    for i, ch in zip(ids, chunks):
        rk, rv = store.read_kv(i)
        recs.append({"k": O.bf16_bits_to_f32(rk), "v": O.bf16_bits_to_f32(rv), "tokens": ch, "native_start": S + 1})
    sys_kv = (O.bf16_bits_to_f32(k[:, :S]), O.bf16_bits_to_f32(v[:, :S])) if S else None
    out = om.reprocess(sys_kv, recs, question, ratio, inject=crit, emulate_bf16=True)
    fresh = np.zeros(T, bool)
    fresh[crit - 1] = True
    fresh[T - nq:] = True
    ok = O.f32_to_bf16_bits(out["k"])
    assert np.array_equal(k[:, ~fresh], ok[:, ~fresh])  # stitched rows (K1) bit-exact
    assert _rel_l2(res.logits()[0], out["logits"]) <= 2e-2 and _cos(res.logits()[0], out["logits"]) >= 0.999
    gk, rk = O.bf16_bits_to_f32(k[:, fresh]), O.bf16_bits_to_f32(ok[:, fresh])
    assert _rel_l2(gk, rk) <= 2e-2


def test_no_chunks_is_question_prefill(cuda):
    """A request with no retrieved chunks is the plain prefill of cat(S, Q)."""
    from paper_2601_12904_b200 import fusion as F
    eng = F.Engine("tiny", seed=99)
    store = F.ChunkKVStore(eng.cfg)
    rng = np.random.default_rng(3)
    system = rng.integers(0, eng.cfg.vocab, 4).tolist()
    question = rng.integers(0, eng.cfg.vocab, 12).tolist()
    res = F.Result(eng, 16)
    eng.reprocess(store, question, [], 0.15, res, system=system)
    assert len(res.crit()) == 0
    fa = F.Result(eng, 16)
    eng.full_prefill(question, fa, system=system)
    assert _rel_l2(res.logits()[0], fa.logits()[0]) <= 1e-2
    assert np.argmax(res.logits()[0]) == np.argmax(fa.logits()[0]) or \
        np.sort(fa.logits()[0])[-1] - np.sort(fa.logits()[0])[-2] < 1e-2
