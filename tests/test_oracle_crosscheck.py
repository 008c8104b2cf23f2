"""Cross-check of the CPU oracle's transformer (oracle/fusion_oracle.cpp) against
a second, independent restatement of SPEC.md's tiny_transformer written here
in torch float64 straight from the spec text: pre-norm RMS blocks, RoPE on Q
and K with θ_i = base^(−2i/d), i = 1..d/2, interleaved pairs and
rotate(k) = [−k2, k1, −k4, k3, …], attention scale 1/√dh
with the causal-by-position mask, gated feed-forward
silu(gate)·up, final norm, lm_head; GQA maps query head h to KV head
h / (Hq / Hkv). The oracle is the parity checker of every
GPU test, and the reference ships no executable model to pin it against, so
two independent restatements agreeing (≤ 1e−5 relative) is the pin for this
part of it. Weight layout: every projection stored [out][in] row-major."""
import numpy as np
import pytest
import torch

from oracle import oracle as O

CFGS = {
    "tiny": dict(layers=2, d_model=256, n_heads=4, n_kv_heads=4, head_dim=64, ffn_dim=1024, vocab=256,
                 rope_base=10000.0, norm_eps=1e-5),
    # GQA, non-square projections (Hq*dh != d), a Llama-3-style RoPE base
    "gqa": dict(layers=3, d_model=96, n_heads=4, n_kv_heads=2, head_dim=32, ffn_dim=160, vocab=64,
                rope_base=500000.0, norm_eps=1e-5),
}


def _w(m, name, layer, shape):
    return torch.from_numpy(np.array(m.tensor(name, layer), dtype=np.float64).reshape(shape))


def _rope(x, pos, base):
    """x [n, heads, dh]; pos [n] (1-based positions as given)."""
    dh = x.shape[-1]
    i = torch.arange(1, dh // 2 + 1, dtype=torch.float64)
    theta = base ** (-2.0 * i / dh)                                   # [dh/2]
    ang = pos.to(torch.float64)[:, None] * theta[None, :]             # [n, dh/2]
    cos, sin = torch.cos(ang)[:, None, :], torch.sin(ang)[:, None, :]
    a, b = x[..., 0::2], x[..., 1::2]                                 # pairs (k_{2i-1}, k_{2i})
    out = torch.empty_like(x)
    out[..., 0::2] = a * cos - b * sin                                # k·cos + rotate(k)·sin, rotate = [-k2, k1, ...]
    out[..., 1::2] = b * cos + a * sin
    return out


def _rms(x, g, eps):
    return x / torch.sqrt((x * x).mean(-1, keepdim=True) + eps) * g


def _forward(m, c, tokens, pos):
    d, Hq, Hkv, dh, F, V = c["d_model"], c["n_heads"], c["n_kv_heads"], c["head_dim"], c["ffn_dim"], c["vocab"]
    x = _w(m, "emb", 0, (V, d))[torch.as_tensor(tokens)]
    n = x.shape[0]
    mask = pos[None, :] <= pos[:, None]                               # key position <= query position
    for l in range(c["layers"]):
        h = _rms(x, _w(m, "attn_norm", l, (d,)), c["norm_eps"])
        q = (h @ _w(m, "wq", l, (Hq * dh, d)).T).view(n, Hq, dh)
        k = (h @ _w(m, "wk", l, (Hkv * dh, d)).T).view(n, Hkv, dh)
        v = (h @ _w(m, "wv", l, (Hkv * dh, d)).T).view(n, Hkv, dh)
        q, k = _rope(q, pos, c["rope_base"]), _rope(k, pos, c["rope_base"])
        kv = torch.arange(Hq) // (Hq // Hkv)
        s = torch.einsum("qhd,khd->hqk", q, k[:, kv]) / dh ** 0.5
        s = s.masked_fill(~mask[None], float("-inf"))
        p = torch.softmax(s, dim=-1)
        o = torch.einsum("hqk,khd->qhd", p, v[:, kv]).reshape(n, Hq * dh)
        x = x + o @ _w(m, "wo", l, (d, Hq * dh)).T
        h = _rms(x, _w(m, "ffn_norm", l, (d,)), c["norm_eps"])
        g = h @ _w(m, "w_gate", l, (F, d)).T
        u = h @ _w(m, "w_up", l, (F, d)).T
        x = x + (torch.nn.functional.silu(g) * u) @ _w(m, "w_down", l, (d, F)).T
    x = _rms(x, _w(m, "final_norm", 0, (d,)), c["norm_eps"])
    return x @ _w(m, "lm_head", 0, (V, d)).T


@pytest.mark.parametrize("name", sorted(CFGS))
@pytest.mark.parametrize("seed", [3, 11])
def test_oracle_forward_equals_independent_restatement(name, seed):
    c = CFGS[name]
    m = O.Model(c).init_seed(seed)
    rng = np.random.default_rng(seed)
    n = 40
    tokens = rng.integers(0, c["vocab"], n)
    pos = np.arange(1, n + 1, dtype=np.int32) + 5                      # positions need not start at 1
    ck, cv, cp = m.new_cache(n)
    logits, _ = m.forward(tokens, pos, np.arange(n, dtype=np.int32), ck, cv, cp, logit_rows=np.arange(n))
    ref = _forward(m, c, tokens, torch.as_tensor(pos.astype(np.int64))).numpy()
    rel = np.linalg.norm(logits - ref) / np.linalg.norm(ref)
    assert rel <= 1e-5, rel


def test_oracle_forward_with_out_of_order_positions_equals_restatement():
    """Stitched caches are out of array order (the mask is keyed on
    positions); the restatement's mask is too -- a permuted position list must
    agree as well."""
    c = CFGS["gqa"]
    m = O.Model(c).init_seed(5)
    rng = np.random.default_rng(9)
    n = 24
    tokens = rng.integers(0, c["vocab"], n)
    pos = (rng.permutation(n) + 1).astype(np.int32)
    ck, cv, cp = m.new_cache(n)
    logits, _ = m.forward(tokens, pos, np.arange(n, dtype=np.int32), ck, cv, cp, logit_rows=np.arange(n))
    ref = _forward(m, c, tokens, torch.as_tensor(pos.astype(np.int64))).numpy()
    assert np.linalg.norm(logits - ref) / np.linalg.norm(ref) <= 1e-5


@pytest.mark.parametrize("Hq,Hkv", [(4, 4), (8, 2)])
@pytest.mark.parametrize("raw", [False, True])
def test_oracle_query_guided_scores_equal_independent_restatement(Hq, Hkv, raw):
    """select_query_guided's column scores: scaled dot
    products of every (question token, head) final-layer query with every
    chunk key of its KV head, softmax jointly over all chunk keys per (token,
    head) (raw=True: the un-normalised variant behind the flag),
    summed over heads and question tokens; then the global top-k with the
    lower index winning ties."""
    rng = np.random.default_rng(Hq * 10 + Hkv + raw)
    nq, dh, N, k = 5, 32, 300, 45
    q = rng.standard_normal((nq, Hq, dh)).astype(np.float32)
    keys = rng.standard_normal((N, Hkv, dh)).astype(np.float32)
    scores, sel = O.select(q, keys, k, raw=raw)
    qt, kt = torch.from_numpy(q).double(), torch.from_numpy(keys).double()
    kv = torch.arange(Hq) // (Hq // Hkv)
    s = torch.einsum("thd,nhd->thn", qt, kt[:, kv]) / dh ** 0.5    # [nq, Hq, N]
    w = s if raw else torch.softmax(s, dim=-1)
    ref = w.sum(dim=(0, 1)).numpy()
    assert np.allclose(scores, ref, rtol=1e-5, atol=1e-6 * np.abs(ref).max())
    order = sorted(range(N), key=lambda j: (-ref[j], j))[:k]
    assert sel.tolist() == sorted(order)


def test_oracle_stitch_equals_independent_shift():
    """stitch_full_reuse: each chunk's K re-rotated by
    delta = target_start - native_start as apply_rope(k, delta), V copied,
    chunks placed at their destination rows."""
    c = CFGS["gqa"]

    class Cfg:  # the oracle reads these fields
        pass
    cfg = Cfg()
    for f, v in c.items():
        setattr(cfg, f, v)
    rng = np.random.default_rng(4)
    L, Hkv, dh = c["layers"], c["n_kv_heads"], c["head_dim"]
    chunks, cap = [], 0
    for n, native, dst in [(7, 1, 0), (11, 9, 7), (5, 1, 18)]:
        k = rng.standard_normal((L, n, Hkv, dh)).astype(np.float32)
        v = rng.standard_normal((L, n, Hkv, dh)).astype(np.float32)
        chunks.append((k, v, native, dst))
        cap = max(cap, dst + n)
    ko, vo = O.stitch(cfg, chunks, cap, round_bf16=False)
    for k, v, native, dst in chunks:
        n = k.shape[1]
        delta = (dst + 1) - native  # target position of the chunk's first row (1-based) minus its native start
        for l in range(L):
            ref = _rope(torch.from_numpy(k[l]).double(), torch.full((n,), float(delta)), c["rope_base"]).numpy()
            assert np.allclose(ko[l, dst:dst + n], ref, rtol=0, atol=2e-6), (l, dst)
            assert np.array_equal(vo[l, dst:dst + n], v[l])


def _layers(m, c, x, pos, cache_k, cache_v, cache_pos, rows=None):
    """Run hidden states x [n, d] at positions pos through every layer. Each
    layer writes the new rows' K/V into the cache (at `rows`, or appended when
    rows is None) and attends over every cache entry whose position is <= the
    query's. Returns the final hidden states and the last layer's post-RoPE
    queries."""
    d, Hq, Hkv, dh, F = c["d_model"], c["n_heads"], c["n_kv_heads"], c["head_dim"], c["ffn_dim"]
    n = x.shape[0]
    kv = torch.arange(Hq) // (Hq // Hkv)
    q_last = None
    for l in range(c["layers"]):
        h = _rms(x, _w(m, "attn_norm", l, (d,)), c["norm_eps"])
        q = _rope((h @ _w(m, "wq", l, (Hq * dh, d)).T).view(n, Hq, dh), pos, c["rope_base"])
        k = _rope((h @ _w(m, "wk", l, (Hkv * dh, d)).T).view(n, Hkv, dh), pos, c["rope_base"])
        v = (h @ _w(m, "wv", l, (Hkv * dh, d)).T).view(n, Hkv, dh)
        if rows is None:
            K, Vv, P = torch.cat([cache_k[l], k]), torch.cat([cache_v[l], v]), torch.cat([cache_pos, pos])
        else:
            cache_k[l][rows], cache_v[l][rows] = k, v  # fresh rows replace the stale ones
            K, Vv, P = cache_k[l], cache_v[l], cache_pos
        s = torch.einsum("qhd,khd->hqk", q, K[:, kv]) / dh ** 0.5
        s = s.masked_fill(~(P[None, :] <= pos[:, None])[None], float("-inf"))
        o = torch.einsum("hqk,khd->qhd", torch.softmax(s, dim=-1), Vv[:, kv]).reshape(n, Hq * dh)
        x = x + o @ _w(m, "wo", l, (d, Hq * dh)).T
        h = _rms(x, _w(m, "ffn_norm", l, (d,)), c["norm_eps"])
        x = x + (torch.nn.functional.silu(h @ _w(m, "w_gate", l, (F, d)).T) * (h @ _w(m, "w_up", l, (F, d)).T)) \
            @ _w(m, "w_down", l, (d, F)).T
        q_last = q
    return x, q_last


@pytest.mark.parametrize("ratio,S", [(0.0, 0), (0.15, 0), (0.4, 0), (0.15, 4)])
def test_oracle_reprocess_equals_independent_pipeline(ratio, S):
    """The whole online reprocessing path restated
    independently: records = each chunk prefilled alone at positions 1..n;
    stitch_full_reuse (K re-rotated by target - native, V copied); the
    question prefilled at T-|Q|+1..T against the stitched cache; query-guided
    scores over the chunk keys of the last layer, global top-k (k = floor(r N +
    0.5), lower index on ties); sparse prefill of crit ∪ question through every
    layer with each layer's fresh K/V replacing the stale rows before that
    layer's attention; logits of the last row. Oracle: orc_reprocess in fp32
    (emulate_bf16 off)."""
    c = CFGS["gqa"]
    L, Hkv, dh, d = c["layers"], c["n_kv_heads"], c["head_dim"], c["d_model"]
    m = O.Model(c).init_seed(21)
    rng = np.random.default_rng(int(ratio * 100) + 1)
    lens = [13, 9, 17]
    chunks = [rng.integers(0, c["vocab"], n) for n in lens]
    question = rng.integers(0, c["vocab"], 6)
    emb = _w(m, "emb", 0, (c["vocab"], d))
    # system prompt (S tokens at positions 1..S), then each chunk prefilled
    # alone after it at native positions S+1..S+n (preprocess_isolated)
    sys_tok = rng.integers(0, c["vocab"], S)
    sys_k = torch.zeros(L, S, Hkv, dh, dtype=torch.float64)
    sys_v = torch.zeros_like(sys_k)
    if S:
        _layers(m, c, emb[torch.as_tensor(sys_tok)], torch.arange(1, S + 1), sys_k, sys_v, torch.arange(1, S + 1),
                rows=torch.arange(S))
    records = []
    for ch in chunks:
        n = len(ch)
        ck = torch.cat([sys_k, torch.zeros(L, n, Hkv, dh, dtype=torch.float64)], dim=1)
        cv = torch.cat([sys_v, torch.zeros(L, n, Hkv, dh, dtype=torch.float64)], dim=1)
        _layers(m, c, emb[torch.as_tensor(ch)], torch.arange(S + 1, S + n + 1), ck, cv, torch.arange(1, S + n + 1),
                rows=torch.arange(S, S + n))
        records.append({"k": ck[:, S:].float().numpy(), "v": cv[:, S:].float().numpy(), "tokens": ch.tolist(),
                        "native_start": S + 1})
    sys_kv = (sys_k.float().numpy(), sys_v.float().numpy()) if S else None
    out = m.reprocess(sys_kv, records, question.tolist(), ratio, emulate_bf16=False)

    N, nq = sum(lens), len(question)
    T = S + N + nq
    # stitch: S rows, then the chunks from row S (records and system KV as the oracle got them: fp32)
    sk = torch.zeros(L, T, Hkv, dh, dtype=torch.float64)
    sv = torch.zeros_like(sk)
    if S:
        sk[:, :S] = torch.from_numpy(sys_kv[0]).double()
        sv[:, :S] = torch.from_numpy(sys_kv[1]).double()
    off = S
    for rec, n in zip(records, lens):
        k = torch.from_numpy(rec["k"]).double()
        for l in range(L):
            sk[l, off:off + n] = _rope(k[l], torch.full((n,), float(off + 1 - rec["native_start"])), c["rope_base"])
        sv[:, off:off + n] = torch.from_numpy(rec["v"]).double()
        off += n
    # question pass against the stitched cache (side-effect free on it)
    qpos = torch.arange(S + N + 1, T + 1)
    _, qf = _layers(m, c, emb[torch.as_tensor(question)], qpos, sk[:, :S + N].clone(), sv[:, :S + N].clone(),
                    torch.arange(1, S + N + 1))
    kvh = torch.arange(c["n_heads"]) // (c["n_heads"] // Hkv)
    keys = sk[L - 1, S:S + N][:, kvh]  # chunk keys only: never S or Q
    sc = torch.softmax(torch.einsum("thd,nhd->thn", qf, keys) / dh ** 0.5, dim=-1).sum(dim=(0, 1))
    k_sel = int(np.floor(ratio * N + 0.5))
    crit = sorted(sorted(range(N), key=lambda j: (-float(sc[j]), j))[:k_sel])
    assert out["crit"].tolist() == [S + j + 1 for j in crit]  # 1-based positions
    # sparse prefill of crit ∪ question over the stitched cache
    rows = torch.tensor([S + j for j in crit] + list(range(S + N, T)), dtype=torch.long)
    toks = torch.as_tensor(np.concatenate([sys_tok, np.concatenate(chunks), question]))[rows]
    cache_k, cache_v = sk.clone(), sv.clone()
    x, _ = _layers(m, c, emb[toks], rows + 1, cache_k, cache_v, torch.arange(1, T + 1), rows=rows)
    logits = _rms(x[-1:], _w(m, "final_norm", 0, (d,)), c["norm_eps"]) @ _w(m, "lm_head", 0, (c["vocab"], d)).T
    ref = logits[0].numpy()
    assert np.linalg.norm(out["logits"] - ref) / np.linalg.norm(ref) <= 1e-5
    rel_k = np.linalg.norm(out["k"] - cache_k.numpy()) / np.linalg.norm(cache_k.numpy())
    rel_v = np.linalg.norm(out["v"] - cache_v.numpy()) / np.linalg.norm(cache_v.numpy())
    assert rel_k <= 1e-5 and rel_v <= 1e-5, (rel_k, rel_v)


def test_oracle_kv_deviation_equals_independent_restatement():
    """kv_deviation (Eq. 7): Full Attention over cat(S,
    chunks) vs the stitched Full Reuse cache, Δ[t, l, c] = Σ_j (KV_FA −
    KV_FR)² per chunk token, layer and component (K, V), first layers."""
    c = CFGS["gqa"]
    L, Hkv, dh, d = c["layers"], c["n_kv_heads"], c["head_dim"], c["d_model"]
    m = O.Model(c).init_seed(33)
    rng = np.random.default_rng(2)
    lens = [10, 14]
    chunks = [rng.integers(0, c["vocab"], n) for n in lens]
    emb = _w(m, "emb", 0, (c["vocab"], d))
    records = []
    for ch in chunks:
        n = len(ch)
        ck = torch.zeros(L, n, Hkv, dh, dtype=torch.float64)
        cv = torch.zeros_like(ck)
        _layers(m, c, emb[torch.as_tensor(ch)], torch.arange(1, n + 1), ck, cv, torch.arange(1, n + 1),
                rows=torch.arange(n))
        records.append({"k": ck.float().numpy(), "v": cv.float().numpy(), "tokens": ch.tolist(), "native_start": 1})
    dev = m.kv_deviation(None, records, n_layers=2, emulate_bf16=False)
    N = sum(lens)
    # Full Attention KV of the concatenation
    fk = torch.zeros(L, N, Hkv, dh, dtype=torch.float64)
    fv = torch.zeros_like(fk)
    _layers(m, c, emb[torch.as_tensor(np.concatenate(chunks))], torch.arange(1, N + 1), fk, fv,
            torch.arange(1, N + 1), rows=torch.arange(N))
    # Full Reuse (stitched) KV
    rk = torch.zeros_like(fk)
    rv = torch.zeros_like(fk)
    off = 0
    for rec, n in zip(records, lens):
        k = torch.from_numpy(rec["k"]).double()
        for l in range(L):
            rk[l, off:off + n] = _rope(k[l], torch.full((n,), float(off)), c["rope_base"])
        rv[:, off:off + n] = torch.from_numpy(rec["v"]).double()
        off += n
    ref = np.stack([((fk[:2] - rk[:2]) ** 2).sum(dim=(2, 3)).T.numpy(),
                    ((fv[:2] - rv[:2]) ** 2).sum(dim=(2, 3)).T.numpy()], axis=-1)  # [N][2 layers][K, V]
    assert np.allclose(dev, ref, rtol=1e-4, atol=1e-9 * np.abs(ref).max()), np.abs(dev - ref).max()
    assert np.abs(ref[:, 0]).max() < 1e-9 * max(np.abs(ref).max(), 1.0)  # first layer: FR == FA
