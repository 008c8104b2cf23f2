"""Kernel-level parity on the B200: each sm_100a kernel against a plain fp32
(or fp64) PyTorch restatement of the same op, called through the C ABI."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _lib():
    from paper_2601_12904_b200 import _lib
    return _lib


def _gemm(a, b, c, epi, force_bn=0):
    L = _lib()
    L.check(L.lib.frag_kernel_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), a.shape[0], b.shape[0], a.shape[1],
                                   epi, force_bn, None))


@pytest.mark.parametrize("M,N,K", [(1, 256, 64), (37, 512, 256), (128, 768, 256), (300, 1024, 512),
                                   (2490, 1536, 4096), (129, 64, 192), (32, 4096, 14336), (1, 4096, 14336)])
@pytest.mark.parametrize("bn", [0, 64, 128, 256])
def test_gemm_tcgen05_vs_torch(cuda, M, N, K, bn):
    """1-CTA tcgen05 GEMM; K = 14336 at <= 128 rows is the question pass's down
    projection: split-K over strided k-blocks (gemm_tc.cu k_strided_for)."""
    import torch
    if bn and N % bn:
        pytest.skip("N not a multiple of BN")
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    a = torch.randn(M, K, device=cuda, generator=g).to(torch.bfloat16)
    b = torch.randn(N, K, device=cuda, generator=g).to(torch.bfloat16)
    ref = a.double() @ b.double().T
    c = torch.empty(M, N, device=cuda, dtype=torch.float32)
    _gemm(a, b, c, 1, bn)
    torch.cuda.synchronize()
    err = (c.double() - ref).abs().max().item()
    assert err <= 2e-5 * math.sqrt(K) * ref.abs().max().item() + 1e-4, err
    cb = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
    _gemm(a, b, cb, 0, bn)
    torch.cuda.synchronize()
    assert torch.equal(cb, c.to(torch.bfloat16))
    # residual epilogue: C += A B^T
    r0 = torch.randn(M, N, device=cuda, generator=g)
    r = r0.clone()
    _gemm(a, b, r, 2, bn)
    torch.cuda.synchronize()
    assert torch.allclose(r, r0 + c, rtol=0, atol=1e-4 * ref.abs().max().item() + 1e-5)


def test_gemm_swiglu_epilogue(cuda):
    import torch
    M, F, K = 200, 512, 256
    g = torch.Generator(device="cuda").manual_seed(3)
    a = torch.randn(M, K, device=cuda, generator=g).to(torch.bfloat16) * 0.5
    wg = torch.randn(F, K, device=cuda, generator=g).to(torch.bfloat16) * 0.1
    wu = torch.randn(F, K, device=cuda, generator=g).to(torch.bfloat16) * 0.1
    packed = torch.empty(2 * F, K, device=cuda, dtype=torch.bfloat16)
    idx = torch.arange(F, device=cuda)
    packed[(idx // 32) * 64 + idx % 32] = wg
    packed[(idx // 32) * 64 + 32 + idx % 32] = wu
    out = torch.empty(M, F, device=cuda, dtype=torch.bfloat16)
    _gemm(a, packed, out, 3)
    torch.cuda.synchronize()
    gg = a.float() @ wg.float().T
    uu = a.float() @ wu.float().T
    ref = torch.nn.functional.silu(gg) * uu
    assert (out.float() - ref).abs().max().item() <= 1e-2 * ref.abs().max().item()


def _attn_ref(q, k, v, rows, scale):
    # q [M,Hq,dh], k/v [T,Hkv,dh]; row i sees keys 0..rows[i]
    import torch
    M, Hq, dh = q.shape
    G = Hq // k.shape[1]
    out = torch.empty(M, Hq, dh, dtype=torch.float64, device=q.device)
    kk = k.double().repeat_interleave(G, dim=1)
    vv = v.double().repeat_interleave(G, dim=1)
    for i in range(M):
        p = int(rows[i]) + 1
        s = torch.einsum("hd,thd->ht", q[i].double(), kk[:p]) * scale
        w = torch.softmax(s, dim=-1)
        out[i] = torch.einsum("ht,thd->hd", w, vv[:p])
    return out


@pytest.mark.parametrize("Hq,Hkv,dh,T,M,split", [(4, 4, 64, 700, 90, 0), (32, 8, 128, 1500, 150, 0),
                                                 (32, 8, 128, 3000, 20, 512), (8, 1, 128, 600, 64, 256)])
def test_sparse_q_attention_vs_torch(cuda, Hq, Hkv, dh, T, M, split):
    import torch
    g = torch.Generator(device="cuda").manual_seed(T + M)
    q = torch.randn(M, Hq, dh, device=cuda, generator=g).to(torch.bfloat16)
    k = torch.randn(T, Hkv, dh, device=cuda, generator=g).to(torch.bfloat16)
    v = torch.randn(T, Hkv, dh, device=cuda, generator=g).to(torch.bfloat16)
    rows = torch.sort(torch.randperm(T, device=cuda, generator=g)[:M]).values.to(torch.int32)
    out = torch.empty(M, Hq, dh, device=cuda, dtype=torch.bfloat16)
    L = _lib()
    L.check(L.lib.frag_kernel_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), rows.data_ptr(), out.data_ptr(),
                                        M, T, Hq, Hkv, dh, split, None))
    ref = _attn_ref(q, k, v, rows.cpu(), 1.0 / math.sqrt(dh))
    err = (out.double() - ref).abs().max().item()
    assert err < 2e-2, err


def test_attention_one_thread_per_row_variant(cuda):
    """The dh=128 kernel defaults to two softmax threads per query row; the
    one-thread-per-row kernel (FRAG_ATTN_SPLIT=0, read once per process) must
    stay correct too."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, FRAG_ATTN_SPLIT="0")
    p = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        "tests/test_kernels_gpu.py", "-k", "sparse_q_attention_vs_torch"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]
    assert "4 passed" in p.stdout, p.stdout[-500:]


def _rope_shift_ref(kbits, delta, base):
    dh = kbits.shape[-1]
    k = (kbits.astype(np.uint32) << 16).view(np.float32)
    half = dh // 2
    th = base ** (-2.0 * (np.arange(half) + 1) / dh)
    c = np.cos(delta * th).astype(np.float32)
    s = np.sin(delta * th).astype(np.float32)
    k0, k1 = k[..., 0::2], k[..., 1::2]
    o0 = (k0.astype(np.float64) * c - np.float32(k1 * s)).astype(np.float32)  # fma(k0,c,-(k1*s)) exactly rounded
    o1 = (k1.astype(np.float64) * c + np.float32(k0 * s)).astype(np.float32)
    out = np.empty_like(k)
    out[..., 0::2], out[..., 1::2] = o0, o1
    b = out.view(np.uint32)
    rnd = ((b >> 16) & 1) + 0x7FFF
    return ((b + rnd) >> 16).astype(np.uint16)


@pytest.mark.parametrize("delta", [0, 1, 257, 5000, -3])
def test_rope_shift_bit_exact(cuda, delta):
    import torch
    L_, n, Hkv, dh = 2, 70, 4, 64
    rng = np.random.default_rng(delta + 11)
    kf = rng.standard_normal((L_, n, Hkv, dh)).astype(np.float32)
    kbits = (kf.view(np.uint32) >> 16).astype(np.uint16)
    src = torch.from_numpy(kbits.view(np.int16)).to(cuda)
    dst = torch.empty_like(src)
    native = 10
    L = _lib()
    L.check(L.lib.frag_kernel_rope_shift(src.data_ptr(), dst.data_ptr(), L_, n, Hkv, dh, native, native + delta,
                                         1e4, None))
    got = dst.cpu().numpy().view(np.uint16)
    exp = kbits if delta == 0 else _rope_shift_ref(kbits, float(delta), 1e4)
    assert np.array_equal(got, exp)


@pytest.mark.parametrize("M,N,K", [(256, 256, 64), (300, 512, 256), (2490, 1024, 4096), (1000, 768, 512),
                                   (2490, 4096, 4096), (1000, 6144, 512)])
@pytest.mark.parametrize("bn", [128, 192, 224, 256])
@pytest.mark.parametrize("tail", [0, 1])
def test_gemm_cta_pair_vs_torch(cuda, M, N, K, bn, tail):
    """cta_group::2 GEMM (256-row tiles shared by a CTA pair); tail=1 splits the
    last partial wave of pairs along K (deterministic cooperative reduction);
    BN=192 / 224 leave a partial last N tile when N % BN != 0."""
    import torch
    if bn not in (192, 224) and N % bn:
        pytest.skip("N not a multiple of BN")
    g = torch.Generator(device="cuda").manual_seed(M + N + K + bn)
    a = torch.randn(M, K, device=cuda, generator=g).to(torch.bfloat16)
    b = torch.randn(N, K, device=cuda, generator=g).to(torch.bfloat16)
    ref = a.double() @ b.double().T
    c = torch.empty(M, N, device=cuda, dtype=torch.float32)
    flags = bn | 0x40000 | (0x10000 if tail else 0)
    _gemm(a, b, c, 1, flags)
    torch.cuda.synchronize()
    err = (c.double() - ref).abs().max().item()
    assert err <= 2e-5 * math.sqrt(K) * ref.abs().max().item() + 1e-4, err
    c2 = torch.empty_like(c)
    _gemm(a, b, c2, 1, flags)
    torch.cuda.synchronize()
    assert torch.equal(c, c2)  # deterministic (split reduction in split order)
    r0 = torch.randn(M, N, device=cuda, generator=g)
    r = r0.clone()
    _gemm(a, b, r, 2, flags)
    torch.cuda.synchronize()
    assert torch.allclose(r, r0 + c, rtol=0, atol=1e-4 * ref.abs().max().item() + 1e-5)


@pytest.mark.parametrize("M,N,K", [(32, 6144, 4096), (1, 4096, 14336), (100, 1280, 512), (128, 512, 256),
                                   (32, 28672, 4096)])
@pytest.mark.parametrize("bn", [64, 128])
def test_gemm_stream_k_vs_torch(cuda, M, N, K, bn):
    """Stream-K decomposition of the one-M-tile (question pass) GEMM: tiles
    shared by several CTAs finished by their owner in CTA order."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(M + N + K + bn)
    a = torch.randn(M, K, device=cuda, generator=g).to(torch.bfloat16)
    b = torch.randn(N, K, device=cuda, generator=g).to(torch.bfloat16)
    ref = a.double() @ b.double().T
    flags = bn | 0x2000000
    c = torch.empty(M, N, device=cuda, dtype=torch.float32)
    _gemm(a, b, c, 1, flags)
    torch.cuda.synchronize()
    err = (c.double() - ref).abs().max().item()
    assert err <= 2e-5 * math.sqrt(K) * ref.abs().max().item() + 1e-4, err
    c2 = torch.empty_like(c)
    _gemm(a, b, c2, 1, flags)
    torch.cuda.synchronize()
    assert torch.equal(c, c2)
    r0 = torch.randn(M, N, device=cuda, generator=g)
    r = r0.clone()
    _gemm(a, b, r, 2, flags)
    torch.cuda.synchronize()
    assert torch.equal(r, r0 + c)
    F = N // 2
    out = torch.empty(M, F, device=cuda, dtype=torch.bfloat16)
    _gemm(a, b, out, 3, flags)
    torch.cuda.synchronize()
    idx = torch.arange(F, device=cuda)
    gg = c[:, (idx // 32) * 64 + idx % 32]
    uu = c[:, (idx // 32) * 64 + 32 + idx % 32]
    want = torch.nn.functional.silu(gg) * uu
    assert (out.float() - want).abs().max().item() <= 1e-2 * want.abs().max().item() + 1e-3


@pytest.mark.parametrize("bn", [192, 256])
def test_gemm_pair_swiglu_partial_tile(cuda, bn):
    import torch
    M, F, K = 600, 1280, 512   # 2F = 2560 = 13.3 tiles of 192
    g = torch.Generator(device="cuda").manual_seed(bn)
    a = torch.randn(M, K, device=cuda, generator=g).to(torch.bfloat16) * 0.5
    wg = torch.randn(F, K, device=cuda, generator=g).to(torch.bfloat16) * 0.1
    wu = torch.randn(F, K, device=cuda, generator=g).to(torch.bfloat16) * 0.1
    packed = torch.empty(2 * F, K, device=cuda, dtype=torch.bfloat16)
    idx = torch.arange(F, device=cuda)
    packed[(idx // 32) * 64 + idx % 32] = wg
    packed[(idx // 32) * 64 + 32 + idx % 32] = wu
    out = torch.empty(M, F, device=cuda, dtype=torch.bfloat16)
    _gemm(a, packed, out, 3, bn | 0x40000)
    torch.cuda.synchronize()
    ref = torch.nn.functional.silu(a.float() @ wg.float().T) * (a.float() @ wu.float().T)
    assert (out.float() - ref).abs().max().item() <= 1e-2 * ref.abs().max().item()


@pytest.mark.parametrize("nq,Hq,Hkv,dh,N,raw", [(32, 32, 8, 128, 16384, 0), (64, 32, 8, 128, 3000, 0),
                                               (5, 4, 2, 64, 1000, 0), (32, 32, 8, 128, 2050, 1),
                                               (1, 8, 8, 128, 129, 0), (2, 8, 2, 64, 60000, 0)])
def test_qg_score_tcgen05_vs_fp64(cuda, nq, Hq, Hkv, dh, N, raw):
    """K9 on the tensor cores (3-term bf16 split of the fp32 queries) against
    the fp64 materialise + column-sum oracle; K10 against the
    stable sort up to an epsilon window at the k-th score."""
    import torch
    from oracle import oracle as O
    g = torch.Generator(device="cuda").manual_seed(N + nq)
    q = (torch.randn(nq, Hq, dh, device=cuda, generator=g) * 2.0).float()
    k = torch.randn(N, Hkv, dh, device=cuda, generator=g).to(torch.bfloat16)
    k_sel = int(0.15 * N + 0.5)
    scores = torch.empty(N, device=cuda, dtype=torch.float32)
    sel = torch.empty(max(k_sel, 1), device=cuda, dtype=torch.int32)
    L = _lib()
    L.check(L.lib.frag_kernel_qg_select(q.data_ptr(), k.data_ptr(), nq, Hq, Hkv, dh, N, k_sel, raw,
                                        scores.data_ptr(), sel.data_ptr(), None))
    ref, ref_sel = O.select(q.cpu().numpy(), k.float().cpu().numpy(), k_sel, raw=bool(raw))
    got = scores.cpu().numpy().astype(np.float64)
    tol = 1e-4 * np.abs(ref).max() if raw else 0.0
    assert np.allclose(got, ref, rtol=1e-4, atol=max(tol, 1e-7)), np.abs(got - ref).max()
    gs = sel[:k_sel].cpu().numpy()
    tau = np.sort(ref)[::-1][k_sel - 1]
    eps = 1e-4 * np.abs(ref).mean()
    diff = set(gs.tolist()) ^ set(ref_sel.tolist())
    assert all(abs(ref[j] - tau) <= eps for j in diff)
    # bit-deterministic (no atomics)
    s2 = torch.empty_like(scores)
    L.check(L.lib.frag_kernel_qg_select(q.data_ptr(), k.data_ptr(), nq, Hq, Hkv, dh, N, k_sel, raw,
                                        s2.data_ptr(), sel.data_ptr(), None))
    assert torch.equal(scores, s2)


@pytest.mark.parametrize("N,k", [(16384, 2458), (3000, 3000), (1000, 0), (777, 1), (60000, 9000)])
def test_topk_ties_go_to_lower_index(cuda, N, k):
    """All scores tie (zero queries -> uniform softmax): the k lowest chunk
    indices are selected."""
    import torch
    q = torch.zeros(4, 8, 64, device=cuda, dtype=torch.float32)
    kk = torch.randn(N, 2, 64, device=cuda).to(torch.bfloat16)
    scores = torch.empty(N, device=cuda, dtype=torch.float32)
    sel = torch.full((max(k, 1),), -1, device=cuda, dtype=torch.int32)
    L = _lib()
    L.check(L.lib.frag_kernel_qg_select(q.data_ptr(), kk.data_ptr(), 4, 8, 2, 64, N, k, 0, scores.data_ptr(),
                                        sel.data_ptr(), None))
    assert torch.all(scores == scores[0])
    assert sel[:k].cpu().tolist() == list(range(k))


@pytest.mark.slow
@pytest.mark.parametrize("T,M,split", [(16416, 2490, 0), (16416, 32, 1024), (32800, 4947, 0)])
def test_sparse_q_attention_headline_shapes(cuda, T, M, split):
    """K6 at the bench's shapes: the sparse pass (2490 rows x 16416 keys, 8B;
    4947 x 32800, Mistral-7B) with the longest-first two-tile dispatch, and the
    question pass (32 rows, split-KV 1024 keys = the engine's split policy for
    16416 keys on 148 SMs) with its LSE combine. The last rows and 64 sampled
    rows are checked against fp64 (|err| < 2e-2 on unit-normal inputs)."""
    import torch
    Hq, Hkv, dh = 32, 8, 128
    g = torch.Generator(device="cuda").manual_seed(T + M)
    q = torch.randn(M, Hq, dh, device=cuda, generator=g).to(torch.bfloat16)
    k = torch.randn(T, Hkv, dh, device=cuda, generator=g).to(torch.bfloat16)
    v = torch.randn(T, Hkv, dh, device=cuda, generator=g).to(torch.bfloat16)
    if M == 32:
        rows = torch.arange(T - M, T, device=cuda, dtype=torch.int32)
    else:
        sel = torch.sort(torch.randperm(T - 32, device=cuda, generator=g)[:M - 32]).values
        rows = torch.cat([sel, torch.arange(T - 32, T, device=cuda)]).to(torch.int32)
    out = torch.empty(M, Hq, dh, device=cuda, dtype=torch.bfloat16)
    L = _lib()
    L.check(L.lib.frag_kernel_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), rows.data_ptr(), out.data_ptr(),
                                        M, T, Hq, Hkv, dh, split, None))
    torch.cuda.synchronize()
    pick = torch.unique(torch.cat([torch.randperm(M, device=cuda, generator=g)[:64],
                                   torch.arange(max(0, M - 4), M, device=cuda), torch.zeros(1, device=cuda).long()]))
    ref = _attn_ref(q[pick], k, v, rows[pick].cpu(), 1.0 / math.sqrt(dh))
    err = (out[pick].double() - ref).abs().max().item()
    assert err < 2e-2, err


@pytest.mark.slow
@pytest.mark.parametrize("N,K,epi", [(4096, 14336, 2), (6144, 4096, 1), (28672, 4096, 3), (4096, 4096, 2)])
def test_gemm_headline_shapes(cuda, N, K, epi):
    """The sparse pass's GEMMs at M = 2490 rows (8B, r = 0.15) through the
    engine's own dispatch policy (CTA-pair tiles, the tail split along K for
    the down projection K = 14336): QKV (N = 6144), O (4096 x 4096, residual),
    gate/up (SwiGLU over the 32-row interleave), down (residual)."""
    import torch
    M = 2490
    g = torch.Generator(device="cuda").manual_seed(N + K)
    a = (torch.randn(M, K, device=cuda, generator=g) * 0.5).to(torch.bfloat16)
    b = (torch.randn(N, K, device=cuda, generator=g) * 0.02).to(torch.bfloat16)
    ref = a.double() @ b.double().T
    if epi == 1:
        c = torch.empty(M, N, device=cuda, dtype=torch.float32)
        _gemm(a, b, c, 1)
        torch.cuda.synchronize()
        err = (c.double() - ref).abs().max().item()
        assert err <= 2e-5 * math.sqrt(K) * ref.abs().max().item() + 1e-4, err
    elif epi == 2:
        r0 = torch.randn(M, N, device=cuda, generator=g)
        r = r0.clone()
        _gemm(a, b, r, 2)
        torch.cuda.synchronize()
        err = (r.double() - r0.double() - ref).abs().max().item()
        assert err <= 2e-5 * math.sqrt(K) * ref.abs().max().item() + 1e-4, err
        r2 = r0.clone()
        _gemm(a, b, r2, 2)
        torch.cuda.synchronize()
        assert torch.equal(r, r2)  # deterministic split-K reduction
    else:
        F = N // 2
        out = torch.empty(M, F, device=cuda, dtype=torch.bfloat16)
        _gemm(a, b, out, 3)
        torch.cuda.synchronize()
        idx = torch.arange(F, device=cuda)
        gg = ref[:, (idx // 32) * 64 + idx % 32]
        uu = ref[:, (idx // 32) * 64 + 32 + idx % 32]
        want = torch.nn.functional.silu(gg) * uu
        assert (out.double() - want).abs().max().item() <= 1e-2 * want.abs().max().item() + 1e-3
