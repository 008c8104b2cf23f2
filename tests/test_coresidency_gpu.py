"""Co-residency of the persistent kernels (split-K fixups, stream-K owners,
the per-layer GEMM chain), SPEC.md:181 ("kernel calls are pure per call") and
SPEC.md:458 (concurrent requests).

* Two engines on one device driven from concurrent host threads: the device
  work of every engine is serialised per device, process wide (engine.h
  device_mutex), so neither grid can hold SMs another grid spins on; every
  request equals its serial result bit for bit and nothing hangs.
* A grid that does not get all its CTAs (simulated by a wait limit far below
  any real wait) abandons its inter-CTA waits, the call returns FRAG_E_CUDA
  (CudaError) instead of hanging, and the next call on the same engine and
  result -- counters re-armed -- is bit-identical to the undisturbed run.
"""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _request_set(F, eng, store, n, seed):
    rng = np.random.default_rng(seed)
    c = eng.cfg
    chunks = [rng.integers(0, c.vocab, 256).tolist() for _ in range(4)]
    ids = [eng.preprocess_isolated(store, ch) for ch in chunks]
    qs = [rng.integers(0, c.vocab, 32).tolist() for _ in range(n)]
    return ids, qs


def test_two_engines_concurrent_threads(cuda):
    from paper_2601_12904_b200 import fusion as F
    engines = [F.Engine("tiny", seed=s) for s in (5, 6)]
    stores = [F.ChunkKVStore(e.cfg) for e in engines]
    work = [_request_set(F, e, st, 6, 40 + i) for i, (e, st) in enumerate(zip(engines, stores))]
    T = 4 * 256 + 32
    serial = []
    for e, st, (ids, qs) in zip(engines, stores, work):
        res = F.Result(e, T)
        out = []
        for q in qs:
            e.reprocess(st, q, ids, 0.15, res)
            out.append((res.logits()[0].copy(), res.crit().copy()))
        serial.append(out)
        res.close()
    got = [[None] * 6 for _ in engines]
    errs = []

    def worker(i, rounds):
        try:
            e, st, (ids, qs) = engines[i], stores[i], work[i]
            res = F.Result(e, T)
            for _ in range(rounds):
                for j, q in enumerate(qs):
                    e.reprocess(st, q, ids, 0.15, res)
                    got[i][j] = (res.logits()[0].copy(), res.crit().copy())
            res.close()
        except Exception as ex:  # surfaced below
            errs.append(ex)

    threads = [threading.Thread(target=worker, args=(i, 3)) for i in range(2) for _ in range(2)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in threads), "concurrent requests hung"
    assert not errs, errs
    for i in range(2):
        for j in range(6):
            assert np.array_equal(got[i][j][0], serial[i][j][0]) and np.array_equal(got[i][j][1], serial[i][j][1])


def test_abandoned_wait_reports_error_and_recovers(cuda):
    from paper_2601_12904_b200 import _lib as L
    from paper_2601_12904_b200 import fusion as F
    cfg = F.preset("llama3-8b")
    cfg.layers = 2
    eng = F.Engine(cfg, seed=3)
    store = F.ChunkKVStore(cfg)
    ids, qs = _request_set(F, eng, store, 1, 9)
    res = F.Result(eng, 4 * 256 + 32)
    eng.reprocess(store, qs[0], ids, 0.15, res)
    want_logits, want_k = res.logits()[0].copy(), res.fused_kv()[0].copy()
    prev = L.lib.frag_set_spin_limit_ms(1e-6)  # 1 ns: every wait that does not succeed at once is abandoned
    try:
        raised = None
        for _ in range(3):
            try:
                eng.reprocess(store, qs[0], ids, 0.15, res)
            except F.CudaError as ex:
                raised = ex
                break
        assert raised is not None and "co-resident" in str(raised)
    finally:
        L.lib.frag_set_spin_limit_ms(prev)
    for _ in range(2):  # the same engine and result work again, bit-identically
        eng.reprocess(store, qs[0], ids, 0.15, res)
        assert np.array_equal(res.logits()[0], want_logits)
        assert np.array_equal(res.fused_kv()[0], want_k)
    res.close()
    store.close()
    eng.close()
