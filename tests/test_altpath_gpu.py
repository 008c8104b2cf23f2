"""alternative_path_match through the C ABI against the
oracle restatement (oracle.alt_path_match) on random contexts: the store's
prefix index (PrefixKey = rolling hash over (system id, chunk ids),
SPEC.md:259-261) registered by preprocess_isolated / preprocess_fused and
register_prefix."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_store_match_equals_oracle(cuda):
    from oracle import oracle as O
    from paper_2601_12904_b200 import fusion as F
    eng = F.Engine("tiny", seed=1234)
    store = F.ChunkKVStore(eng.cfg)
    rng = np.random.default_rng(9)
    system = rng.integers(0, eng.cfg.vocab, 8).tolist()
    chunks = [rng.integers(0, eng.cfg.vocab, 64).tolist() for _ in range(6)]
    ids = [eng.preprocess_isolated(store, c, system=system) for c in chunks]  # cached under (S, [c])
    key = lambda cid: bytes(cid.bytes)  # noqa: E731
    sid = "S"
    cached = {(sid, (key(i),)) for i in ids}
    records = {key(i) for i in ids}
    # a FUSED record of a new chunk under (S, [ids[0], ids[1]]) (Eq. 10) -> path (c0, c1, x)
    x = rng.integers(0, eng.cfg.vocab, 64).tolist()
    xid = eng.preprocess_fused(store, x, [ids[0], ids[1]], system=system)
    cached.add((sid, (key(ids[0]), key(ids[1]), key(xid))))
    records.add(key(xid))
    # paths registered by hand (a query that cached c3 after c2, c5 after c4 c1)
    for p in ([ids[2], ids[3]], [ids[4], ids[1], ids[5]]):
        store.register_prefix(p, system=system)
        cached.add((sid, tuple(key(i) for i in p)))
    unknown = [F.hash_tokens([7, 7, i]) for i in range(3)]
    pool = ids + [xid] + unknown
    for t in range(200):
        n = int(rng.integers(1, 7))
        ctx = [pool[j] for j in rng.choice(len(pool), n, replace=False)]
        got = [(key(c), via, pos, start) for c, via, pos, start in store.match(ctx, system=system)]
        ref = O.alt_path_match(cached, records, [key(c) for c in ctx], sid)
        assert got == ref, (t, got, ref)
    # paper's Query3 shape and the other system prompt: nothing registered under it
    got = store.match([ids[2], ids[3]], system=system)
    assert [g[1] for g in got] == ["PREFIX", "PREFIX"]
    got = store.match([ids[1], ids[0]], system=[1, 2, 3])
    assert [g[1] for g in got] == ["ALT_PATH", "ALT_PATH"]  # records exist; completeness
    with pytest.raises(F.ContractError):
        store.match([], system=system)
