"""Chunk-partitioned store on the GPU: records owned by
another store are read in place by K1 (rope_shift_assemble) and the request is
bit-identical to one served from a store holding every record.

* same process: frag_store_attach_peer (on a multi-GPU box the peer store sits
  on another device and K1 reads over NVLink; here both stores share cuda:0,
  which exercises the same fetch/pin/stitch path);
* one process per GPU: CUDA-IPC export/import between two processes (both on
  cuda:0 here; on an 8-GPU box the mapping is a peer mapping over NVSwitch).
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _setup(F, seed=5, n_chunks=8):
    eng = F.Engine("tiny", seed=1234)
    rng = np.random.default_rng(seed)
    system = rng.integers(0, eng.cfg.vocab, 8).tolist()
    chunks = [rng.integers(0, eng.cfg.vocab, 256).tolist() for _ in range(n_chunks)]
    question = rng.integers(0, eng.cfg.vocab, 32).tolist()
    return eng, system, chunks, question


def _run(F, eng, store, system, ids, question, ratio=0.15):
    res = F.Result(eng, 8 + len(ids) * 256 + 32)
    eng.reprocess(store, question, ids, ratio, res, system=system)
    k, v = res.fused_kv()
    return res.logits().copy(), k, v, res.crit().copy()


def test_attach_peer_same_process(cuda):
    from paper_2601_12904_b200 import fusion as F
    eng, system, chunks, question = _setup(F)
    full = F.ChunkKVStore(eng.cfg)
    ids = [eng.preprocess_isolated(full, c, system=system) for c in chunks]
    # split the corpus: even chunks in `a` (the remote owner), odd ones in `b`
    a, b = F.ChunkKVStore(eng.cfg), F.ChunkKVStore(eng.cfg)
    for i, c in enumerate(chunks):
        eng.preprocess_isolated(a if i % 2 == 0 else b, c, system=system)
    with pytest.raises(F.StoreError):
        b.fetch(ids[0])  # not attached yet
    b.attach_peer(a)
    b.attach_peer(a)  # idempotent
    with pytest.raises(F.ContractError):
        b.attach_peer(b)
    assert len(b) == 4 and b.bytes_used == full.bytes_used // 2
    h0 = a.peek(ids[0]).heat
    for ratio in (0.0, 0.15, 1.0):
        ref = _run(F, eng, full, system, ids, question, ratio)
        got = _run(F, eng, b, system, ids, question, ratio)
        for x, y in zip(ref, got):
            assert np.array_equal(x, y)
    assert a.peek(ids[0]).heat == h0 + 3  # the owning store keeps heat
    assert b.peek(ids[0]).tier == F.TIER_GPU  # a's own HBM record, seen through b
    assert np.array_equal(b.read_kv(ids[2])[0], full.read_kv(ids[2])[0])
    # the owner's records were only read
    for i in ids[::2]:
        assert np.array_equal(a.read_kv(i)[1], full.read_kv(i)[1])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2601_12904_b200 import fusion as F
        from paper_2601_12904_b200 import partition as P
        eng, system, chunks, question = _setup(F)
        qrng = np.random.default_rng(100 + rank)
        question = qrng.integers(0, eng.cfg.vocab, 32).tolist()
        ids = [F.hash_tokens(c) for c in chunks]
        own = P.owners(ids, world)
        st = F.ChunkKVStore(eng.cfg)
        owned = {}
        for cid, c, o in zip(ids, chunks, own):
            if o == rank:
                assert eng.preprocess_isolated(st, c, system=system) == cid
                owned[cid] = c
        where = P.share_records(st, owned)
        info = {"n": len(st), "owned": len(owned), "where": len(where)}
        tiers = [st.peek(i).tier for i in ids]
        info["tiers_ok"] = all((t == F.TIER_GPU) == (o == rank) for t, o in zip(tiers, own))
        info["peer_tier"] = [t for t, o in zip(tiers, own) if o != rank][:1]
        # replicated reference: every record local
        full = F.ChunkKVStore(eng.cfg)
        for c in chunks:
            eng.preprocess_isolated(full, c, system=system)
        info["bytes_ok"] = st.bytes_used == full.bytes_used * len(owned) // len(chunks)
        res = {}
        for ratio in (0.15, 1.0):
            ref = _run(F, eng, full, system, ids, question, ratio)
            got = _run(F, eng, st, system, ids, question, ratio)
            res[ratio] = all(np.array_equal(x, y) for x, y in zip(ref, got))
        info["equal"] = res
        # an exported record is never replaced under its importers
        mine = next(iter(owned))
        try:
            eng.preprocess_isolated(st, owned[mine], system=system, overwrite=True)
            info["overwrite_exported"] = "allowed"
        except F.StoreError:
            info["overwrite_exported"] = "StoreError"
        # importing this process's own export is a contract error (attach_peer instead)
        try:
            st.import_record(st.export_record(mine), owned[mine], overwrite=True)
            info["self_import"] = "allowed"
        except F.ContractError:
            info["self_import"] = "ContractError"
        out[rank] = info
        dist.barrier()
        full.close()
        st.close()  # importers close their mappings before any owner frees its pages
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_ipc_partitioned_store_two_processes(cuda):
    import torch.multiprocessing as mp
    from paper_2601_12904_b200 import fusion as F
    from paper_2601_12904_b200 import partition as P
    eng, system, chunks, _ = _setup(F)
    own = P.owners([F.hash_tokens(c) for c in chunks], 2)
    assert 0 < sum(own) < len(own)
    del eng
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_ipc_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    for r in range(2):
        info = out[r]
        assert info["n"] == 8 and info["where"] == 8
        assert info["owned"] == sum(1 for o in own if o == r)
        assert info["tiers_ok"] and info["peer_tier"] == [F.TIER_PEER]
        assert info["bytes_ok"]  # peer views take no local HBM
        assert info["equal"] == {0.15: True, 1.0: True}
        assert info["overwrite_exported"] == "StoreError"
        assert info["self_import"] == "ContractError"
