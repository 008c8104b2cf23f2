"""Chunk-partitioned store host logic on CPU (gloo, world_size 2; SURVEY.md
§8(e)): the owner function (frag_chunk_owner, pure host code in libfrag.so),
and paper_2601_12904_b200.partition.share_records — every rank exports the
records it owns, all-gathers the 128-byte descriptors once at setup, and
imports exactly the records the other ranks own (single copy per chunk id
across GPUs). The stores are fakes with the ChunkKVStore
export/import surface; the GPU side (CUDA IPC, NVLink reads inside K1) is
tests/test_partition_gpu.py."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2601_12904_b200 import fusion as F
from paper_2601_12904_b200 import partition as P


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class FakeStore:
    def __init__(self, rank):
        self.rank = rank
        self.exported, self.imported = [], []

    def export_record(self, cid):
        self.exported.append(bytes(cid.bytes))
        return bytes([self.rank]) * 128

    def import_record(self, blob, toks):
        assert len(blob) == 128
        self.imported.append((blob[0], tuple(toks)))


def _chunks(n=12):
    rng = np.random.default_rng(5)
    return [rng.integers(0, 1000, 16).tolist() for _ in range(n)]


def _worker(rank, world, port, out, dup):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        chunks = _chunks()
        ids = [F.hash_tokens(c) for c in chunks]
        own = P.owners(ids, world)
        owned = {cid: c for cid, c, o in zip(ids, chunks, own) if o == rank}
        if dup and rank == 1:  # rank 1 also claims one of rank 0's chunks
            j = own.index(0)
            owned[ids[j]] = chunks[j]
        st = FakeStore(rank)
        try:
            where = P.share_records(st, owned)
            out[rank] = ("ok", st.exported, st.imported, {k.hex(): v for k, v in where.items()})
        except RuntimeError as ex:
            out[rank] = ("err", str(ex))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_chunk_owner_matches_restatement():
    for i in range(200):
        cid = F.hash_tokens([i, i + 1])
        for n in (1, 2, 3, 8):
            assert F.chunk_owner(cid, n) == int.from_bytes(bytes(cid.bytes[:8]), "little") % n
    with pytest.raises(F.ContractError):
        F.chunk_owner(F.hash_tokens([1]), 0)
    # content hashes spread uniformly over 8 owners
    counts = np.bincount([F.chunk_owner(F.hash_tokens([i]), 8) for i in range(4000)], minlength=8)
    assert counts.min() > 400


def test_share_records_gloo():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out, False), nprocs=world, join=True)
    chunks = _chunks()
    ids = [F.hash_tokens(c) for c in chunks]
    own = P.owners(ids, world)
    assert 0 < sum(own) < len(own)  # both ranks own something
    for r in range(world):
        status, exported, imported, where = out[r]
        assert status == "ok"
        assert sorted(exported) == sorted(bytes(i.bytes) for i, o in zip(ids, own) if o == r)
        # imports: exactly the other rank's records, tagged with the owner's blob
        assert sorted(imported) == sorted((1 - r, tuple(c)) for c, o in zip(chunks, own) if o != r)
        assert where == {i.hex(): o for i, o in zip(ids, own)}


def test_share_records_rejects_two_owners():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out, True), nprocs=world, join=True)
    for r in range(world):
        assert out[r][0] == "err" and "single-copy" in out[r][1]
