"""Chunk-partitioned KV store across the GPUs of one box.

Each chunk's record is preprocessed into, and owned by, exactly one GPU's
store: owner = frag_chunk_owner(chunk_id, world) (the spec's single-copy
invariant, held across GPUs). One process per GPU: every owner
exports its records as 128-byte CUDA-IPC descriptors (frag_store_export), the
descriptors and the chunks' token ids travel once through
torch.distributed.all_gather_object (setup, not the data path), and every other
rank imports them as FRAG_TIER_PEER views (frag_store_import). At request time
K1 (rope_shift_assemble) reads a peer record's pages in place over
NVLink 5 / NVSwitch into the local fused cache, so fetch and re-positioning
are one pass; no collective runs per request.

The store objects are duck-typed here (export_record / import_record) so the
exchange logic is testable on CPU with gloo (tests/test_partition_cpu.py).
"""
from __future__ import annotations

from typing import Callable, Mapping, Sequence


def owners(chunk_ids: Sequence, world: int, owner_fn: Callable | None = None) -> list[int]:
    """Owning rank of every chunk id."""
    if owner_fn is None:
        from .fusion import chunk_owner as owner_fn
    return [int(owner_fn(cid, world)) for cid in chunk_ids]


def share_records(store, owned: Mapping, *, group=None) -> dict:
    """Export this rank's records, all-gather the descriptors, import the
    other ranks' records into `store`.

    owned: {chunk_id: token ids} of the records this rank holds (and owns).
    Returns {chunk_id: owner rank} over the whole world. A chunk id owned by
    two ranks violates the single-copy invariant and raises.
    """
    import torch.distributed as dist

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    mine = [(bytes(cid.bytes), store.export_record(cid), [int(t) for t in toks]) for cid, toks in owned.items()]
    gathered: list = [None] * world
    dist.all_gather_object(gathered, mine, group=group)
    where: dict = {}
    for r, entries in enumerate(gathered):
        for key, blob, toks in entries:
            if key in where:
                raise RuntimeError(f"chunk {key.hex()} is owned by ranks {where[key]} and {r} (single-copy invariant)")
            where[key] = r
            if r != rank:
                store.import_record(blob, toks)
    return where
