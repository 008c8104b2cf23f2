"""Python mirror of the reference's reprocessing surface over the C ABI.

Names follow SPEC.md: ``ChunkKVStore.put_record`` / ``fetch`` (SPEC.md:265,
SPEC.md:283), ``preprocess_isolated``, ``reprocess`` =
``stitch_full_reuse`` + ``select_query_guided`` + ``sparse_prefill_and_decode``
up to the first-token logits. Errors are the reference's
taxonomy (common.hpp:17-40): ``ContractError``, ``StoreError``, ``FormatError``.

Every call goes to libfrag.so (CUDA, sm_100a). There is no CPU path here.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np

from ._lib import (ChunkId, FkvcHeader, ContractError, CudaError, FormatError, FragError, Match, ModelCfg,
                   OutOfMemory, PeerRecord, Request, RecordView, ReprocessOpts, StoreError, Timing, check, lib)

__all__ = ["ModelCfg", "ChunkId", "Engine", "ChunkKVStore", "Result", "preset", "hash_tokens",
           "ContractError", "StoreError", "FormatError", "CudaError", "OutOfMemory", "FragError",
           "ISOLATED", "FUSED", "launch_count", "memcpy", "fkvc_write", "fkvc_read", "chunk_owner",
           "PeerRecord", "TIER_GPU", "TIER_PEER", "manifest_validate"]

ISOLATED, FUSED = 0, 1
TIER_GPU, TIER_CPU, TIER_DISK, TIER_PEER = 0, 1, 2, 3
SELECTORS = {"query_guided": 0, "cacheblend": 1}
DEV_COMPONENTS = {"k": 0, "v": 1, "kv": 2}
WEIGHT_IDS = {"emb": 0, "lm_head": 1, "wq": 2, "wk": 3, "wv": 4, "wo": 5, "w_gate": 6, "w_up": 7,
              "w_down": 8, "attn_norm": 9, "ffn_norm": 10, "final_norm": 11}


def preset(name: str) -> ModelCfg:
    cfg = ModelCfg()
    check(lib.frag_model_preset(name.encode(), C.byref(cfg)))
    return cfg


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _i32p(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def hash_tokens(tokens: Sequence[int], salt: int = 0) -> ChunkId:
    t = _i32(tokens)
    out = ChunkId()
    lib.frag_hash_tokens(_i32p(t), len(t), salt, C.byref(out))
    return out


def chunk_owner(chunk_id: ChunkId, n_owners: int) -> int:
    """Owning rank of a chunk in the chunk-partitioned store (frag_chunk_owner)."""
    r = int(lib.frag_chunk_owner(C.byref(chunk_id), int(n_owners)))
    if r < 0:
        raise ContractError("n_owners must be >= 1")
    return r


def launch_count() -> int:
    return int(lib.frag_launch_count())


def set_shared_v(on: bool | None = None) -> bool:
    """Shared V pages on/off (process wide; None only queries). Returns the
    previous setting (frag_set_shared_v)."""
    return bool(lib.frag_set_shared_v(-1 if on is None else int(bool(on))))


def memcpy(dst_ptr: int, src_ptr: int, nbytes: int) -> None:
    check(lib.frag_memcpy(C.c_void_p(dst_ptr), C.c_void_p(src_ptr), nbytes))


def _stream_ptr(stream) -> C.c_void_p:
    if stream is None:
        return C.c_void_p(0)
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(int(stream.cuda_stream))  # torch.cuda.Stream


class Engine:
    """init_model: weights from the seeded splitmix64 Rng, bf16 on the GPU."""

    def __init__(self, cfg: ModelCfg | str, device: int = 0, seed: int = 1234):
        self.cfg = preset(cfg) if isinstance(cfg, str) else cfg
        self.device = device
        self.seed = seed
        self._h = C.c_void_p()
        check(lib.frag_engine_create(C.byref(self.cfg), device, seed, C.byref(self._h)))

    def close(self):
        if self._h:
            check(lib.frag_engine_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def weight(self, name: str, layer: int = 0) -> np.ndarray:
        """Canonical [out][in] weight as float32 (values are exactly the bf16 weights)."""
        c = self.cfg
        d, V, F, qc, kc = c.d_model, c.vocab, c.ffn_dim, c.n_heads * c.head_dim, c.n_kv_heads * c.head_dim
        shapes = {"emb": (V, d), "lm_head": (V, d), "wq": (qc, d), "wk": (kc, d), "wv": (kc, d),
                  "wo": (d, qc), "w_gate": (F, d), "w_up": (F, d), "w_down": (d, F), "attn_norm": (d,),
                  "ffn_norm": (d,), "final_norm": (d,)}
        shp = shapes[name]
        buf = np.empty(int(np.prod(shp)), dtype=np.uint16)
        check(lib.frag_engine_weight(self._h, layer, WEIGHT_IDS[name], buf.ctypes.data_as(C.c_void_p), buf.size))
        return (buf.astype(np.uint32) << 16).view(np.float32).reshape(shp)

    def profile(self, enable: bool = True):
        check(lib.frag_engine_profile(self._h, int(enable)))

    def profile_read(self, klass: int, reset: bool = False) -> dict:
        ms, fl, by, n = C.c_double(), C.c_double(), C.c_double(), C.c_int64()
        check(lib.frag_engine_profile_read(self._h, klass, C.byref(ms), C.byref(fl), C.byref(by), C.byref(n),
                                           int(reset)))
        return {"ms": ms.value, "flops": fl.value, "bytes": by.value, "launches": n.value}

    # ---- pipeline entry points
    def preprocess_isolated(self, store: "ChunkKVStore", tokens: Sequence[int], system: Sequence[int] = (),
                            overwrite: bool = False) -> ChunkId:
        t, s = _i32(tokens), _i32(system)
        out = ChunkId()
        check(lib.frag_preprocess_isolated(self._h, store._h, _i32p(s), len(s), _i32p(t), len(t), int(overwrite),
                                           C.byref(out)))
        return out

    def preprocess_fused(self, store: "ChunkKVStore", chunk: Sequence[int], neighbors: Sequence[ChunkId],
                         system: Sequence[int] = (), *, dst: "ChunkKVStore | None" = None, budget: int = 2048,
                         overwrite: bool = False) -> ChunkId:
        """Eq. 10: prefill `chunk` against KV_S + its neighbours'
        ISOLATED records (descending similarity order) -> FUSED record in dst."""
        t, s = _i32(chunk), _i32(system)
        nb = (ChunkId * max(len(neighbors), 1))(*neighbors)
        cid = ChunkId()
        check(lib.frag_preprocess_fused(self._h, store._h, (dst if dst is not None else store)._h, _i32p(s), len(s), _i32p(t), len(t),
                                        nb, len(neighbors), int(budget), int(overwrite), C.byref(cid)))
        return cid

    def reprocess(self, store: "ChunkKVStore", question: Sequence[int], chunk_ids: Sequence[ChunkId],
                  ratio: float, result: "Result", system: Sequence[int] = (), *, raw_scores: bool = False,
                  all_logits: bool = False, timing: bool = False, inject_crit: Sequence[int] | None = None,
                  logits_on_device: bool = False, stream=None, question_dev_ptr: int | None = None,
                  n_question: int | None = None, selector: str = "query_guided", deviation_layer: int = 2,
                  deviation_component: str = "k", fallback: Sequence[Sequence[int] | None] | None = None
                  ) -> "Result":
        """One request of the online reprocessing stage.
        selector: "query_guided" (FusionRAG) or "cacheblend"
        (layer-`deviation_layer` KV deviation; component "k", "v"
        or "kv"). fallback: per chunk its token ids (or None) -- a chunk the
        store does not hold is then prefilled in isolation on the fly and
        inserted (flag-gated); without it a miss is StoreError."""
        s = _i32(system)
        ids = (ChunkId * max(len(chunk_ids), 1))(*chunk_ids)
        opts = ReprocessOpts()
        opts.raw_scores = int(raw_scores)
        opts.all_logits = int(all_logits)
        opts.timing = int(timing)
        opts.logits_on_device = int(logits_on_device)
        opts.selector = SELECTORS[selector]
        opts.deviation_layer = int(deviation_layer)
        opts.deviation_component = DEV_COMPONENTS[deviation_component]
        keep = []
        if fallback is not None:
            if len(fallback) != len(chunk_ids):
                raise ContractError("fallback needs one entry per chunk id")
            arrs = [None if f is None else _i32(f) for f in fallback]
            keep.append(arrs)
            ptrs = (C.POINTER(C.c_int32) * max(len(arrs), 1))(
                *[C.POINTER(C.c_int32)() if a is None else _i32p(a) for a in arrs])
            lens = _i32([0 if a is None else len(a) for a in arrs])
            keep += [ptrs, lens]
            opts.fallback_tokens = C.cast(ptrs, C.POINTER(C.POINTER(C.c_int32)))
            opts.fallback_lens = _i32p(lens)
        inj = None
        if inject_crit is not None:
            inj = _i32(inject_crit)
            opts.inject_crit = _i32p(inj)
            opts.n_inject = len(inj)
        if question_dev_ptr is not None:
            check(lib.frag_reprocess_dev(self._h, store._h, _i32p(s), len(s), C.c_void_p(question_dev_ptr),
                                         int(n_question), ids, len(chunk_ids), float(ratio), C.byref(opts),
                                         _stream_ptr(stream), result._h))
        else:
            q = _i32(question)
            check(lib.frag_reprocess(self._h, store._h, _i32p(s), len(s), _i32p(q), len(q), ids, len(chunk_ids),
                                     float(ratio), C.byref(opts), _stream_ptr(stream), result._h))
        return result

    def reprocess_batch(self, store: "ChunkKVStore", requests: Sequence, result: "Result", slot_tokens: int, *,
                        raw_scores: bool = False, timing: bool = False, logits_on_device: bool = False,
                        stream=None) -> "Result":
        """Multi-request batching: requests = [(question, chunk_ids, ratio[, system])]; request b
        occupies fused-cache rows [b*slot_tokens, ...) of `result` (capacity >= len * slot_tokens).
        Logits: one row per request; critical positions via result.batch_crit(b)."""
        keep = []
        arr = (Request * len(requests))()
        for i, rq in enumerate(requests):
            q, ids, ratio = rq[0], rq[1], rq[2]
            sysm = rq[3] if len(rq) > 3 else ()
            qa, sa = _i32(q), _i32(sysm)
            ia = (ChunkId * max(len(ids), 1))(*ids)
            keep += [qa, sa, ia]
            arr[i].sys = _i32p(sa)
            arr[i].n_sys = len(sa)
            arr[i].question = _i32p(qa)
            arr[i].n_q = len(qa)
            arr[i].chunk_ids = ia
            arr[i].n_chunks = len(ids)
            arr[i].recompute_ratio = float(ratio)
        opts = ReprocessOpts()
        opts.raw_scores = int(raw_scores)
        opts.timing = int(timing)
        opts.logits_on_device = int(logits_on_device)
        check(lib.frag_reprocess_batch(self._h, store._h, arr, len(requests), int(slot_tokens), C.byref(opts),
                                       _stream_ptr(stream), result._h))
        return result

    def full_prefill(self, tokens: Sequence[int], result: "Result", system: Sequence[int] = (), *,
                     timing: bool = False, stream=None) -> "Result":
        t, s = _i32(tokens), _i32(system)
        opts = ReprocessOpts()
        opts.timing = int(timing)
        check(lib.frag_full_prefill(self._h, _i32p(s), len(s), _i32p(t), len(t), C.byref(opts), _stream_ptr(stream),
                                    result._h))
        return result

    def kv_deviation(self, store: "ChunkKVStore", chunk_ids: Sequence[ChunkId], result: "Result",
                     system: Sequence[int] = (), n_layers: int = 2, *, stream=None) -> np.ndarray:
        """kv_deviation (Eq. 7): [N][n_layers][2] fp32 sums of
        squared K / V differences between Full Attention and Full Reuse over
        cat(system, chunks); `result` holds the Full-Reuse cache afterwards."""
        s = _i32(system)
        ids = (ChunkId * max(len(chunk_ids), 1))(*chunk_ids)
        n = sum(store.peek(i).n_tok for i in chunk_ids)
        out = np.empty((max(n, 1), n_layers, 2), np.float32)
        check(lib.frag_kv_deviation(self._h, store._h, _i32p(s), len(s), ids, len(chunk_ids), int(n_layers),
                                    _stream_ptr(stream), result._h, C.c_void_p(out.ctypes.data)))
        return out[:n]

    def decode(self, result: "Result", max_new_tokens: int, *, stream=None) -> np.ndarray:
        """Greedy decoding continuing the last reprocess / full prefill of
        `result` (sparse_prefill_and_decode): max_new_tokens ids,
        the first one from the prefill logits; decoded tokens' K/V are appended
        to the result's fused cache."""
        out = np.empty(max(int(max_new_tokens), 1), dtype=np.int32)
        check(lib.frag_decode(self._h, result._h, int(max_new_tokens), _stream_ptr(stream), _i32p(out)))
        return out[:max_new_tokens]


@dataclass
class Record:
    id: ChunkId
    n_tok: int
    native_start: int
    variant: int
    tier: int
    heat: int
    last_access: int
    size_bytes: int
    k_dev: int
    v_dev: int
    tokens_dev: int


class ChunkKVStore:
    """HBM-resident chunk-KV store (GPU tier only)."""

    def __init__(self, cfg: ModelCfg, device: int = 0, capacity_bytes: int = 0):
        self.cfg = cfg
        self._h = C.c_void_p()
        check(lib.frag_store_create(C.byref(cfg), device, capacity_bytes, C.byref(self._h)))

    def close(self):
        if self._h:
            check(lib.frag_store_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __len__(self):
        return int(lib.frag_store_count(self._h))

    @property
    def bytes_used(self) -> int:
        return int(lib.frag_store_bytes_used(self._h))

    def put_record(self, chunk_id: ChunkId, tokens: Sequence[int], native_start: int, k_ptr: int, v_ptr: int,
                   variant: int = ISOLATED, overwrite: bool = False):
        """k_ptr/v_ptr: host or device addresses of [L][n][Hkv][dh] bf16."""
        t = _i32(tokens)
        check(lib.frag_store_put(self._h, C.byref(chunk_id), _i32p(t), len(t), native_start, variant,
                                 C.c_void_p(k_ptr), C.c_void_p(v_ptr), int(overwrite)))

    def fetch(self, chunk_id: ChunkId) -> Record:
        v = RecordView()
        check(lib.frag_store_fetch(self._h, C.byref(chunk_id), C.byref(v)))
        return self._rec(v)

    def release(self, chunk_id: ChunkId):
        check(lib.frag_store_release(self._h, C.byref(chunk_id)))

    def peek(self, chunk_id: ChunkId) -> Record:
        v = RecordView()
        check(lib.frag_store_peek(self._h, C.byref(chunk_id), C.byref(v)))
        return self._rec(v)

    def read_kv(self, chunk_id: ChunkId) -> tuple[np.ndarray, np.ndarray]:
        """Record K, V as uint16 (bf16 bits) host arrays [L][n][Hkv][dh]."""
        r = self.peek(chunk_id)
        c = self.cfg
        shp = (c.layers, r.n_tok, c.n_kv_heads, c.head_dim)
        k = np.empty(shp, dtype=np.uint16)
        v = np.empty(shp, dtype=np.uint16)
        memcpy(k.ctypes.data, r.k_dev, k.nbytes)
        memcpy(v.ctypes.data, r.v_dev, v.nbytes)
        return k, v

    # ------------------------------------------------ FKVC files
    def save_record(self, chunk_id: ChunkId, path: str):
        """serialize_record: the record as an FKVC file (fp32, exact)."""
        check(lib.frag_store_save(self._h, C.byref(chunk_id), str(path).encode()))

    def load_record(self, path: str, tokens: Sequence[int], *, overwrite: bool = False, stream=None) -> ChunkId:
        """deserialize_record + DISK -> GPU load: the file's
        record (id from the file) with the caller's token ids."""
        t = _i32(tokens)
        cid = ChunkId()
        check(lib.frag_store_load(self._h, str(path).encode(), _i32p(t), len(t), int(overwrite),
                                  _stream_ptr(stream), C.byref(cid)))
        return cid

    def save_manifest(self, directory: str, name: str = "manifest.json") -> int:
        """Every record this store owns as <directory>/<id hex>.fkvc plus the
        JSON manifest; returns the number of records."""
        n = C.c_int32()
        check(lib.frag_store_save_manifest(self._h, str(directory).encode(), name.encode(), C.byref(n)))
        return n.value

    def load_manifest(self, path: str, *, overwrite: bool = False, stream=None) -> int:
        """Load every record a manifest lists (DISK -> GPU)."""
        n = C.c_int32()
        check(lib.frag_store_load_manifest(self._h, str(path).encode(), int(overwrite), _stream_ptr(stream),
                                           C.byref(n)))
        return n.value

    # ------------------------------------------------ alternative_path_match
    def register_prefix(self, path: Sequence[ChunkId], system: Sequence[int] | None = None):
        """Record that path[-1]'s record was computed under (system, path[:-1])."""
        ids = (ChunkId * max(len(path), 1))(*path)
        sid = hash_tokens(system) if system else None
        check(lib.frag_store_register_prefix(self._h, None if sid is None else C.byref(sid), ids, len(path)))

    def match(self, context: Sequence[ChunkId], system: Sequence[int] | None = None) -> list[tuple]:
        """[(chunk_id, "PREFIX" | "ALT_PATH", position, path_start)] for every
        context chunk with a record (in context order); others are absent."""
        n = len(context)
        ids = (ChunkId * max(n, 1))(*context)
        out = (Match * max(n, 1))()
        got = C.c_int32()
        sid = hash_tokens(system) if system else None
        check(lib.frag_store_match(self._h, None if sid is None else C.byref(sid), ids, n, out, C.byref(got)))
        res = []
        for m in out[:got.value]:
            cid = ChunkId()
            C.memmove(C.byref(cid), C.byref(m.id), 16)
            res.append((cid, "PREFIX" if m.matched_via == 0 else "ALT_PATH", m.position, m.path_start))
        return res

    # ------------------------------------------------ chunk-partitioned store
    def attach_peer(self, other: "ChunkKVStore"):
        """Serve misses from `other` (a store on another GPU of this process);
        its pages are read in place over NVLink. `other` must outlive self."""
        check(lib.frag_store_attach_peer(self._h, other._h))
        self._peers = getattr(self, "_peers", []) + [other]  # keep the owner alive

    def export_record(self, chunk_id: ChunkId) -> bytes:
        """CUDA-IPC export of an owned record: 128 bytes for any transport."""
        pr = PeerRecord()
        check(lib.frag_store_export(self._h, C.byref(chunk_id), C.byref(pr)))
        return bytes(pr)

    def import_record(self, blob: bytes, tokens: Sequence[int], *, overwrite: bool = False) -> ChunkId:
        """Register another process's exported record as a FRAG_TIER_PEER view."""
        if len(blob) != C.sizeof(PeerRecord):
            raise ContractError("peer record blob must be 128 bytes")
        pr = PeerRecord.from_buffer_copy(blob)
        t = _i32(tokens)
        check(lib.frag_store_import(self._h, C.byref(pr), _i32p(t), len(t), int(overwrite)))
        cid = ChunkId()
        C.memmove(C.byref(cid), C.byref(pr.id), 16)
        return cid

    @staticmethod
    def _rec(v: RecordView) -> Record:
        cid = ChunkId()
        C.memmove(C.byref(cid), C.byref(v.id), 16)
        return Record(cid, v.n_tok, v.native_start, v.variant, v.tier, v.heat, v.last_access, v.size_bytes,
                      v.k_dev or 0, v.v_dev or 0, v.tokens_dev or 0)


class Result:
    """Per-request fused KV cache + logits (reusable across requests)."""

    def __init__(self, engine: Engine, max_tokens: int):
        self.engine = engine
        self._h = C.c_void_p()
        check(lib.frag_result_create(engine._h, max_tokens, C.byref(self._h)))
        self.max_tokens = max_tokens

    def close(self):
        if self._h:
            check(lib.frag_result_free(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sync(self):
        check(lib.frag_result_sync(self._h))

    @property
    def n_tokens(self) -> int:
        n = C.c_int32()
        check(lib.frag_result_fused_kv(self._h, None, None, C.byref(n)))
        return n.value

    def memory(self) -> tuple[int, bool]:
        """(device bytes held by the result, whether its last request used shared V pages)."""
        b, sv = C.c_uint64(), C.c_int32()
        check(lib.frag_result_memory(self._h, C.byref(b), C.byref(sv)))
        return int(b.value), bool(sv.value)

    def fused_ptrs(self) -> tuple[int, int]:
        k, v = C.c_void_p(), C.c_void_p()
        check(lib.frag_result_fused_kv(self._h, C.byref(k), C.byref(v), None))
        return k.value, v.value

    def fused_kv(self) -> tuple[np.ndarray, np.ndarray]:
        """Fused K, V as uint16 bf16 bits [L][T][Hkv][dh] (copied to host)."""
        c = self.engine.cfg
        T = self.n_tokens
        kp, vp = self.fused_ptrs()
        out = []
        for p in (kp, vp):
            a = np.empty((c.layers, self.max_tokens, c.n_kv_heads, c.head_dim), dtype=np.uint16)
            memcpy(a.ctypes.data, p, a.nbytes)
            out.append(np.ascontiguousarray(a[:, :T]))
        return out[0], out[1]

    def logits(self) -> np.ndarray:
        p = C.POINTER(C.c_float)()
        rows, vocab = C.c_int32(), C.c_int32()
        check(lib.frag_result_logits(self._h, C.byref(p), C.byref(rows), C.byref(vocab), 0))
        return np.ctypeslib.as_array(p, shape=(rows.value, vocab.value)).copy()

    def logits_dev_ptr(self) -> int:
        p = C.POINTER(C.c_float)()
        check(lib.frag_result_logits(self._h, C.byref(p), None, None, 1))
        return C.cast(p, C.c_void_p).value

    def crit(self) -> np.ndarray:
        k = lib.frag_result_crit(self._h, None, 0)
        out = np.empty(max(k, 1), dtype=np.int32)
        if k > 0:
            lib.frag_result_crit(self._h, _i32p(out), k)
        return out[:k]

    def batch_crit(self, b: int) -> np.ndarray:
        """Critical positions (1-based) of request b of the last reprocess_batch."""
        n = int(lib.frag_result_batch_crit(self._h, int(b), None, 0))
        if n < 0:
            raise ContractError("no such request in the last batch")
        out = np.empty(max(n, 1), dtype=np.int32)
        lib.frag_result_batch_crit(self._h, int(b), _i32p(out), n)
        return out[:n]

    def timing(self) -> dict:
        t = Timing()
        check(lib.frag_result_timing(self._h, C.byref(t)))
        return t.as_dict()

    def debug(self) -> dict:
        qf, sc = C.c_void_p(), C.c_void_p()
        nq, n = C.c_int32(), C.c_int32()
        check(lib.frag_result_debug(self._h, C.byref(qf), C.byref(sc), C.byref(nq), C.byref(n)))
        c = self.engine.cfg
        q = np.empty((nq.value, c.n_heads, c.head_dim), dtype=np.float32)
        s = np.empty(max(n.value, 1), dtype=np.float32)
        if nq.value and qf.value:  # the cacheblend selector runs no question pass
            memcpy(q.ctypes.data, qf.value, q.nbytes)
        if n.value:
            memcpy(s.ctypes.data, sc.value, n.value * 4)
        return {"q_final": q, "scores": s[:n.value]}


def manifest_validate(path: str) -> int:
    """Host-only check of an FKVC manifest and the headers of the files it
    lists (no device); returns the number of records."""
    n = C.c_int32()
    check(lib.frag_manifest_validate(str(path).encode(), C.byref(n)))
    return n.value


def fkvc_write(path: str, chunk_id: ChunkId, k: np.ndarray, v: np.ndarray, native_start: int,
               variant: int = ISOLATED):
    """Host FKVC writer (no GPU): k, v fp32 [layers][tokens][heads][head_dim]."""
    k = np.ascontiguousarray(k, np.float32)
    v = np.ascontiguousarray(v, np.float32)
    assert k.shape == v.shape and k.ndim == 4
    h = FkvcHeader()
    C.memmove(C.byref(h.id), C.byref(chunk_id), 16)
    h.variant, h.native_start = variant, native_start
    h.layers, h.tokens, h.heads, h.head_dim = k.shape
    check(lib.frag_fkvc_write(str(path).encode(), C.byref(h), C.c_void_p(k.ctypes.data), C.c_void_p(v.ctypes.data)))


def fkvc_read(path: str, header_only: bool = False):
    """Host FKVC reader (no GPU) -> (header dict, k, v) with fp32 [layers][tokens][heads][head_dim]."""
    h = FkvcHeader()
    check(lib.frag_fkvc_read(str(path).encode(), C.byref(h), None, None, 0))
    cid = ChunkId()
    C.memmove(C.byref(cid), C.byref(h.id), 16)
    hd = {"id": cid, "variant": h.variant, "native_start": h.native_start, "layers": h.layers, "heads": h.heads,
          "head_dim": h.head_dim, "tokens": h.tokens}
    if header_only:
        return hd, None, None
    shp = (h.layers, h.tokens, h.heads, h.head_dim)
    k = np.empty(shp, np.float32)
    v = np.empty(shp, np.float32)
    check(lib.frag_fkvc_read(str(path).encode(), C.byref(h), C.c_void_p(k.ctypes.data), C.c_void_p(v.ctypes.data),
                             k.size))
    return hd, k, v
