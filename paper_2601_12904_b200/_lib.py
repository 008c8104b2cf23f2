"""ctypes binding of libfrag.so (include/frag/frag_c.h).

The product path has no CPU fallback: if the library is missing this module
raises at import time, and every entry point reports a CUDA error when no
device is present.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libfrag.so"

FRAG_OK, FRAG_E_CONTRACT, FRAG_E_STORE, FRAG_E_FORMAT, FRAG_E_CUDA, FRAG_E_OOM = range(6)


class ModelCfg(C.Structure):
    _fields_ = [("layers", C.c_int32), ("d_model", C.c_int32), ("n_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("ffn_dim", C.c_int32),
                ("vocab", C.c_int32), ("rope_base", C.c_double), ("norm_eps", C.c_float)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class ChunkId(C.Structure):
    _fields_ = [("bytes", C.c_uint8 * 16)]

    def hex(self) -> str:
        return bytes(self.bytes).hex()

    def __eq__(self, other):
        return isinstance(other, ChunkId) and bytes(self.bytes) == bytes(other.bytes)

    def __hash__(self):
        return hash(bytes(self.bytes))


class FkvcHeader(C.Structure):
    _fields_ = [("id", ChunkId), ("variant", C.c_int32), ("native_start", C.c_int32), ("layers", C.c_int32),
                ("heads", C.c_int32), ("head_dim", C.c_int32), ("tokens", C.c_int32)]


class RecordView(C.Structure):
    _fields_ = [("id", ChunkId), ("n_tok", C.c_int32), ("native_start", C.c_int32), ("variant", C.c_int32),
                ("tier", C.c_int32), ("heat", C.c_uint64), ("last_access", C.c_uint64),
                ("size_bytes", C.c_uint64), ("k_dev", C.c_void_p), ("v_dev", C.c_void_p),
                ("tokens_dev", C.c_void_p)]


class PeerRecord(C.Structure):
    """frag_peer_record: one exported record (CUDA IPC handle + metadata), 128 bytes."""
    _fields_ = [("id", ChunkId), ("n_tok", C.c_int32), ("native_start", C.c_int32), ("variant", C.c_int32),
                ("owner_device", C.c_int32), ("layers", C.c_int32), ("n_kv_heads", C.c_int32),
                ("head_dim", C.c_int32), ("owner_pci", C.c_int32), ("kv_bytes", C.c_uint64),
                ("owner_pid", C.c_uint64), ("ipc_handle", C.c_uint8 * 64)]


assert C.sizeof(PeerRecord) == 128


class Match(C.Structure):
    _fields_ = [("id", ChunkId), ("matched_via", C.c_int32), ("position", C.c_int32), ("path_start", C.c_int32)]


class Request(C.Structure):
    _fields_ = [("sys", C.POINTER(C.c_int32)), ("n_sys", C.c_int32), ("question", C.POINTER(C.c_int32)),
                ("n_q", C.c_int32), ("chunk_ids", C.POINTER(ChunkId)), ("n_chunks", C.c_int32),
                ("recompute_ratio", C.c_float)]


class ReprocessOpts(C.Structure):
    _fields_ = [("raw_scores", C.c_int32), ("all_logits", C.c_int32), ("timing", C.c_int32),
                ("inject_crit", C.POINTER(C.c_int32)), ("n_inject", C.c_int32),
                ("logits_on_device", C.c_int32), ("selector", C.c_int32), ("deviation_layer", C.c_int32),
                ("deviation_component", C.c_int32),
                ("fallback_tokens", C.POINTER(C.POINTER(C.c_int32))), ("fallback_lens", C.POINTER(C.c_int32))]


class Timing(C.Structure):
    _fields_ = [("stitch_ms", C.c_float), ("question_ms", C.c_float), ("select_ms", C.c_float),
                ("sparse_ms", C.c_float), ("lm_head_ms", C.c_float), ("total_ms", C.c_float),
                ("host_prep_ms", C.c_float)]

    def as_dict(self):
        return {f: float(getattr(self, f)) for f, _ in self._fields_}


_P = C.c_void_p
_I32P = C.POINTER(C.c_int32)
_SIGS = {
    "frag_last_error": (C.c_char_p, []),
    "frag_version": (C.c_char_p, []),
    "frag_model_preset": (C.c_int, [C.c_char_p, C.POINTER(ModelCfg)]),
    "frag_hash_tokens": (None, [_I32P, C.c_int32, C.c_uint64, C.POINTER(ChunkId)]),
    "frag_launch_count": (C.c_uint64, []),
    "frag_set_spin_limit_ms": (C.c_double, [C.c_double]),
    "frag_set_shared_v": (C.c_int32, [C.c_int32]),
    "frag_result_memory": (C.c_int, [_P, C.POINTER(C.c_uint64), _I32P]),
    "frag_memcpy": (C.c_int, [_P, _P, C.c_size_t]),
    "frag_engine_create": (C.c_int, [C.POINTER(ModelCfg), C.c_int, C.c_uint64, C.POINTER(_P)]),
    "frag_engine_destroy": (C.c_int, [_P]),
    "frag_engine_config": (C.c_int, [_P, C.POINTER(ModelCfg)]),
    "frag_engine_weight": (C.c_int, [_P, C.c_int32, C.c_int32, _P, C.c_size_t]),
    "frag_engine_weight_seed": (C.c_uint64, [C.c_uint64, C.c_int32]),
    "frag_engine_profile": (C.c_int, [_P, C.c_int32]),
    "frag_engine_profile_read": (C.c_int, [_P, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                           C.POINTER(C.c_double), C.POINTER(C.c_int64), C.c_int32]),
    "frag_store_create": (C.c_int, [C.POINTER(ModelCfg), C.c_int, C.c_size_t, C.POINTER(_P)]),
    "frag_store_destroy": (C.c_int, [_P]),
    "frag_store_put": (C.c_int, [_P, C.POINTER(ChunkId), _I32P, C.c_int32, C.c_int32, C.c_int32, _P, _P,
                                 C.c_int32]),
    "frag_store_fetch": (C.c_int, [_P, C.POINTER(ChunkId), C.POINTER(RecordView)]),
    "frag_store_release": (C.c_int, [_P, C.POINTER(ChunkId)]),
    "frag_store_peek": (C.c_int, [_P, C.POINTER(ChunkId), C.POINTER(RecordView)]),
    "frag_store_count": (C.c_int64, [_P]),
    "frag_store_register_prefix": (C.c_int, [_P, C.POINTER(ChunkId), C.POINTER(ChunkId), C.c_int32]),
    "frag_store_match": (C.c_int, [_P, C.POINTER(ChunkId), C.POINTER(ChunkId), C.c_int32, C.POINTER(Match), _I32P]),
    "frag_chunk_owner": (C.c_int32, [C.POINTER(ChunkId), C.c_int32]),
    "frag_store_attach_peer": (C.c_int, [_P, _P]),
    "frag_store_export": (C.c_int, [_P, C.POINTER(ChunkId), C.POINTER(PeerRecord)]),
    "frag_store_import": (C.c_int, [_P, C.POINTER(PeerRecord), _I32P, C.c_int32, C.c_int32]),
    "frag_preprocess_fused": (C.c_int, [_P, _P, _P, _I32P, C.c_int32, _I32P, C.c_int32, C.POINTER(ChunkId),
                                        C.c_int32, C.c_int32, C.c_int32, C.POINTER(ChunkId)]),
    "frag_last_format_kind": (C.c_int32, []),
    "frag_fkvc_write": (C.c_int, [C.c_char_p, C.POINTER(FkvcHeader), _P, _P]),
    "frag_fkvc_read": (C.c_int, [C.c_char_p, C.POINTER(FkvcHeader), _P, _P, C.c_size_t]),
    "frag_store_save": (C.c_int, [_P, C.POINTER(ChunkId), C.c_char_p]),
    "frag_store_load": (C.c_int, [_P, C.c_char_p, _I32P, C.c_int32, C.c_int32, _P, C.POINTER(ChunkId)]),
    "frag_store_save_manifest": (C.c_int, [_P, C.c_char_p, C.c_char_p, _I32P]),
    "frag_store_load_manifest": (C.c_int, [_P, C.c_char_p, C.c_int32, _P, _I32P]),
    "frag_manifest_validate": (C.c_int, [C.c_char_p, _I32P]),
    "frag_store_bytes_used": (C.c_uint64, [_P]),
    "frag_preprocess_isolated": (C.c_int, [_P, _P, _I32P, C.c_int32, _I32P, C.c_int32, C.c_int32,
                                           C.POINTER(ChunkId)]),
    "frag_result_create": (C.c_int, [_P, C.c_int32, C.POINTER(_P)]),
    "frag_result_free": (C.c_int, [_P]),
    "frag_reprocess": (C.c_int, [_P, _P, _I32P, C.c_int32, _I32P, C.c_int32, C.POINTER(ChunkId), C.c_int32,
                                 C.c_float, C.POINTER(ReprocessOpts), _P, _P]),
    "frag_reprocess_dev": (C.c_int, [_P, _P, _I32P, C.c_int32, _P, C.c_int32, C.POINTER(ChunkId), C.c_int32,
                                     C.c_float, C.POINTER(ReprocessOpts), _P, _P]),
    "frag_full_prefill": (C.c_int, [_P, _I32P, C.c_int32, _I32P, C.c_int32, C.POINTER(ReprocessOpts), _P, _P]),
    "frag_decode": (C.c_int, [_P, _P, C.c_int32, _P, _I32P]),
    "frag_reprocess_batch": (C.c_int, [_P, _P, C.POINTER(Request), C.c_int32, C.c_int32, C.POINTER(ReprocessOpts),
                                       _P, _P]),
    "frag_result_batch_crit": (C.c_int32, [_P, C.c_int32, _I32P, C.c_int32]),
    "frag_kv_deviation": (C.c_int, [_P, _P, _I32P, C.c_int32, C.POINTER(ChunkId), C.c_int32, C.c_int32, _P, _P,
                                    _P]),
    "frag_result_sync": (C.c_int, [_P]),
    "frag_result_fused_kv": (C.c_int, [_P, C.POINTER(_P), C.POINTER(_P), _I32P]),
    "frag_result_logits": (C.c_int, [_P, C.POINTER(C.POINTER(C.c_float)), _I32P, _I32P, C.c_int32]),
    "frag_result_crit": (C.c_int32, [_P, _I32P, C.c_int32]),
    "frag_result_timing": (C.c_int, [_P, C.POINTER(Timing)]),
    "frag_result_debug": (C.c_int, [_P, C.POINTER(_P), C.POINTER(_P), _I32P, _I32P]),
    "frag_kernel_gemm": (C.c_int, [_P, _P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P]),
    "frag_kernel_rope_shift": (C.c_int, [_P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                         C.c_int32, C.c_double, _P]),
    "frag_kernel_qg_select": (C.c_int, [_P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                        C.c_int32, C.c_int32, _P, _P, _P]),
    "frag_kernel_attention": (C.c_int, [_P, _P, _P, _P, _P, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                        C.c_int32, C.c_int32, _P]),
}

if not LIB_PATH.exists():
    raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2601_12904_b200.build` "
                      "(the reprocessing path has no CPU fallback)")

lib = C.CDLL(str(LIB_PATH))
for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


class FragError(RuntimeError):
    code = -1


class ContractError(FragError):
    code = FRAG_E_CONTRACT


class StoreError(FragError):
    code = FRAG_E_STORE


class FormatError(FragError):
    """FormatError::Kind (common.hpp:33) in .kind: BadMagic, BadVersion, Truncated, Malformed, Io."""
    code = FRAG_E_FORMAT
    KINDS = ("BadMagic", "BadVersion", "Truncated", "Malformed", "Io")

    def __init__(self, msg, kind=None):
        super().__init__(msg)
        self.kind = kind


class CudaError(FragError):
    code = FRAG_E_CUDA


class OutOfMemory(FragError):
    code = FRAG_E_OOM


_ERRS = {FRAG_E_CONTRACT: ContractError, FRAG_E_STORE: StoreError, FRAG_E_FORMAT: FormatError,
         FRAG_E_CUDA: CudaError, FRAG_E_OOM: OutOfMemory}


def check(status: int) -> None:
    if status != FRAG_OK:
        msg = lib.frag_last_error().decode(errors="replace")
        if status == FRAG_E_FORMAT:
            k = int(lib.frag_last_format_kind())
            raise FormatError(msg, FormatError.KINDS[k] if 0 <= k < len(FormatError.KINDS) else None)
        raise _ERRS.get(status, FragError)(msg)


def declared_symbols(header: Path | None = None) -> list[str]:
    """Names of every FRAG_API function declared in include/frag/frag_c.h."""
    import re
    header = header or (LIB_PATH.parent.parent / "include" / "frag" / "frag_c.h")
    txt = header.read_text()
    return re.findall(r"FRAG_API\s+[\w\s\*]+?\b(frag_\w+)\s*\(", txt)
