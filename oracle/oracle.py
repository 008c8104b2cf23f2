"""numpy front-end of the CPU oracle (oracle/fusion_oracle.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py. The product path
(paper_2601_12904_b200, libfrag.so) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "build" / "libfragoracle.so"

_F = np.float32


class OrcCfg(C.Structure):
    _fields_ = [("layers", C.c_int32), ("d_model", C.c_int32), ("n_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("ffn_dim", C.c_int32),
                ("vocab", C.c_int32), ("rope_base", C.c_double), ("norm_eps", C.c_float)]


def build():
    subprocess.run(["make", "-C", str(HERE), "all"], check=True, capture_output=True)


def _load():
    if not LIB.exists():
        build()
    lib = C.CDLL(str(LIB))
    P, I32P = C.c_void_p, C.POINTER(C.c_int32)
    sig = {
        "orc_rng": (None, [C.c_uint64, C.c_int, C.c_int, C.c_uint64, P]),
        "orc_weight_seed": (C.c_uint64, [C.c_uint64, C.c_int]),
        "orc_gen_normal": (None, [C.c_uint64, C.c_size_t, C.c_float, C.c_int, C.c_int, P]),
        "orc_set_threads": (None, [C.c_int]),
        "orc_get_threads": (C.c_int, []),
        "orc_model_create": (P, [C.POINTER(OrcCfg)]),
        "orc_model_free": (None, [P]),
        "orc_model_tensor": (C.POINTER(C.c_float), [P, C.c_int, C.c_int, C.POINTER(C.c_size_t)]),
        "orc_model_init_seed": (None, [P, C.c_uint64]),
        "orc_rope_apply": (None, [P, C.c_int, C.c_double, C.c_double]),
        "orc_shift_rope": (None, [P, C.c_int, C.c_int, C.c_int, C.c_double]),
        "orc_forward": (C.c_int, [P, C.c_int, P, P, P, P, P, P, C.c_int, P, P, C.c_int, P, P, C.c_int, C.c_int]),
        "orc_stitch": (C.c_int, [C.POINTER(OrcCfg), C.c_int, P, P, P, P, P, P, P, C.c_int, C.c_int]),
        "orc_select": (None, [P, P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, P, P]),
        "orc_q_sparse_attn": (C.c_int, [P, P, P, C.c_int, P, P, P, P, C.c_int, C.c_int, C.c_int, P]),
        "orc_build_equivalent_mask": (None, [P, P, C.c_int, C.c_int, P]),
        "orc_kv_deviation": (C.c_int, [P, C.c_int, P, P, C.c_int, P, P, P, P, P, C.c_int, C.c_int, P]),
        "orc_select_cacheblend": (None, [P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, P]),
        "orc_reprocess": (C.c_int, [P, C.c_int, P, P, P, C.c_int, P, P, P, P, P, C.c_int, P, C.c_float, C.c_int,
                                    P, C.c_int, C.c_int, P, P, C.c_int, P, P, P, P, P, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()


def _p(a: np.ndarray | None):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _c(a, dtype) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=dtype))


def set_threads(n: int):
    lib.orc_set_threads(n)


def threads() -> int:
    return lib.orc_get_threads()


# ---------------------------------------------------------------- Rng (common.hpp:45-100)
def rng(seed: int, kind: str, n: int, arg: int = 0) -> np.ndarray:
    kinds = {"next_u64": (0, np.uint64), "normal": (1, np.float64), "normal_f_0.02": (2, np.float32),
             "below": (3, np.uint64), "next_float": (4, np.float32), "next_double": (5, np.float64),
             "range": (6, np.int64)}
    k, dt = kinds[kind]
    out = np.empty(n, dtype=dt)
    lib.orc_rng(seed, k, n, arg, _p(out))
    return out


def weight_seed(seed: int, tensor_id: int) -> int:
    return int(lib.orc_weight_seed(seed, tensor_id))


def gen_normal(stream_seed: int, n: int, sigma: float = 0.02, sequential: bool = False,
               round_bf16: bool = True) -> np.ndarray:
    out = np.empty(n, dtype=_F)
    lib.orc_gen_normal(stream_seed, n, sigma, int(sequential), int(round_bf16), _p(out))
    return out


def bf16_round(x: np.ndarray) -> np.ndarray:
    b = np.ascontiguousarray(x, dtype=_F).view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return b.astype(np.uint32).view(_F)


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(bits).astype(np.uint32) << 16).view(_F)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    return (bf16_round(x).view(np.uint32) >> 16).astype(np.uint16)


# ---------------------------------------------------------------- rope
def rope_apply(v: np.ndarray, pos: float, base: float = 1e4) -> np.ndarray:
    out = _c(v, _F).copy()
    lib.orc_rope_apply(_p(out), out.shape[-1], float(pos), base)
    return out


def shift_rope(v: np.ndarray, old: int, new: int, base: float = 1e4) -> np.ndarray:
    out = _c(v, _F).copy()
    lib.orc_shift_rope(_p(out), out.shape[-1], int(old), int(new), base)
    return out


WEIGHT_IDS = {"emb": 0, "lm_head": 1, "wq": 2, "wk": 3, "wv": 4, "wo": 5, "w_gate": 6, "w_up": 7,
              "w_down": 8, "attn_norm": 9, "ffn_norm": 10, "final_norm": 11}


class Model:
    """fp32 oracle model; weights filled from the GPU engine or from the seed."""

    def __init__(self, cfg):
        self.cfg = OrcCfg(*[getattr(cfg, f) for f, _ in OrcCfg._fields_]) if not isinstance(cfg, dict) else \
            OrcCfg(**cfg)
        self._h = C.c_void_p(lib.orc_model_create(C.byref(self.cfg)))

    def __del__(self):
        try:
            lib.orc_model_free(self._h)
        except Exception:
            pass

    def tensor(self, name: str, layer: int = 0) -> np.ndarray:
        n = C.c_size_t()
        ptr = lib.orc_model_tensor(self._h, layer, WEIGHT_IDS[name], C.byref(n))
        return np.ctypeslib.as_array(ptr, shape=(n.value,))

    def load_from_engine(self, engine) -> "Model":
        names = ["emb", "lm_head", "final_norm"]
        for nm in names:
            self.tensor(nm)[:] = engine.weight(nm).ravel()
        for l in range(self.cfg.layers):
            for nm in ["wq", "wk", "wv", "wo", "w_gate", "w_up", "w_down", "attn_norm", "ffn_norm"]:
                self.tensor(nm, l)[:] = engine.weight(nm, l).ravel()
        return self

    def init_seed(self, seed: int) -> "Model":
        lib.orc_model_init_seed(self._h, seed)
        return self

    # ------------------------------------------------------------ forward
    def forward(self, tokens, positions, slots, cache_k, cache_v, cache_pos, mask=None, logit_rows=None,
                want_q=False, stop_after_last_q=False, emulate_bf16=False):
        c = self.cfg
        tokens, positions, slots = _c(tokens, np.int32), _c(positions, np.int32), _c(slots, np.int32)
        n = len(tokens)
        cap = cache_k.shape[1]
        assert cache_k.dtype == _F and cache_k.flags.c_contiguous and cache_pos.dtype == np.int32
        lr = None if logit_rows is None else _c(logit_rows, np.int32)
        logits = None if lr is None else np.empty((len(lr), c.vocab), dtype=_F)
        q = np.empty((n, c.n_heads, c.head_dim), dtype=_F) if want_q else None
        m = None if mask is None else _c(mask, np.uint8)
        rc = lib.orc_forward(self._h, n, _p(tokens), _p(positions), _p(slots), _p(cache_k), _p(cache_v),
                             _p(cache_pos), cap, _p(m), _p(logits), 0 if lr is None else len(lr), _p(lr), _p(q),
                             int(stop_after_last_q), int(emulate_bf16))
        if rc != 0:
            raise ValueError(f"orc_forward contract violation ({rc})")
        return logits, q

    def new_cache(self, cap: int):
        c = self.cfg
        shp = (c.layers, cap, c.n_kv_heads, c.head_dim)
        return np.zeros(shp, _F), np.zeros(shp, _F), np.zeros(cap, np.int32)

    # ------------------------------------------------------------ pipeline
    def reprocess(self, sys_kv, records, question, ratio, raw=False, inject=None, emulate_bf16=True, cap=None):
        """records: list of dicts {k, v: [L][n][Hkv][dh] f32, tokens, native_start}; sys_kv: (k, v) or None."""
        c = self.cfg
        S = 0 if sys_kv is None else sys_kv[0].shape[1]
        N = sum(len(r["tokens"]) for r in records)
        q = _c(question, np.int32)
        T = S + N + len(q)
        cap = cap or T
        kc, vc = np.zeros((c.layers, cap, c.n_kv_heads, c.head_dim), _F), np.zeros(
            (c.layers, cap, c.n_kv_heads, c.head_dim), _F)
        ks = [_c(r["k"], _F) for r in records]
        vs = [_c(r["v"], _F) for r in records]
        toks = [_c(r["tokens"], np.int32) for r in records]
        nat = _c([r["native_start"] for r in records], np.int32)
        ns = _c([len(t) for t in toks], np.int32)
        kp = (C.c_void_p * max(len(ks), 1))(*[a.ctypes.data for a in ks])
        vp = (C.c_void_p * max(len(vs), 1))(*[a.ctypes.data for a in vs])
        tp = (C.c_void_p * max(len(toks), 1))(*[a.ctypes.data for a in toks])
        sk = sv = None
        if S:
            sk, sv = _c(sys_kv[0], _F), _c(sys_kv[1], _F)
        logits = np.empty(c.vocab, _F)
        crit = np.empty(max(N, 1), np.int32)
        kk = C.c_int32()
        qf = np.empty((len(q), c.n_heads, c.head_dim), _F)
        scores = np.zeros(max(N, 1), np.float64)
        stages = np.zeros(4, np.float64)
        inj = None if inject is None else _c(inject, np.int32)
        rc = lib.orc_reprocess(self._h, S, _p(sk), _p(sv), None, len(records), kp, vp, tp, _p(ns), _p(nat), len(q),
                               _p(q), float(ratio), int(raw), _p(inj), 0 if inj is None else len(inj),
                               int(emulate_bf16), _p(kc), _p(vc), cap, _p(logits), _p(crit), C.byref(kk), _p(qf),
                               _p(scores), _p(stages))
        if rc != 0:
            raise ValueError(f"orc_reprocess failed ({rc})")
        k = kk.value
        return {"k": kc[:, :T], "v": vc[:, :T], "logits": logits, "crit": crit[:k].copy(), "q_final": qf,
                "scores": scores[:N], "stage_seconds": stages, "T": T, "k_cache": kc, "v_cache": vc}

    # ------------------------------------------------------------ CacheBlend
    def kv_deviation(self, sys_kv, records, n_layers=2, emulate_bf16=True):
        """Eq. 7 over cat(S, chunks): [N][n_layers][2] fp64 (K, V)."""
        S = 0 if sys_kv is None else sys_kv[0].shape[1]
        N = sum(len(r["tokens"]) for r in records)
        ks = [_c(r["k"], _F) for r in records]
        vs = [_c(r["v"], _F) for r in records]
        toks = [_c(r["tokens"], np.int32) for r in records]
        kp = (C.c_void_p * len(ks))(*[a.ctypes.data for a in ks])
        vp = (C.c_void_p * len(vs))(*[a.ctypes.data for a in vs])
        tp = (C.c_void_p * len(toks))(*[a.ctypes.data for a in toks])
        ns = _c([len(t) for t in toks], np.int32)
        nat = _c([r["native_start"] for r in records], np.int32)
        sk = sv = None
        if S:
            sk, sv = _c(sys_kv[0], _F), _c(sys_kv[1], _F)
        dev = np.zeros((N, n_layers, 2), np.float64)
        rc = lib.orc_kv_deviation(self._h, S, _p(sk), _p(sv), len(records), kp, vp, tp, _p(ns), _p(nat),
                                  int(n_layers), int(emulate_bf16), _p(dev))
        if rc != 0:
            raise ValueError(f"orc_kv_deviation failed ({rc})")
        return dev

    # ------------------------------------------------------------ decode
    def decode_forced(self, cache_k, cache_v, T, tokens, emulate_bf16=True):
        """Decode steps of sparse_prefill_and_decode with given inputs: token i
        is fed at position T+i+1 (cache slot T+i) against the fused cache, its
        K/V appended (exclusive pages); returns the logits after each step
        [len(tokens)][V]. Greedy decoding = feeding back the argmax."""
        cap = cache_k.shape[1]
        assert T + len(tokens) <= cap
        pos = np.zeros(cap, np.int32)
        pos[:T] = np.arange(1, T + 1, dtype=np.int32)
        out = []
        for i, t in enumerate(tokens):
            lg, _ = self.forward([int(t)], [T + i + 1], [T + i], cache_k, cache_v, pos, logit_rows=[0],
                                 emulate_bf16=emulate_bf16)
            out.append(lg[0].copy())
        return np.array(out)

    def greedy_decode(self, cache_k, cache_v, T, first_logits, n, emulate_bf16=True):
        """Greedy decoding of n tokens (token 0 = argmax(first_logits), lowest
        index on ties)."""
        toks = [int(np.argmax(first_logits))]
        for i in range(n - 1):
            pos_T = T + i
            cap = cache_k.shape[1]
            pos = np.zeros(cap, np.int32)
            pos[:pos_T] = np.arange(1, pos_T + 1, dtype=np.int32)
            lg, _ = self.forward([toks[-1]], [pos_T + 1], [pos_T], cache_k, cache_v, pos, logit_rows=[0],
                                 emulate_bf16=emulate_bf16)
            toks.append(int(np.argmax(lg[0])))
        return np.array(toks, np.int32)


def stitch(cfg, chunks, cap, round_bf16=True):
    """chunks: list of (k, v, native_start, dst_row) with k/v [L][n][Hkv][dh] f32."""
    oc = OrcCfg(*[getattr(cfg, f) for f, _ in OrcCfg._fields_])
    ks = [_c(ch[0], _F) for ch in chunks]
    vs = [_c(ch[1], _F) for ch in chunks]
    kp = (C.c_void_p * len(ks))(*[a.ctypes.data for a in ks])
    vp = (C.c_void_p * len(vs))(*[a.ctypes.data for a in vs])
    ns = _c([a.shape[1] for a in ks], np.int32)
    nat = _c([ch[2] for ch in chunks], np.int32)
    dst = _c([ch[3] for ch in chunks], np.int32)
    shp = (oc.layers, cap, oc.n_kv_heads, oc.head_dim)
    ko, vo = np.zeros(shp, _F), np.zeros(shp, _F)
    lib.orc_stitch(C.byref(oc), len(ks), kp, vp, _p(ns), _p(nat), _p(dst), _p(ko), _p(vo), cap, int(round_bf16))
    return ko, vo


def select(q, keys, k, raw=False):
    """q [nq][Hq][dh] f32, keys [N][Hkv][dh] f32 -> (scores f64 [N], sel int32 [k] ascending)."""
    q, keys = _c(q, _F), _c(keys, _F)
    nq, Hq, dh = q.shape
    N, Hkv, _ = keys.shape
    scores = np.empty(N, np.float64)
    sel = np.empty(max(k, 1), np.int32)
    lib.orc_select(_p(q), _p(keys), nq, Hq, Hkv, dh, N, k, int(raw), _p(scores), _p(sel))
    return scores, sel[:k].copy()


def select_cacheblend(dev, k, layer=2, comp=0):
    """argTopk of dev[:, layer-1, comp] (comp 2 = K+V), lower index on ties,
    ascending 0-based chunk-token indices."""
    dev = _c(dev, np.float64)
    N, L, _ = dev.shape
    sel = np.empty(max(k, 1), np.int32)
    lib.orc_select_cacheblend(_p(dev), N, L, int(layer), int(comp), int(k), _p(sel))
    return sel[:k].copy()


def q_sparse_attn(q, shared_k, shared_v, fresh_k, fresh_v, q_idx, is_new):
    q, sk, sv, fk, fv = (_c(a, _F) for a in (q, shared_k, shared_v, fresh_k, fresh_v))
    qi, nw = _c(q_idx, np.int32), _c(is_new, np.uint8)
    nq, H, dh = q.shape
    out = np.empty_like(q)
    rc = lib.orc_q_sparse_attn(_p(q), _p(sk), _p(sv), sk.shape[0], _p(fk), _p(fv), _p(qi), _p(nw), nq, H, dh, _p(out))
    if rc != 0:
        raise ValueError(f"invalid QIndexPlan ({rc})")
    return out


def build_equivalent_mask(q_idx, is_new, T):
    qi, nw = _c(q_idx, np.int32), _c(is_new, np.uint8)
    W = T + int(nw.sum())
    m = np.empty((len(qi), W), np.uint8)
    lib.orc_build_equivalent_mask(_p(qi), _p(nw), len(qi), T, _p(m))
    return m


# ------------------------------------------------------------ alternative_path_match
def alt_path_match(cached_paths, records, context, sys_id=None):
    """Restatement of alternative_path_match (design decision
    SPEC.md:317; §4.1 "progressive backtracking"): cached_paths is a
    set of (sys_id, tuple of chunk ids) whose last chunk's record was computed
    under the preceding ones; records the set of chunk ids holding a record.
    For each context chunk with a record: PREFIX if (sys, context[:i+1]) is
    cached, else drop the earliest remaining preceding chunk until a cached
    path ending at the chunk is found (ALT_PATH); a chunk with a record but no
    cached path still matches ALT_PATH on its own (completeness).
    Returns [(chunk, via, position, path_start)]."""
    out = []
    for i, c in enumerate(context):
        if c not in records:
            continue
        hit = None
        for start in range(0, i + 1):
            if (sys_id, tuple(context[start:i + 1])) in cached_paths:
                hit = start
                break
        out.append((c, "PREFIX" if hit == 0 else "ALT_PATH", i, i if hit is None else hit))
    return out
