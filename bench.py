#!/usr/bin/env python
"""Benchmark of the FusionRAG online reprocessing stage on B200.

Workload (BASELINE.json configs[1]): Llama-3-8B-shaped model (32 layers, GQA
32/8, d=4096, random init), 8 retrieved chunks x 2048 tokens (16k prompt),
32-token question, 15% recompute. One "step" = one reprocess request
(stitch -> question pass -> query-guided select -> sparse prefill -> first-token
logits). Chunk records are HBM-resident (preprocessed on the GPU at setup).

  value  : effective prefill tok/s = prompt tokens / TTFT, whole job (sum over
           ranks / max-over-ranks device time), question tokens already on device.
  e2e    : same metric through the C-ABI call a user makes (frag_reprocess with
           host question tokens, host logits), H2D/D2H inside the timed region.
  extra  : TTFT ms, the same kernels' full-attention prefill TTFT and the speedup.

`--impl reference` times the reference's CPU path (the C++ oracle restatement;
the reference ships no implementation) on the host cores.

Launch: python bench.py [--gpus N --steps K --warmup W]. N>1: under torchrun
(one rank per GPU), or without it bench.py spawns the N ranks itself through
torch.distributed.run on 127.0.0.1.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_CLASSES = 8  # frag_engine_profile_read classes (frag_c.h)
CLASS_NAMES = ["gemm", "attention", "stitch", "norm", "select", "gemm_stream", "gemm_gateup", "vwindow"]
METRIC = "TTFT ms at 16k-token RAG prompt, 15% recompute vs full prefill; prefill tok/s"
CONFIGS = {
    "llama3-8b": dict(preset="llama3-8b", chunks=8, chunk_len=2048, qlen=32, ratio=0.15),
    "mistral-7b": dict(preset="mistral-7b", chunks=32, chunk_len=1024, qlen=32, ratio=0.15),
    # 64 independent queries, each picking 32 of a
    # 256-chunk corpus, split round-robin over the ranks (steps = queries/rank)
    "mistral-7b-batch": dict(preset="mistral-7b", chunks=32, chunk_len=1024, qlen=32, ratio=0.15, corpus=256,
                             queries=64),
    # the full 80-layer model fits one B200 (141 GB bf16
    # weights); the chunk-KV store is partitioned over the ranks (NVLink peer reads)
    "llama3-70b": dict(preset="llama3-70b", chunks=8, chunk_len=2048, qlen=32, ratio=0.15, partition=True),
    "tiny": dict(preset="tiny", chunks=8, chunk_len=256, qlen=32, ratio=0.15),
}


def l2_note(w, c):
    """c: model shape as a dict (layers, d_model, n_heads, ...)."""
    per_layer = (c["n_heads"] + 2 * c["n_kv_heads"]) * c["head_dim"] * c["d_model"] \
        + c["n_heads"] * c["head_dim"] * c["d_model"] + 3 * c["d_model"] * c["ffn_dim"]
    wbytes = 2 * (c["layers"] * per_layer + 2 * c["vocab"] * c["d_model"])
    T = w["chunks"] * w["chunk_len"] + w["qlen"]
    kv = 2 * c["layers"] * T * c["n_kv_heads"] * c["head_dim"] * 2
    if wbytes + kv < 126e6:
        return "fits in L2 (tiny test config, not a headline run)"
    return (f"inputs larger than L2 ({wbytes / 1e9:.1f} GB weights, {kv / 2e9:.1f} GB fused K + "
            f"{kv / 2e9:.1f} GB of the records' V pages per request, streamed every step)")


def cpu_model() -> str:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="llama3-8b", choices=sorted(CONFIGS))
    p.add_argument("--ratio", type=float, default=None)
    p.add_argument("--seed", type=int, default=1234)
    p.add_argument("--full-steps", type=int, default=2)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-layers", type=int, default=1)
    p.add_argument("--sweep", default="0,0.05,0.3,1.0",
                   help="comma list of extra ratios to time (BASELINE.json configs[2]; '' to skip)")
    p.add_argument("--partition", action="store_true",
                   help="chunk-partitioned store: each chunk's record lives on rank hash(id) mod N only and "
                        "the other ranks read it over NVLink inside K1 (SURVEY.md §8(e))")
    p.add_argument("--batch", type=int, default=None,
                   help="also time multi-request batching (frag_reprocess_batch) with this many requests; 0 = skip "
                        "(default 8 for the batched corpus config, else 4)")
    p.add_argument("--selftest", action="store_true",
                   help="CPU/gloo check of the multi-rank launcher (no GPU work)")
    p.add_argument("--with-load", action="store_true",
                   help="also time TTFT including the FKVC record load (DISK -> GPU, SPEC.md:301-308)")
    return p.parse_args()


# ---------------------------------------------------------------- multi-rank
def max_over_ranks(vals, device):
    """Element-wise max of per-rank device times (one process per GPU; no
    collective touches the data path -- requests are independent)."""
    import torch
    t = torch.tensor([float(v) for v in vals], dtype=torch.float64, device=device)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return t.tolist()


def job_throughput(world, steps, tokens_per_request, max_ms):
    """Whole-job tok/s: every rank served `steps` requests of `tokens_per_request`
    prompt tokens; the job took the slowest rank's time (weak scaling)."""
    return world * steps * tokens_per_request / (max_ms / 1e3)


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for n, v in zip(names, s[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        pw = [float(s[3]) for s in self.samples if s[3].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples),
                "power_w": statistics.median(pw) if pw else None}


class EnergyMeter:
    """Board energy over a region from NVML's cumulative counter (mJ), plus the
    enforced power limit: the request runs at the power cap, so its TTFT is
    set by joules per request (profiles/gemm_tile_width_r02.md)."""

    def __init__(self, gpu: int):
        self.h = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(gpu)
        except Exception:
            self.h = None

    def read_mj(self):
        if self.h is None:
            return None
        try:
            return self.nv.nvmlDeviceGetTotalEnergyConsumption(self.h)
        except Exception:
            return None

    def limit_w(self):
        if self.h is None:
            return None
        try:
            return self.nv.nvmlDeviceGetEnforcedPowerLimit(self.h) / 1e3
        except Exception:
            return None


def peaks():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        d = json.loads(f.read_text())
        return d.get("bf16_tflops_sustained", 1397.5), d.get("bf16_tflops", 1693.4), d.get("hbm_gbs", 6450.9), \
            "measured"
    return 1400.0, 1590.0, 6650.0, "fallback"


# ---------------------------------------------------------------- CPU baseline (oracle)
class CpuBaseline:
    """The reference's CPU path (the C++/OpenMP oracle restatement, the
    reference ships no implementation) on this host's cores, on a bounded
    sample of the workload: the full request at full width and prompt length
    on `layers` of the model's layers (synthetic random chunk KV). A step is
    one oracle reprocess of that sample; its per-layer stage times are
    extrapolated to the model depth (labelled as such). Reads the shapes from
    oracle/presets.py: nothing here loads the product library."""

    def __init__(self, cfg_name, ratio, layers, seed=1234):
        from oracle import oracle as O
        from oracle import presets as OP
        self.O = O
        self.w = CONFIGS[cfg_name]
        self.name, self.ratio = cfg_name, ratio
        self.full = OP.preset(self.w["preset"])
        c = dict(self.full)
        c["layers"] = layers = min(layers, self.full["layers"])
        self.layers = layers
        self.om = O.Model(c).init_seed(seed)
        rng = np.random.default_rng(seed)
        Hkv, dh = c["n_kv_heads"], c["head_dim"]
        self.recs = []
        for _ in range(self.w["chunks"]):
            n = self.w["chunk_len"]
            self.recs.append({"k": (rng.standard_normal((layers, n, Hkv, dh), dtype=np.float32) * 0.5),
                              "v": (rng.standard_normal((layers, n, Hkv, dh), dtype=np.float32) * 0.5),
                              "tokens": rng.integers(0, c["vocab"], n).astype(np.int32), "native_start": 1})
        self.qrng = np.random.default_rng(seed + 1)
        self.cores = O.threads()

    def step(self):
        """One sample request: returns (wall seconds, extrapolated full-depth TTFT seconds, T)."""
        q = self.qrng.integers(0, self.full["vocab"], self.w["qlen"])
        t0 = time.perf_counter()
        out = self.om.reprocess(None, self.recs, q, self.ratio, emulate_bf16=False)
        wall = time.perf_counter() - t0
        st = out["stage_seconds"]  # stitch, question, select, sparse(+lm_head)
        scale = self.full["layers"] / self.layers
        return wall, (st[0] + st[1] + st[3]) * scale + st[2], out["T"]

    def sample(self, wall=None):
        s = (f"oracle reprocess (C++/OpenMP fp32, {self.cores} threads, {cpu_model()}), {self.name} width, "
             f"{self.layers}/{self.full['layers']} layers, T={self.w['chunks'] * self.w['chunk_len'] + self.w['qlen']}, "
             f"r={self.ratio}, random chunk KV; value = per-layer stage times x{self.full['layers'] / self.layers:g} "
             f"(extrapolated to the full depth)")
        return s + (f"; wall {wall:.1f}s per sample" if wall is not None else "")


def tiny_reference(seed=1234):
    """configs[0] measured in full on the CPU (2 layers, d=256, 8x256 chunks +
    32 question, r=0.15): no extrapolation."""
    b = CpuBaseline("tiny", 0.15, 2, seed)
    b.step()
    walls = [b.step()[0] for _ in range(3)]
    T = b.w["chunks"] * b.w["chunk_len"] + b.w["qlen"]
    ms = statistics.median(walls) * 1e3
    return {"config": "tiny (BASELINE.json configs[0]), all layers, measured", "ttft_ms": ms,
            "tok_s": T / (ms / 1e3), "cores": b.cores}


def cpu_baseline(cfg_name, ratio, layers, seed=1234):
    """One bounded sample of the oracle on the host (rank 0, N=1 only)."""
    b = CpuBaseline(cfg_name, ratio, layers, seed)
    wall, ttft, T = b.step()
    return T / ttft, ttft, b.cores, b.sample(wall)


# ---------------------------------------------------------------- ours
def run_ours(args, rank, world, local_rank):
    import torch
    from paper_2601_12904_b200 import fusion as F

    w = CONFIGS[args.config]
    ratio = w["ratio"] if args.ratio is None else args.ratio
    if args.batch is None:
        args.batch = 8 if w.get("corpus") else 4
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    eng = F.Engine(w["preset"], device=local_rank, seed=args.seed)
    c = eng.cfg
    store = F.ChunkKVStore(c, device=local_rank)
    rng = np.random.default_rng(1000 + rank)
    if w.get("corpus"):
        # the same seeded corpus on every rank (store replica); this rank serves
        # queries rank, rank + world, ... each over 32 Rng-picked chunks
        crng = np.random.default_rng(args.seed)
        pool = [crng.integers(0, c.vocab, w["chunk_len"]).astype(np.int32) for _ in range(w["corpus"])]
        if args.partition or w.get("partition"):
            from paper_2601_12904_b200 import partition as P
            pool_ids = [F.hash_tokens(ch) for ch in pool]
            owned = {}
            for cid, ch, o in zip(pool_ids, pool, P.owners(pool_ids, world)):
                if o == rank:
                    eng.preprocess_isolated(store, ch)
                    owned[cid] = ch
            if world > 1:
                P.share_records(store, owned)
        else:
            pool_ids = [eng.preprocess_isolated(store, ch) for ch in pool]
        mine = [q for q in range(w["queries"]) if q % world == rank]
        picks = [np.random.default_rng(args.seed * 1000 + q).choice(w["corpus"], w["chunks"], replace=False)
                 for q in mine]
        id_sets = [[pool_ids[j] for j in pk] for pk in picks]
        chunks = [pool[j] for j in picks[0]]
        args.steps = len(mine)
    elif args.partition or w.get("partition"):
        # one shared set of chunks; rank hash(id) mod N owns each record, the
        # others import a CUDA-IPC view of it (K1 reads it over NVLink)
        from paper_2601_12904_b200 import partition as P
        crng = np.random.default_rng(args.seed)
        chunks = [crng.integers(0, c.vocab, w["chunk_len"]).astype(np.int32) for _ in range(w["chunks"])]
        cids = [F.hash_tokens(ch) for ch in chunks]
        owned = {}
        for cid, ch, o in zip(cids, chunks, P.owners(cids, world)):
            if o == rank:
                eng.preprocess_isolated(store, ch)
                owned[cid] = ch
        if world > 1:
            P.share_records(store, owned)
        id_sets = [cids]
    else:
        chunks = [rng.integers(0, c.vocab, w["chunk_len"]).astype(np.int32) for _ in range(w["chunks"])]
        id_sets = [[eng.preprocess_isolated(store, ch) for ch in chunks]]
    ids = id_sets[0]
    N = w["chunks"] * w["chunk_len"]
    T = N + w["qlen"]
    n_q = args.warmup + args.steps
    questions = [rng.integers(0, c.vocab, w["qlen"]).astype(np.int32) for _ in range(2 * n_q + 4)]
    q_dev = [torch.from_numpy(q).to(dev) for q in questions]
    n_dec = 16
    res = F.Result(eng, T + n_dec)  # + room for the greedy decode leg
    stream = torch.cuda.current_stream(dev)

    def step_dev(i, r=ratio, **kw):
        # request i serves query (i - warmup): the timed loop covers every query of this rank once
        eng.reprocess(store, None, id_sets[(i - args.warmup) % len(id_sets)], r, res, stream=stream,
                      question_dev_ptr=q_dev[i].data_ptr(), n_question=w["qlen"], logits_on_device=True, **kw)

    for i in range(args.warmup):
        step_dev(i)
    torch.cuda.synchronize()

    # ---- timed region (device-resident inputs)
    launches0 = F.launch_count()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    meter = EnergyMeter(local_rank)
    with ClockSampler(local_rank) as clk:
        e_start, t_start = meter.read_mj(), time.perf_counter()  # the device is idle here (synchronized)
        ev0.record(stream)
        for i in range(args.steps):
            step_dev(args.warmup + i)
        ev1.record(stream)
        torch.cuda.synchronize()
        e_end, t_end = meter.read_mj(), time.perf_counter()  # before the sampler thread is joined
    energy = None
    if e_start is not None and e_end is not None and e_end > e_start:
        energy = {"j_per_request": (e_end - e_start) / 1e3 / args.steps,
                  "avg_power_w": (e_end - e_start) / 1e3 / (t_end - t_start),
                  "power_limit_w": meter.limit_w(),
                  "source": "NVML total energy counter around the timed requests (board, this GPU)"}
    if world > 1:
        torch.distributed.barrier()
    ms = ev0.elapsed_time(ev1)
    launches = F.launch_count() - launches0
    crit = res.crit()
    mem_shared = res.memory()  # before any V read-back / full prefill allocates a private fused V

    # ---- per-kernel-class device time: the same K requests again with CUDA
    # events around every launch on the launching stream (kept out of the
    # headline loop because the ~700 event records per request cost host time)
    eng.profile(True)
    for k in range(N_CLASSES):
        eng.profile_read(k, reset=True)
    for i in range(args.steps):
        step_dev(args.warmup + i)
    torch.cuda.synchronize()
    prof = {k: eng.profile_read(k) for k in range(N_CLASSES)}
    eng.profile(False)

    # ---- stage breakdown (one extra request with per-stage events)
    step_dev(0, timing=True)
    stages = res.timing()

    # ---- greedy decode after the reprocess (sparse_prefill_and_decode);
    # one untimed decode first: its steps are the first sighting and the graph
    # capture of the decode-step shape, which the timed decode then replays
    step_dev(0)
    eng.decode(res, n_dec, stream=stream)
    step_dev(0)
    d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    d0.record(stream)
    answer = eng.decode(res, n_dec, stream=stream)
    d1.record(stream)
    torch.cuda.synchronize()
    decode_ms = d0.elapsed_time(d1) / (n_dec - 1)

    # ---- TTFT including the record load from FKVC files (optional)
    load_leg = None
    if args.with_load:
        import shutil
        import tempfile
        tdir = tempfile.mkdtemp(prefix="frag_fkvc_")
        try:
            paths = []
            for i, cid in enumerate(ids):
                pth = os.path.join(tdir, f"c{i}.fkvc")
                store.save_record(cid, pth)
                paths.append(pth)
            fbytes = sum(os.path.getsize(pth) for pth in paths)
            st_l = F.ChunkKVStore(c, device=local_rank)
            runs = []
            for it in range(2):  # the second pass reads from the page cache
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                for pth, ch in zip(paths, chunks):
                    st_l.load_record(pth, ch, overwrite=True, stream=stream)
                t1 = time.perf_counter()
                eng.reprocess(st_l, questions[it], ids, ratio, res, stream=stream)
                t2 = time.perf_counter()
                runs.append({"load_ms": (t1 - t0) * 1e3, "ttft_with_load_ms": (t2 - t0) * 1e3,
                             "load_gbs": fbytes / (t1 - t0) / 1e9})
            load_leg = {"file_bytes": fbytes, "runs": runs,
                        "note": "host wall clock: FKVC fp32 files read layer by layer into pinned ping-pong "
                                "buffers, H2D + bf16 conversion overlapped with the next layer's read"}
            del st_l
        finally:
            shutil.rmtree(tdir, ignore_errors=True)

    # ---- e2e through the C-ABI call with host buffers (two untimed requests
    # first: a device buffer grown by the legs above -- the decode's RoPE table
    # -- invalidates the captured request graph, which the first re-runs eagerly
    # and the second re-captures)
    for i in range(2):
        eng.reprocess(store, questions[n_q + i], id_sets[i % len(id_sets)], ratio, res, stream=stream)
        _ = res.logits()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        eng.reprocess(store, questions[n_q + i], id_sets[i % len(id_sets)], ratio, res,
                      stream=stream)
        _ = res.logits()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    dh = c.head_dim
    h2d = w["qlen"] * 4 * 2 + (w["chunks"]) * 32 + w["chunks"] * (dh // 2) * 8 + 4
    d2h = c.vocab * 4

    # ---- ratio sweep, after the e2e leg and before the full prefill: a 300 ms
    # full-power burst leaves the next requests at lower clocks
    # (tools/r0_check.py); r = 1.0 comes last in the default list
    sweep = {}
    for r in [float(x) for x in args.sweep.split(",") if x.strip()]:
        step_dev(1, r=r)  # first sighting of this request shape: eager
        step_dev(1, r=r)  # second: graph capture; the timed requests replay it
        step_dev(1, r=r)
        per = []
        for i in range(3):  # median of three device-timed requests
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            step_dev(2 + i, r=r)
            s1.record(stream)
            torch.cuda.synchronize()
            per.append(s0.elapsed_time(s1))
        sweep[str(r)] = round(sorted(per)[1], 3)

    # ---- same kernels' full-attention prefill (every chunk token recomputed, no question pass/select)
    fa = res
    toks = np.concatenate(chunks + [questions[0]])
    eng.full_prefill(toks, fa, stream=stream)
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(args.full_steps):
        eng.full_prefill(toks, fa, stream=stream)
    f1.record(stream)
    torch.cuda.synchronize()
    full_ms = f0.elapsed_time(f1) / args.full_steps
    mem_private = res.memory()  # the full prefill keeps a private fused V [L][max_tokens]

    # ---- CacheBlend selector on the same requests: 2-layer
    # Full-Attention pass + layer-2 K deviation instead of the question pass + K9
    step_dev(1, selector="cacheblend")
    step_dev(2, selector="cacheblend")
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record(stream)
    for i in range(2):
        step_dev(3 + i, selector="cacheblend")
    c1.record(stream)
    torch.cuda.synchronize()
    cacheblend_ms = c0.elapsed_time(c1) / 2
    step_dev(1, selector="cacheblend", timing=True)
    cacheblend_stages = res.timing()

    # ---- multi-request batching: B requests (this rank's next queries) in one
    # fused cache, one question pass + one sparse pass streaming the weights once
    batch_leg = None
    kv_bytes = 2 * c.layers * T * c.n_kv_heads * c.head_dim * 2
    free_b = torch.cuda.mem_get_info(dev)[0]
    if args.batch and args.batch > 1 and args.batch * kv_bytes * 1.3 > free_b:
        batch_leg = {"skipped": f"{args.batch} x {kv_bytes / 1e9:.1f} GB fused KV does not fit the "
                                f"{free_b / 1e9:.0f} GB free"}
    elif args.batch and args.batch > 1:
        B = args.batch
        rb = F.Result(eng, B * T)
        reqs = [(questions[(3 + i) % len(questions)], id_sets[i % len(id_sets)], ratio) for i in range(B)]
        for _ in range(2):  # eager first sighting, then the graph capture; the timed batches replay it
            eng.reprocess_batch(store, reqs, rb, T, stream=stream, logits_on_device=True)
        torch.cuda.synchronize()
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        nb = 3
        b0.record(stream)
        for _ in range(nb):
            eng.reprocess_batch(store, reqs, rb, T, stream=stream, logits_on_device=True)
        b1.record(stream)
        torch.cuda.synchronize()
        bms = b0.elapsed_time(b1) / nb
        eng.reprocess_batch(store, reqs, rb, T, stream=stream, timing=True)
        batch_leg = {"requests": B, "batch_ms": bms, "ms_per_request": bms / B, "tok_s": B * T / (bms / 1e3),
                     "stage_ms": rb.timing(),
                     "note": "frag_reprocess_batch: every request's TTFT is the batch latency; throughput leg, "
                             "not in value"}
        del rb

    if world > 1:
        torch.distributed.barrier()  # peers may still read this rank's records until every rank is done
    return dict(ms=ms, e2e_ms=e2e_ms, full_ms=full_ms, launches=launches, prof=prof, stages=stages, T=T,
                crit=crit, clocks=clk.summary(), energy=energy, cfg=c, w=w, ratio=ratio, h2d=h2d, d2h=d2h, sweep=sweep,
                k=len(crit), decode_ms=decode_ms, n_dec=len(answer), load_leg=load_leg,
                cacheblend_ms=cacheblend_ms, cacheblend_stages=cacheblend_stages, batch_leg=batch_leg,
                mem_shared=mem_shared, mem_private=mem_private)


def spawn_ranks(n: int, argv: list[str], backend_env: dict | None = None) -> int:
    """`bench.py --gpus N` outside torchrun: launch N ranks (one process per
    GPU) through torch.distributed.run on 127.0.0.1 and return its exit code;
    rank 0's JSON line goes to this process's stdout."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *argv]
    env = dict(os.environ, **(backend_env or {}))
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("OMP_NUM_THREADS", str(max(1, (os.cpu_count() or n) // n)))
    print(f"bench: spawning {n} ranks (torch.distributed.run, master 127.0.0.1:{port})", file=sys.stderr, flush=True)
    return subprocess.run(cmd, env=env).returncode


def selftest_ranks(args, rank, world):
    """CPU check of the launcher plumbing (gloo): every rank reports a
    rank-dependent 'device time', rank 0 prints the contract line built from
    the max over ranks. tests/test_bench_multirank.py runs it at world 2."""
    import torch
    torch.distributed.init_process_group("gloo")
    ms = max_over_ranks([100.0 + 10.0 * rank], torch.device("cpu"))[0]
    T = 16416
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": job_throughput(world, args.steps, T, ms), "unit": "tok/s",
                          "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                          "selftest": True}), flush=True)
    torch.distributed.destroy_process_group()
    return 0


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn_ranks(args.gpus, sys.argv[1:])
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and rank == 0:
        print(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}; reporting n_gpus={world}", file=sys.stderr)
    if args.selftest:
        return selftest_ranks(args, rank, world)
    w = CONFIGS[args.config]
    ratio = w["ratio"] if args.ratio is None else args.ratio
    cfg_json = {"workload": f"{args.config}: {w['chunks']}x{w['chunk_len']}-token chunks + {w['qlen']}-token "
                            f"question, r={ratio}", "model": w["preset"], "chunks": w["chunks"],
                "chunk_len": w["chunk_len"], "question_len": w["qlen"], "recompute_ratio": ratio,
                "seq_len": w["chunks"] * w["chunk_len"] + w["qlen"],
                "parallelism": f"dp{world} (independent queries)"}
    part = args.partition or w.get("partition", False)
    cfg_json["store"] = ("partitioned: record on rank hash(chunk_id) mod N only, read by the other ranks over "
                         "NVLink inside K1 (CUDA IPC views)") if part else "replicated per rank"
    if w.get("corpus"):
        cfg_json.update({"corpus_chunks": w["corpus"], "queries": w["queries"],
                         "steps_note": "steps = this rank's share of the queries (round-robin)"})

    if args.impl == "reference":
        if rank != 0:
            return 0
        from oracle import presets as OP
        cfg_json["l2"] = l2_note(w, OP.preset(w["preset"]))
        base = CpuBaseline(args.config, ratio, args.cpu_layers, args.seed)
        for _ in range(args.warmup):
            base.step()
        walls, ttfts = [], []
        for _ in range(max(1, args.steps)):
            wall, ttft, T = base.step()
            walls.append(wall)
            ttfts.append(ttft)
        value = T / statistics.median(ttfts)
        ms_step = statistics.mean(walls) * 1e3
        line = {"metric": METRIC, "value": value, "unit": "tok/s", "impl": "reference", "n_gpus": 1,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic", "config": cfg_json,
                "value_basis": (f"extrapolated: each step measures the full request on {base.layers} of "
                                f"{base.full['layers']} layers (ms_per_step = that measured wall time); value = "
                                f"prompt tokens / (per-layer stage times x{base.full['layers'] / base.layers:g})"),
                "ttft_ms_extrapolated": statistics.median(ttfts) * 1e3,
                "cpu": {"model": cpu_model(), "threads": base.cores, "host_cpus": os.cpu_count()},
                "cpu_baseline": {"value": value, "unit": "tok/s", "cores": base.cores, "kind": "port",
                                 "sample": base.sample(statistics.mean(walls))},
                "e2e": {"value": value, "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        try:
            line["tiny_config"] = tiny_reference(args.seed)
        except Exception as ex:  # reported, never fatal
            line["tiny_config"] = {"failed": str(ex)}
        print(json.dumps(line), flush=True)
        return 0

    from paper_2601_12904_b200 import fusion as F
    cfg_json["l2"] = l2_note(w, F.preset(w["preset"]).as_dict())
    if world > 1:
        import torch
        if torch.cuda.device_count() < world:
            raise SystemExit(f"bench: {world} ranks but only {torch.cuda.device_count()} visible GPUs "
                             "(one process per GPU)")
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    r = run_ours(args, rank, world, local_rank)
    import torch
    ms, e2e_ms, full_ms = r["ms"], r["e2e_ms"], r["full_ms"]
    if world > 1:
        ms, e2e_ms, full_ms = max_over_ranks([ms, e2e_ms, full_ms], torch.device("cuda", local_rank))
    T = r["T"]
    ttft = ms / args.steps
    value = job_throughput(world, args.steps, T, ms)
    e2e_value = job_throughput(world, args.steps, T, e2e_ms)
    sus, burst, hbm, src = peaks()
    g = r["prof"][0]
    gemm_tflops = g["flops"] / (g["ms"] / 1e3) / 1e12 if g["ms"] > 0 else None
    # roofline kernel: the gate/up projection GEMM of the sparse pass
    # (gemm_tc2_kernel<256, EPI_SWIGLU>, the single largest launch: its own
    # profile class, events around each of its launches); traffic = its DRAM
    # bytes per launch from the committed ncu --set full capture of the same
    # kernel (profiles/ncu_traffic.json, cold-cache, one launch)
    gu = r["prof"][6]
    gu_tflops = gu["flops"] / (gu["ms"] / 1e3) / 1e12 if gu["ms"] > 0 else None
    traffic, traffic_src = None, None
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if tf.exists():
        try:
            js = json.loads(tf.read_text())
            traffic = js.get("gemm_tc2_gateup_bytes_per_launch")
            traffic_src = js.get("source")
        except Exception:
            traffic = None
    c = r["cfg"]
    # attention FLOPs: 4*Hq*dh*sum_rows(p_i) per layer (each query row sees exactly
    # p_i keys); the last layer attends only for the logit row (no other
    # consumer of its output)
    crit = r["crit"]
    qpos = np.arange(T - r["w"]["qlen"] + 1, T + 1)
    attn_flops = 4.0 * c.n_heads * c.head_dim * ((c.layers - 1) * (float(np.sum(crit)) + float(np.sum(qpos)))
                                                 + float(T))
    a = r["prof"][1]
    line = {
        "metric": METRIC, "value": value, "unit": "tok/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ttft, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (seeded random weights, tokens and questions)",
        "config": cfg_json,
        "ttft_ms": ttft, "full_prefill_ms": full_ms, "speedup_vs_full_prefill": full_ms / ttft,
        "recomputed_rows": r["k"] + r["w"]["qlen"], "stage_ms": r["stages"],
        "ratio_sweep_ttft_ms": r["sweep"] or None,
        "batched": r["batch_leg"],
        "cacheblend": {"ttft_ms": r["cacheblend_ms"], "stage_ms": r["cacheblend_stages"],
                       "note": "same requests with the CacheBlend selector (2-layer Full-Attention pass + layer-2 "
                               "K deviation, SPEC.md:417) instead of the query-guided one; not in value"},
        "queries_per_s": world * args.steps / (ms / 1e3),
        "ttft_with_load": r["load_leg"],
        "decode": {"ms_per_token": r["decode_ms"], "tokens": r["n_dec"],
                   "note": "greedy single-row steps over the fused cache after the timed requests, graph-replayed (an untimed decode captures the step first); not in value"},
        "e2e": {"value": e2e_value, "unit": "tok/s", "ttft_ms": e2e_ms / args.steps,
                "h2d_bytes_per_step": r["h2d"], "d2h_bytes_per_step": r["d2h"]},
        "gpu_launches": r["launches"],
        "roofline": {"bound": "tensor",
                     "kernel": "gemm_tc2_kernel<256, SWIGLU> (K8 gate/up projection of the sparse pass, tcgen05 "
                               "cta_group::2)",
                     "achieved": gu_tflops, "peak": sus, "unit": "TFLOP/s",
                     "frac": (gu_tflops / sus) if gu_tflops else None, "traffic": traffic,
                     "traffic_source": traffic_src,
                     "algorithmic_flop_per_launch": (gu["flops"] / gu["launches"]) if gu["launches"] else None,
                     "launch_ms": (gu["ms"] / gu["launches"]) if gu["launches"] else None,
                     "peak_source": f"{src} bf16_tflops_sustained (kernel timed inside the long step)",
                     "kernel_share_of_step": gu["ms"] / args.steps / ttft if ttft else None,
                     "all_tensor_gemms": {"achieved": gemm_tflops, "frac": (gemm_tflops / sus) if gemm_tflops else None,
                                          "share_of_step": g["ms"] / ms if ms else None}},
        "kernels": {name: {"ms_per_step": r["prof"][k]["ms"] / args.steps,
                           "launches_per_step": r["prof"][k]["launches"] / args.steps}
                    for k, name in enumerate(CLASS_NAMES)},
        "attention": {"achieved_tflops": attn_flops / (a["ms"] / args.steps / 1e3) / 1e12 if a["ms"] else None,
                      "flops_per_step": attn_flops},
        "stitch": {"achieved_gbs": (r["prof"][2]["bytes"] / (r["prof"][2]["ms"] / 1e3) / 1e9)
                   if r["prof"][2]["ms"] else None, "peak_gbs": hbm,
                   "bytes_per_step": r["prof"][2]["bytes"] / args.steps},
        "vwindow": {"achieved_gbs": (r["prof"][7]["bytes"] / (r["prof"][7]["ms"] / 1e3) / 1e9)
                    if r["prof"][7]["ms"] else None, "peak_gbs": hbm,
                    "note": "shared V pages: per-layer V window fills of the sparse pass (side stream, overlapped "
                            "with the GEMMs)"},
        "hbm_per_request": {"shared_v_bytes": r["mem_shared"][0], "shared_v": r["mem_shared"][1],
                            "private_v_bytes": r["mem_private"][0],
                            "note": "device bytes held by the request's result: fused K + exclusive V slots + "
                                    "staging window + workspaces (shared V pages) vs the same result once it holds "
                                    "a private fused V (full prefill)"},
        "gemm_stream": {"achieved_gbs": (r["prof"][5]["bytes"] / (r["prof"][5]["ms"] / 1e3) / 1e9)
                        if r["prof"][5]["ms"] else None, "peak_gbs": hbm,
                        "note": "one-M-tile GEMMs (question pass, lm_head): algorithmic bytes = weights + rows"},
        "clocks": r["clocks"],
        "energy": r.get("energy"),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            v, t, cores, sample = cpu_baseline(args.config, ratio, args.cpu_layers, args.seed)
            line["cpu_baseline"] = {"value": v, "unit": "tok/s", "cores": cores, "kind": "port", "sample": sample,
                                    "ttft_ms_extrapolated": t * 1e3}
        except Exception as ex:  # reported, never fatal
            line["cpu_baseline"] = {"value": None, "unit": "tok/s", "cores": None, "kind": "port",
                                    "sample": f"failed: {ex}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
