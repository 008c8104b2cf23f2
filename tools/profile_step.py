"""Run the bench workload and bracket ONE reprocess request with
cudaProfilerStart/Stop so ncu (--profile-from-start off) captures exactly the
kernels of a single request (no setup / preprocessing launches).

  ncu --profile-from-start off --metrics gpu__time_duration.sum --csv ... python tools/profile_step.py
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--preset", default="llama3-8b")
    ap.add_argument("--chunks", type=int, default=8)
    ap.add_argument("--chunk-len", type=int, default=2048)
    ap.add_argument("--qlen", type=int, default=32)
    ap.add_argument("--ratio", type=float, default=0.15)
    ap.add_argument("--full", action="store_true", help="profile the full-attention prefill instead")
    a = ap.parse_args()
    import torch
    from paper_2601_12904_b200 import fusion as F
    eng = F.Engine(a.preset, seed=1234)
    c = eng.cfg
    store = F.ChunkKVStore(c)
    rng = np.random.default_rng(3)
    chunks = [rng.integers(0, c.vocab, a.chunk_len).astype(np.int32) for _ in range(a.chunks)]
    ids = [eng.preprocess_isolated(store, ch) for ch in chunks]
    q = rng.integers(0, c.vocab, a.qlen).astype(np.int32)
    T = a.chunks * a.chunk_len + a.qlen
    res = F.Result(eng, T)
    toks = np.concatenate(chunks + [q])
    for _ in range(2):
        if a.full:
            eng.full_prefill(toks, res)
        else:
            eng.reprocess(store, q, ids, a.ratio, res)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    if a.full:
        eng.full_prefill(toks, res)
    else:
        eng.reprocess(store, q, ids, a.ratio, res)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("profiled one request, T =", T)


if __name__ == "__main__":
    main()
