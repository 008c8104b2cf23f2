"""Per-kernel-class device time of one frag_reprocess_batch (B requests, 8B
bench workload) vs B single requests (engine profiler: CUDA events around
every launch on the launching stream)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2601_12904_b200 import fusion as F  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4
eng = F.Engine("llama3-8b", seed=1234)
c = eng.cfg
store = F.ChunkKVStore(c)
rng = np.random.default_rng(3)
ids = [eng.preprocess_isolated(store, rng.integers(0, c.vocab, 2048).astype(np.int32)) for _ in range(8)]
qs = [rng.integers(0, c.vocab, 32).astype(np.int32) for _ in range(B)]
T = 8 * 2048 + 32
names = ["gemm", "attention", "stitch", "norm", "select", "gemm_stream"]
res1 = F.Result(eng, T)
rb = F.Result(eng, B * T)
reqs = [(q, ids, 0.15) for q in qs]
for _ in range(2):
    for q in qs:
        eng.reprocess(store, q, ids, 0.15, res1)
    eng.reprocess_batch(store, reqs, rb, T)
torch.cuda.synchronize()
for label, fn in (("single x B", lambda: [eng.reprocess(store, q, ids, 0.15, res1) for q in qs]),
                  ("batch", lambda: eng.reprocess_batch(store, reqs, rb, T))):
    eng.profile(True)
    for k in range(6):
        eng.profile_read(k, reset=True)
    fn()
    torch.cuda.synchronize()
    prof = {names[k]: eng.profile_read(k) for k in range(6)}
    eng.profile(False)
    tot = sum(v["ms"] for v in prof.values())
    print(label, f"total {tot:.2f} ms", {k: (round(v["ms"], 2), v["launches"]) for k, v in prof.items()})
    g = prof["gemm"]
    print("   gemm TFLOP/s", g["flops"] / (g["ms"] / 1e3) / 1e12 if g["ms"] else None)
