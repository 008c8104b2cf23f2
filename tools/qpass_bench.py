"""Question-pass / weight-streaming A/B on the 8B 16k request: r = 0.15
request with per-stage timing (question pass), r = 0 one-pass TTFT and greedy
decode ms/token, device-timed medians. Switches come from the environment
(e.g. FRAG_CHAIN_PF=0 / 24), so run one process per setting:

    for pf in 0 16 24 32; do FRAG_CHAIN_PF=$pf python tools/qpass_bench.py; done
"""
import os
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_12904_b200 import fusion as F  # noqa: E402

ballast = None
if os.environ.get("QB_BALLAST_GB"):  # extra device memory held during the run (TLB / placement check)
    ballast = torch.empty(int(float(os.environ["QB_BALLAST_GB"]) * 2**30), dtype=torch.uint8, device="cuda")
tag = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith(("FRAG_", "QB_"))) or "defaults"
eng = F.Engine("llama3-8b", seed=1)
c = eng.cfg
store = F.ChunkKVStore(c)
rng = np.random.default_rng(0)
ids = [eng.preprocess_isolated(store, rng.integers(0, c.vocab, 2048).tolist()) for _ in range(8)]
q = rng.integers(0, c.vocab, 32).tolist()
res = F.Result(eng, 8 * 2048 + 32 + 32)


def timed(fn, reps=7, skip=2):
    ms = []
    for i in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if i >= skip:
            ms.append(e0.elapsed_time(e1))
    return statistics.median(ms)


out = {}
out["r0_ms"] = timed(lambda: eng.reprocess(store, q, ids, 0.0, res))
out["r15_ms"] = timed(lambda: eng.reprocess(store, q, ids, 0.15, res))
qs = []
for _ in range(3):
    eng.reprocess(store, q, ids, 0.15, res, timing=True)
    qs.append(res.timing()["question_ms"])
out["question_ms"] = statistics.median(qs)
dec = []
for _ in range(3):
    eng.reprocess(store, q, ids, 0.15, res)
    dec.append(timed(lambda: eng.decode(res, 16), reps=1, skip=0) / 16)
out["decode_ms_per_token"] = statistics.median(dec)
print(f"[{tag}] " + " ".join(f"{k}={v:.3f}" for k, v in out.items()), flush=True)
