"""r = 0 (one-pass Full Reuse) and r = 0.15 TTFT on the 8B 16k request,
graph-replayed, device-timed (median of 5)."""
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_12904_b200 import fusion as F  # noqa: E402

eng = F.Engine("llama3-8b", seed=1)
c = eng.cfg
store = F.ChunkKVStore(c)
rng = np.random.default_rng(0)
ids = [eng.preprocess_isolated(store, rng.integers(0, c.vocab, 2048).tolist()) for _ in range(8)]
q = rng.integers(0, c.vocab, 32).tolist()
res = F.Result(eng, 8 * 2048 + 32)
for r in (0.0, 0.15):
    ms = []
    for i in range(8):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.reprocess(store, q, ids, r, res)
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ms.append(e0.elapsed_time(e1))
    eng.reprocess(store, q, ids, r, res, timing=True)
    print(f"r={r}: {statistics.median(ms):.2f} ms  stages {({k: round(v, 2) for k, v in res.timing().items()})}")
