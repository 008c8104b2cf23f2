"""Greedy decode ms/token after an 8B 16k reprocess, repeated (shared V pages
on / off): device time per token over 16-token runs."""
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
res = F.Result(eng, 8 * 2048 + 32 + 32)
for shared in (True, False, True):
    F.set_shared_v(shared)
    out = []
    for rep in range(4):
        eng.reprocess(store, q, ids, 0.15, res)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.decode(res, 16)
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) / 15)
    print(f"shared_v={shared}: decode ms/token {[round(x, 2) for x in out]}")
