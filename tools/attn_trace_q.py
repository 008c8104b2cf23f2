"""Per-tile timeline of the question-pass attention (DUAL kernel, one query
tile per CTA, split-KV) inside a real 8B request: CTA 0 of each launch --
S issue / S ready / P done / PV issue per key tile and slot (SM cycles from
the first S issue). FRAG_ATTN_TRACE, eager launches."""
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

path = os.path.join(tempfile.mkdtemp(), "attn_trace.bin")
os.environ["FRAG_ATTN_TRACE"] = path
os.environ["FRAG_GRAPHS"] = "0"
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_12904_b200 import fusion as F  # noqa: E402

eng = F.Engine("llama3-8b", seed=1)
c = eng.cfg
store = F.ChunkKVStore(c)
rng = np.random.default_rng(0)
ids = [eng.preprocess_isolated(store, rng.integers(0, c.vocab, 2048).tolist()) for _ in range(8)]
q = rng.integers(0, c.vocab, 32).tolist()
res = F.Result(eng, 8 * 2048 + 32)
eng.reprocess(store, q, ids, 0.15, res)
res.sync()
rec = np.fromfile(path, dtype=np.uint64).reshape(-1, 4, 256, 4).astype(np.int64)
shown = 0
for li, r in enumerate(rec):
    a = r[:2].reshape(-1)  # [(t * 256 + j) * 4 + k]
    tiles = [[a[((t * 256 + j) * 4):((t * 256 + j) * 4 + 4)] for j in range(256)] for t in range(2)]
    n = sum(1 for j in range(256) if tiles[0][j][2] > 0)
    if n == 0 or n > 40:
        continue
    t0 = min(tiles[t][0][2] for t in range(2) if tiles[t][0][2] > 0)
    print(f"launch {li}: {n} tiles")
    for j in range(n):
        row = []
        for t in range(2):
            s_rdy, p_done, s_iss, pv_iss = (int(x) - t0 if x else -1 for x in tiles[t][j])
            row.append(f"slot{t}: S iss {s_iss:6d} rdy {s_rdy:6d} P {p_done:6d} PV iss {pv_iss:6d}")
        print(f"  tile {j}: " + " | ".join(row))
    shown += 1
    if shown >= 2:
        break
