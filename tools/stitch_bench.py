"""K1 (stitch) time inside the 8B request: the per-stage timing of a few
requests (median stitch_ms) and the bytes it moves (K only with shared V
pages, K + V with a private V)."""
import statistics
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_12904_b200 import fusion as F  # noqa: E402

eng = F.Engine("llama3-8b", seed=1)
c = eng.cfg
store = F.ChunkKVStore(c)
rng = np.random.default_rng(0)
ids = [eng.preprocess_isolated(store, rng.integers(0, c.vocab, 2048).tolist()) for _ in range(8)]
q = rng.integers(0, c.vocab, 32).tolist()
res = F.Result(eng, 8 * 2048 + 32)
for shared in (True, False):
    F.set_shared_v(shared)
    ms = []
    for i in range(6):
        eng.reprocess(store, q, ids, 0.15, res, timing=True)
        if i >= 2:
            ms.append(res.timing()["stitch_ms"])
    gb = (2 if shared else 4) * c.layers * 8 * 2048 * c.n_kv_heads * c.head_dim * 2 / 1e9
    t = statistics.median(ms)
    print(f"shared_v={shared}: stitch {t:.3f} ms, {gb:.2f} GB -> {gb / t:.2f} TB/s")
