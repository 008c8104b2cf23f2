"""compute-sanitizer driver: one tiny end-to-end reprocess (tools/sanitize.sh)."""
import sys, numpy as np
sys.path.insert(0, '.')
from paper_2601_12904_b200 import fusion as F
eng = F.Engine("tiny", seed=1234)
store = F.ChunkKVStore(eng.cfg)
rng = np.random.default_rng(6)
chunks = [rng.integers(0, eng.cfg.vocab, 256).tolist() for _ in range(4)]
ids = [eng.preprocess_isolated(store, c) for c in chunks]
question = rng.integers(0, eng.cfg.vocab, 32).tolist()
res = F.Result(eng, 4 * 256 + 32)
eng.reprocess(store, question, ids, 0.15, res)
print("ok", res.logits()[0, :3])
