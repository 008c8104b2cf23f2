"""Per-op timeline of the weight-streaming GEMM chain (gemm_chain.cu) inside
one 8B question pass, from its FRAG_CHAIN_TRACE globaltimer stamps (ns):
per op and CTA [A operand ready, all loads issued, first accumulator ready,
all units published, (split ops) partial written, all siblings arrived]; prints min / median / max over CTAs relative to the
chain's first stamp, for one mid-depth layer."""
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

path = os.path.join(tempfile.mkdtemp(), "chain_trace.bin")
os.environ["FRAG_CHAIN_TRACE"] = path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_12904_b200 import fusion as F  # noqa: E402

eng = F.Engine("llama3-8b", seed=1234)
store = F.ChunkKVStore(eng.cfg)
rng = np.random.default_rng(0)
ids = [eng.preprocess_isolated(store, rng.integers(0, eng.cfg.vocab, 2048).tolist()) for _ in range(8)]
question = rng.integers(0, eng.cfg.vocab, 32).tolist()
res = F.Result(eng, 8 * 2048 + 32)
if os.path.exists(path):
    os.remove(path)
eng.reprocess(store, question, ids, 0.15, res)  # first request of the shape: eager
sms = 148
rec = np.fromfile(path, dtype=np.uint64).reshape(-1, sms, 4, 8).astype(np.int64)
print(f"{len(rec)} chain launches recorded")
names = ["O", "gate/up", "down", "QKV(next)"]
for li in (1, len(rec) // 2):
    r = rec[li]
    t0 = r[:, :, :4][r[:, :, :4] > 0].min()
    print(f"-- chain {li}: span {(r.max() - t0) / 1e3:.1f} us")
    for o in range(4):
        x = r[:, o, :]
        x = x[x[:, 3] > 0]
        if len(x) == 0:
            continue
        cols = []
        for k in range(6):
            v = (x[:, k] - t0) / 1e3
            cols.append(f"{v.min():6.1f}/{np.median(v):6.1f}/{v.max():6.1f}")
        print(f"{names[o]:>10} ({len(x):3d} CTAs)  A-ready {cols[0]}  issued {cols[1]}  first-acc {cols[2]}  "
              f"published {cols[3]}")
        if (x[:, 4] > 0).all():
            print(f"{'':>10}  split-K fixup: partial written {cols[4]}  all siblings arrived {cols[5]}")
