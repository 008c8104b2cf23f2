"""Host-side cost of one reprocess request: wall time of the synchronous call
vs the device time of the same request (CUDA events), llama3-8b bench shape."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_12904_b200 import fusion as F  # noqa: E402

eng = F.Engine(sys.argv[1] if len(sys.argv) > 1 else "llama3-8b", seed=1)
c = eng.cfg
store = F.ChunkKVStore(c)
rng = np.random.default_rng(0)
ids = [eng.preprocess_isolated(store, rng.integers(0, c.vocab, 2048).astype(np.int32)) for _ in range(8)]
res = F.Result(eng, 8 * 2048 + 32)
q = [torch.from_numpy(rng.integers(0, c.vocab, 32).astype(np.int32)).cuda() for _ in range(40)]
s = torch.cuda.current_stream()
for i in range(5):
    eng.reprocess(store, None, ids, 0.15, res, stream=s, question_dev_ptr=q[i].data_ptr(), n_question=32,
                  logits_on_device=True)
torch.cuda.synchronize()
walls, devs, preps = [], [], []
for i in range(20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(s)
    eng.reprocess(store, None, ids, 0.15, res, stream=s, question_dev_ptr=q[i].data_ptr(), n_question=32,
                  logits_on_device=True)
    e1.record(s)
    torch.cuda.synchronize()
    walls.append((time.perf_counter() - t0) * 1e3)
    preps.append(res.timing()["host_prep_ms"])
    devs.append(e0.elapsed_time(e1))
print(f"wall {np.median(walls):.3f} ms  device(e0..e1) {np.median(devs):.3f} ms  host prep {np.median(preps):.3f} ms")
walls = []
for i in range(10):
    t0 = time.perf_counter()
    eng.reprocess(store, None, ids, 0.15, res, stream=s, question_dev_ptr=q[i].data_ptr(), n_question=32,
                  logits_on_device=True, timing=True)
    walls.append((time.perf_counter() - t0) * 1e3)
    devs.append(res.timing()["total_ms"])
print(f"eager+timing: wall {np.median(walls):.3f} ms  total_ms {np.median(devs[-10:]):.3f}")
eng.reprocess(store, None, ids, 0.15, res, stream=s, question_dev_ptr=q[0].data_ptr(), n_question=32,
              logits_on_device=True, timing=True)
print("stages", res.timing())
