"""r = 0 TTFT and decode ms/token on the 8B 16k request before and after the
same Result ran a full prefill (bench.py's order of legs), device-timed."""
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_12904_b200 import _lib as L  # noqa: E402
from paper_2601_12904_b200 import fusion as F  # noqa: E402

L.lib.frag_debug_alloc_epoch.restype = __import__("ctypes").c_ulonglong

eng = F.Engine("llama3-8b", seed=1)
c = eng.cfg
store = F.ChunkKVStore(c)
rng = np.random.default_rng(0)
chunks = [rng.integers(0, c.vocab, 2048).tolist() for _ in range(8)]
ids = [eng.preprocess_isolated(store, ch) for ch in chunks]
qs = [rng.integers(0, c.vocab, 32).tolist() for _ in range(8)]
res = F.Result(eng, 8 * 2048 + 32 + 32)


eps = []


def med(fn, n=5):
    out = []
    for i in range(n + 3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn(i)
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            out.append(e0.elapsed_time(e1))
        eps.append(L.lib.frag_debug_alloc_epoch())
    return round(statistics.median(out), 3)


def dec():
    eng.reprocess(store, qs[0], ids, 0.15, res)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.decode(res, 16)
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / 16, 3)


print("fresh: r0", med(lambda i: eng.reprocess(store, qs[i % 8], ids, 0.0, res)),
      "r15", med(lambda i: eng.reprocess(store, qs[i % 8], ids, 0.15, res)), "decode", dec(), "mem", res.memory(), flush=True)
toks = np.concatenate(chunks + [qs[0]])
eng.full_prefill(toks, res)
torch.cuda.synchronize()
print("after full prefill: r0", med(lambda i: eng.reprocess(store, qs[i % 8], ids, 0.0, res)),
      "r15", med(lambda i: eng.reprocess(store, qs[i % 8], ids, 0.15, res)), "decode", dec(), "mem", res.memory(), flush=True)
res2 = F.Result(eng, 8 * 2048 + 32 + 32)
print("new result: r0", med(lambda i: eng.reprocess(store, qs[i % 8], ids, 0.0, res2)), flush=True)
print("alloc epoch after each timed call:", eps)
