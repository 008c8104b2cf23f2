"""Timeline of the weight-streaming GEMM chain (gemm_chain.cu) in the 8B
question pass, graph-replayed, from its device-side globaltimer ring
(FRAG_CHAIN_TRACE=1; read back with frag_debug_chain_timeline).

Per CTA and launch: entry, PDL wait done, exit; per op: A operand ready, all
loads issued, first accumulator, all units published, (split ops) partial
written, all siblings arrived. Prints one mid-depth layer of the last
replayed request (min / median / max over CTAs, µs from the chain's first
entry) and the gaps between consecutive chains (the layer's attention kernel
+ kernel-boundary costs)."""
import ctypes
import os
import sys
from pathlib import Path

import numpy as np

os.environ["FRAG_CHAIN_TRACE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_12904_b200 import _lib as L  # noqa: E402
from paper_2601_12904_b200 import fusion as F  # noqa: E402

LAUNCHES, CTAS, SLOTS = 64, 160, 40
eng = F.Engine("llama3-8b", seed=1234)
store = F.ChunkKVStore(eng.cfg)
rng = np.random.default_rng(0)
ids = [eng.preprocess_isolated(store, rng.integers(0, eng.cfg.vocab, 2048).tolist()) for _ in range(8)]
question = rng.integers(0, eng.cfg.vocab, 32).tolist()
res = F.Result(eng, 8 * 2048 + 32)
for _ in range(3):  # eager, capture, replay: the ring keeps the last 64 chain launches
    eng.reprocess(store, question, ids, 0.15, res)
buf = np.zeros((LAUNCHES, CTAS, SLOTS), dtype=np.uint64)
fn = L.lib.frag_debug_chain_timeline
fn.restype = ctypes.c_int
seq = fn(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), LAUNCHES)
order = [(seq - 31 + i) % LAUNCHES for i in range(31)]  # the last request's question-pass chains
rec = buf[order].astype(np.int64)
sms = int((rec[0, :, 0] > 0).sum())
rec = rec[:, :sms]
names = ["O", "gate/up", "down", "QKV(next)"]
kn = ["A ready", "issued", "first acc", "published", "partial written", "siblings arrived"]


def fmt(v):
    return f"{v.min():6.1f}/{np.median(v):6.1f}/{v.max():6.1f}"


li = 15
r = rec[li]
t0 = r[:, 0].min()
print(f"sequence {seq}; chain {li} of the last question pass ({sms} CTAs), µs from the first CTA entry")
print(f"  entry {fmt((r[:, 0] - t0) / 1e3)}  PDL wait done {fmt((r[:, 1] - t0) / 1e3)}  exit {fmt((r[:, 2] - t0) / 1e3)}")
for o in range(4):
    x = r[:, 8 + 8 * o: 8 + 8 * o + 6]
    x = x[x[:, 3] > 0]
    if len(x) == 0:
        continue
    cols = [f"{kn[k]} {fmt((x[:, k] - t0) / 1e3)}" for k in range(6) if (x[:, k] > 0).all()]
    print(f"  {names[o]:>10} ({len(x):3d} CTAs)  " + "  ".join(cols))
entry = rec[:, :, 0].min(axis=1)
pdl = rec[:, :, 1].min(axis=1)
exit_ = rec[:, :, 2].max(axis=1)
span = (exit_ - entry) / 1e3
gap = (entry[1:] - exit_[:-1]) / 1e3
wait = (pdl - entry) / 1e3
print(f"chain span (first entry -> last exit) median {np.median(span):.1f} us; first entry -> first PDL-wait "
      f"return median {np.median(wait):.1f} us")
print(f"last exit of chain l -> first entry of chain l+1 (attention kernel + boundaries): median "
      f"{np.median(gap):.1f} us, min {gap.min():.1f}, max {gap.max():.1f}")
print(f"question pass chains: {(exit_[-1] - entry[0]) / 1e3:.0f} us for {len(rec)} layers")
