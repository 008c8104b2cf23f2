"""Device timeline of one graph-replayed 8B request (r = 0.15) from CUPTI
activity records (torch.profiler): per-kernel-class device time, the gaps
between consecutive kernels, and the request's span -- what the per-launch
event profile (which also counts launch gaps) cannot separate."""
import collections
import json
import os
import sys
import tempfile
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
qs = [rng.integers(0, c.vocab, 32).tolist() for _ in range(6)]
res = F.Result(eng, 8 * 2048 + 32)
ratio = float(sys.argv[1]) if len(sys.argv) > 1 else 0.15
for i in range(4):
    eng.reprocess(store, qs[i], ids, ratio, res)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

burst = int(os.environ.get("KT_BURST", "0"))  # requests run back to back before the traced one
# the same request in a device-timed loop (the bench's way): per-request time
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(10):
    eng.reprocess(store, qs[i % 4], ids, ratio, res)
e1.record()
torch.cuda.synchronize()
print(f"loop of 10 requests: {e0.elapsed_time(e1) / 10:.2f} ms per request (events around the loop)")
for i in range(burst):
    eng.reprocess(store, qs[i % 4], ids, ratio, res)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for i in range(3):
        eng.reprocess(store, qs[4 + (i % 2)], ids, ratio, res)
    torch.cuda.synchronize()
path = os.path.join(tempfile.mkdtemp(), "trace.json")
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
nk = len(ev) // 3
for j in range(3):  # three requests: their spans and the idle time between them
    a, b = ev[j * nk], ev[(j + 1) * nk - 1]
    nxt = f", idle before the next {ev[(j + 1) * nk]['ts'] - (b['ts'] + b['dur']):.0f} us" if j < 2 else ""
    print(f"request {j}: span {(b['ts'] + b['dur'] - a['ts']) / 1e3:.2f} ms{nxt}")
ev = ev[2 * nk:]
t0 = ev[0]["ts"]
span = ev[-1]["ts"] + ev[-1]["dur"] - t0
busy = collections.defaultdict(float)
cnt = collections.Counter()
for e in ev:
    n = e["name"].replace("void ", "").replace("(anonymous namespace)::", "").replace("fragk::", "").split("(")[0]
    busy[n] += e["dur"]
    cnt[n] += 1
# union of busy intervals per stream and overall
iv = sorted((e["ts"], e["ts"] + e["dur"]) for e in ev)
union, cur_s, cur_e = 0.0, iv[0][0], iv[0][1]
gaps = []
for s_, e_ in iv[1:]:
    if s_ > cur_e:
        union += cur_e - cur_s
        gaps.append(s_ - cur_e)
        cur_s, cur_e = s_, e_
    else:
        cur_e = max(cur_e, e_)
union += cur_e - cur_s
print(f"r={ratio} (after {burst} back-to-back requests): {len(ev)} kernels, span {span / 1e3:.2f} ms, busy (union) {union / 1e3:.2f} ms, "
      f"idle {(span - union) / 1e3:.2f} ms in {len(gaps)} gaps (largest {sorted(gaps)[-5:] if gaps else []} us)")
for n, d in sorted(busy.items(), key=lambda x: -x[1])[:14]:
    print(f"  {d / 1e3:8.3f} ms  {cnt[n]:4d}x  {n[:90]}")
