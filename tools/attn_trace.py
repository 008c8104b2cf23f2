"""Timeline of one attention CTA (the first-dispatched, longest q-block) at the
8B sparse-pass shape (argv[1] = "question": the 32-row question pass, split-KV
DUAL kernel, the CTA of split 0), from the kernel's FRAG_ATTN_TRACE clock64 stamps:
per key tile j and query tile t: S ready (softmax wakes), P done (softmax
arrives), S issue and PV issue times in the MMA warp. Prints per-tile
softmax durations, S waits and the MMA issue gaps (SM cycles)."""
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

path = os.path.join(tempfile.mkdtemp(), "attn_trace.bin")
os.environ["FRAG_ATTN_TRACE"] = path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2601_12904_b200 import _lib as L  # noqa: E402

dev = torch.device("cuda")
M, T, Hq, Hkv, dh = 2490, 16416, 32, 8, 128
question = len(sys.argv) > 1 and sys.argv[1] == "question"  # 32 rows at the end, split-KV (DUAL kernel)
split = 0
if question:
    M, split = 32, 1024
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(M, Hq, dh, device=dev, generator=g).to(torch.bfloat16)
k = torch.randn(T, Hkv, dh, device=dev, generator=g).to(torch.bfloat16)
v = torch.randn(T, Hkv, dh, device=dev, generator=g).to(torch.bfloat16)
rows = torch.sort(torch.randperm(T, device=dev, generator=g)[:M]).values.to(torch.int32)
if question:
    rows = torch.arange(T - M, T, device=dev, dtype=torch.int32)
out = torch.empty(M, Hq, dh, device=dev, dtype=torch.bfloat16)
for _ in range(3):
    L.check(L.lib.frag_kernel_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), rows.data_ptr(), out.data_ptr(),
                                        M, T, Hq, Hkv, dh, split, None))
torch.cuda.synchronize()
rec = np.fromfile(path, dtype=np.uint64).reshape(-1, 2, 256, 4)[-1].astype(np.int64)
base = rec[rec > 0].min()
n = int((rec[0, :, 0] > 0).sum())
print(f"tiles {n}")
s_ready, p_done, s_iss, pv_iss = (rec[:, :n, i] - base for i in range(4))
for t in range(2):
    sm = p_done[t] - s_ready[t]
    wait = s_ready[t, 1:] - p_done[t, :-1]
    print(f"tile {t}: softmax med {np.median(sm):.0f} cyc (p10 {np.percentile(sm, 10):.0f} p90 "
          f"{np.percentile(sm, 90):.0f}); S wait after P med {np.median(wait):.0f}")
    print(f"   P done -> PV issue med {np.median(pv_iss[t] - p_done[t]):.0f}; "
          f"PV issue -> next S ready med {np.median(s_ready[t, 1:] - pv_iss[t, :-1]):.0f}")
per_tile = (p_done[:, -1].max() - s_ready[:, 0].min()) / n
print(f"period per key tile (both q tiles): {per_tile:.0f} cyc; ideal tensor 2048")
for j in range(8, 14):
    print(j, [int(x) for x in (s_ready[0, j], p_done[0, j], pv_iss[0, j], s_ready[1, j], p_done[1, j], pv_iss[1, j])])
