"""Per-slice timeline of the Q-in-TMEM attention kernel (CTA 0, softmax warp 0):
S ready, after the S load, after the row-max exchange, after the exps, P done
(SM cycles, medians over slices), and the MMA warp's S / PV issue times."""
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
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(M, Hq, dh, device=dev, generator=g).to(torch.bfloat16)
k = torch.randn(T, Hkv, dh, device=dev, generator=g).to(torch.bfloat16)
v = torch.randn(T, Hkv, dh, device=dev, generator=g).to(torch.bfloat16)
rows = torch.sort(torch.randperm(T, device=dev, generator=g)[:M]).values.to(torch.int32)
out = torch.empty(M, Hq, dh, device=dev, dtype=torch.bfloat16)
for _ in range(3):
    L.check(L.lib.frag_kernel_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), rows.data_ptr(), out.data_ptr(),
                                        M, T, Hq, Hkv, dh, 0, None))
torch.cuda.synchronize()
rec = np.fromfile(path, dtype=np.uint64).reshape(-1, 4, 256, 4)[-1].astype(np.int64)
a, b = rec[0], rec[1]
n = int((a[:, 0] > 0).sum())
s_ready, p_done, s_iss, pv_iss = (a[:n, i] for i in range(4))
ld, mx, ex, p_last = (b[:n, i] for i in range(4))
med = lambda x: float(np.median(x))  # noqa: E731
print(f"slices {n}; period {med(np.diff(s_ready)):.0f} cyc per 128 keys")
print(f"  S ready -> S loaded {med(ld - s_ready):.0f}; -> max exchanged {med(mx - ld):.0f}; "
      f"-> exps done {med(ex - mx):.0f}; -> P done {med(p_done - ex):.0f}; P done -> next S ready "
      f"{med(s_ready[1:] - p_done[:-1]):.0f}")
print(f"  last of the 16 softmax warps done {med(p_last - p_done):.0f} after warp 0; -> PV issue "
      f"{med(pv_iss - p_last):.0f}")
print(f"  P done -> PV issue {med(pv_iss - p_done):.0f}; S(u+2) issue - S(u+2) ready "
      f"{med(s_ready[2:] - s_iss[2:]):.0f}")
