"""Per-CTA timeline of the one-M-tile (weight-streaming) GEMM at question-pass
shapes (M=32) from the kernel's FRAG_GEMM_TRACE globaltimer stamps (ns):
start -> PDL wait done -> first stage at the MMA -> last MMA issued ->
accumulator ready -> split partial written -> CTA end."""
import ctypes
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

path = os.path.join(tempfile.mkdtemp(), "gemm_trace.bin")
os.environ["FRAG_GEMM_TRACE"] = path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2601_12904_b200 import _lib as L  # noqa: E402

dev = torch.device("cuda")
M = int(sys.argv[1]) if len(sys.argv) > 1 else 32
shapes = {"qkv": (6144, 4096), "o": (4096, 4096), "gu": (28672, 4096), "down": (4096, 14336)}
names = ["start", "pdl", "first", "lastmma", "acc", "partial", "end"]
for name, (N, K) in shapes.items():
    b = torch.randn(N, K, device=dev).to(torch.bfloat16)
    a = torch.randn(M, K, device=dev).to(torch.bfloat16)
    c = torch.zeros(M, N, device=dev, dtype=torch.float32)
    if os.path.exists(path):
        os.remove(path)
    for _ in range(3):
        L.check(L.lib.frag_kernel_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, 2, 0, None))
    torch.cuda.synchronize()
    rec = np.fromfile(path, dtype=np.uint64).reshape(-1, 256, 8)[-1].astype(np.int64)
    live = rec[:, 0] > 0
    r = rec[live]
    t0 = r[:, 0].min()
    rel = {n: (r[:, i] - t0) / 1e3 for i, n in enumerate(names) if (r[:, i] > 0).any()}
    span = (r[:, 6].max() - t0) / 1e3
    mb = N * K * 2 / 1e6
    print(f"{name}: N={N} K={K} CTAs={int(live.sum())} span {span:.1f} us ({mb / span:.0f} GB/s weights)")
    for n, v in rel.items():
        v = v[v >= 0]
        print(f"   {n:8s} min {v.min():6.1f}  med {np.median(v):6.1f}  max {v.max():6.1f} us")
