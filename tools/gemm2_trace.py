"""Per-CTA timeline of the CTA-pair GEMM (FRAG_GEMM2_TRACE globaltimer stamps)
at the sparse-pass shapes, bf16 store, one traced launch after warm-ups:
entry, prologue done, PDL wait, and per tile first MMA / last MMA issued /
accumulator seen by the epilogue / epilogue done (µs from the earliest entry,
min / median / max over CTAs)."""
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

path = os.path.join(tempfile.mkdtemp(), "g2.bin")
os.environ["FRAG_GEMM2_TRACE"] = path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2601_12904_b200 import _lib as L  # noqa: E402

for (M, N, K, name) in [(2490, 4096, 4096, "O"), (2490, 6144, 4096, "QKV"), (2490, 28672, 4096, "gate/up")]:
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    c = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    if os.path.exists(path):
        os.remove(path)
    for _ in range(4):
        L.check(L.lib.frag_kernel_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, 0, 0, None))
    torch.cuda.synchronize()
    rec = np.fromfile(path, dtype=np.uint64).reshape(-1, 160, 32).astype(np.int64)[-1]
    live = rec[:, 0] > 0
    t0 = rec[live, 0].min()
    us = lambda col: (rec[live, col][rec[live, col] > 0] - t0) / 1e3  # noqa: E731

    def st(col):
        v = us(col)
        return f"{v.min():6.1f}/{np.median(v):6.1f}/{v.max():6.1f}" if len(v) else "   -"
    print(f"{name} M={M} N={N} K={K}: entry {st(0)}  prologue {st(1)}  pdl {st(2)}  exit {st(30)}")
    for t in range(4):
        print(f"   tile {t}: first MMA {st(4 + 4 * t)}  last MMA {st(5 + 4 * t)}  acc seen {st(6 + 4 * t)}  "
              f"epilogue done {st(7 + 4 * t)}")
