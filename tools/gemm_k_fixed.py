"""CTA-pair GEMM at the O-projection tile grid (M = 2490, N = 4096: 220
192-wide tiles, 3 waves of 74 pairs) for several K: time = fixed + per-k-block
slope. The events bracket each host launch, so the fixed part includes the
host's launch latency (tensor-map encoding, launch) as well as the kernel's
prologue, pipeline fill and last-tile drain; tools/gemm2_trace.py separates
the device part. CUDA events, median of 20, bf16 store."""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_12904_b200 import _lib as L  # noqa: E402

M, N = 2490, 4096
pts = []
for K in (1024, 2048, 4096, 8192, 16384):
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    c = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    ts = []
    for i in range(23):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        L.check(L.lib.frag_kernel_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, 0, 192 | 0x40000, None))
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    us = statistics.median(ts)
    pts.append((K, us))
    print(f"K={K}: {us:.1f} us, {2.0 * M * N * K / us / 1e6:.0f} TFLOP/s", flush=True)
(k0, t0), (k1, t1) = pts[1], pts[-1]
slope = (t1 - t0) / (k1 - k0)
print(f"fixed {t0 - slope * k0:.1f} us + {slope * 64:.3f} us per 64-wide k-block (3 waves)")
