"""CTA-pair GEMM time vs K and epilogue (0: bf16 store, 1: fp32 store, 2: fp32
C += acc) at the sparse-pass M: the K -> 0 intercept is the per-launch cost
the epilogue adds (events, 20 launches)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_12904_b200 import _lib as L  # noqa: E402

for (M, N) in [(2490, 4096), (2490, 6144)]:
    for K in [1024, 4096, 14336]:
        a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
        c = torch.zeros(M, N, device="cuda", dtype=torch.float32)
        row = []
        for epi in (0, 1, 2):
            for _ in range(3):
                L.check(L.lib.frag_kernel_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, epi, 0, None))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(20):
                L.check(L.lib.frag_kernel_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, epi, 0, None))
            e1.record()
            torch.cuda.synchronize()
            row.append(e0.elapsed_time(e1) / 20 * 1e3)
        print(f"M={M} N={N} K={K}: epi0 {row[0]:.1f}  epi1 {row[1]:.1f}  epi2 {row[2]:.1f} us "
              f"({2 * M * N * K / row[0] / 1e6:.0f} TFLOP/s with epi0)")
