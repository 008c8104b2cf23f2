"""CTA-pair GEMM tile width at many waves: the same GEMM with BN forced to 256 /
224 / 192 / 128 (bf16 store, CUDA events, median of 10). A (M x K bf16) stays
L2-resident (M = 2490: 20 MB), or the narrower tiles' extra A re-reads from
DRAM would confound the comparison. Results: profiles/gemm_tile_width_r02.md."""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_12904_b200 import _lib as L  # noqa: E402

M, N, K = 2490, 26880, 4096  # 26880 = 105 x 256 = 120 x 224 = 140 x 192 = 210 x 128
a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
c = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
for bn in (256, 224, 192, 128):
    ts = []
    for i in range(13):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        L.check(L.lib.frag_kernel_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, 0, bn | 0x40000, None))
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    us = statistics.median(ts)
    tiles = ((M + 255) // 256) * ((N + bn - 1) // bn)
    print(f"BN={bn}: {us:.1f} us {2.0 * M * N * K / us / 1e6:.0f} TFLOP/s, {tiles} tiles = {tiles / 74:.2f} waves",
          flush=True)
