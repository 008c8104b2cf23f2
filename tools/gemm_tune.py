"""Time the tcgen05 GEMM per (shape, BN, tail split) with CUDA events (inputs
larger than L2 are not needed for a shape sweep; each config repeats 20x)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_12904_b200 import _lib as L  # noqa: E402

dev = torch.device("cuda")
shapes = {"qkv": (6144, 4096), "o": (4096, 4096), "gu": (28672, 4096), "down": (4096, 14336)}
Ms = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["2490", "16416", "32"])]
for M in Ms:
    for name, (N, K) in shapes.items():
        a = torch.randn(M, K, device=dev).to(torch.bfloat16)
        b = torch.randn(N, K, device=dev).to(torch.bfloat16)
        c = torch.zeros(M, N, device=dev, dtype=torch.float32)
        res = []
        for bn in (0, 128, 256, 1128, 1192, 1256):
            for tail in ((0,) if bn == 0 else (0, 1)):
                flags = (bn | (tail << 16) if bn < 1000 else (bn - 1000) | 0x40000 | (tail << 16)) if bn else 0
                try:
                    for _ in range(3):
                        L.check(L.lib.frag_kernel_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, 2, flags, None))
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(20):
                        L.check(L.lib.frag_kernel_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, 2, flags, None))
                    e1.record()
                    torch.cuda.synchronize()
                    us = e0.elapsed_time(e1) / 20 * 1e3
                    nm = (f"pair{bn - 1000}" if bn > 1000 else f"bn{bn or 'auto'}") + ("+tail" if tail else "")
                    res.append((nm, round(us, 1), round(2 * M * N * K / us / 1e6, 0)))
                except Exception as ex:
                    res.append((f"bn{bn}", "err", str(ex)[:40]))
        print(M, name, res, flush=True)
