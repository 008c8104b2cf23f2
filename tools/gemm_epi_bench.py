"""CTA-pair GEMM at the sparse-pass O / QKV / down shapes with different
epilogues (0 bf16 store, 1 fp32 store, 2 residual add): is the epilogue or the
main loop the limit? CUDA events, median of 20. argv: flags (default auto)."""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_12904_b200 import _lib as L  # noqa: E402

flags = int(sys.argv[1], 0) if len(sys.argv) > 1 else 0
for (M, N, K, name) in [(2490, 4096, 4096, "O"), (2490, 6144, 4096, "QKV"), (2490, 4096, 14336, "down"),
                        (2490, 28672, 4096, "gate/up")]:
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    out = {}
    for epi in (0, 1, 2):
        c = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16 if epi == 0 else torch.float32)
        ts = []
        for i in range(23):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            L.check(L.lib.frag_kernel_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, epi, flags, None))
            e1.record()
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(e0.elapsed_time(e1) * 1e3)
        us = statistics.median(ts)
        out[epi] = f"{us:.1f} us ({2.0 * M * N * K / us / 1e6:.0f} TFLOP/s)"
    print(name, out, flush=True)
