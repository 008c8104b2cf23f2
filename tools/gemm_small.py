"""Small-M (question pass) GEMM sweep: BN x split-K, timed over back-to-back
launches (no per-call sync). HBM-bound: reports weight GB/s."""
import ctypes
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_12904_b200 import _lib as L  # noqa: E402

dev = torch.device("cuda")
M = int(sys.argv[1]) if len(sys.argv) > 1 else 32
shapes = {"tiny": (128, 64), "small": (1024, 1024), "qkv": (6144, 4096), "o": (4096, 4096), "gu": (28672, 4096), "down": (4096, 14336),
          "lm": (128256, 4096)}
only = sys.argv[2].split(",") if len(sys.argv) > 2 else None
for name, (N, K) in shapes.items():
    if only and name not in only:
        continue
    # several weight copies so consecutive launches stream from HBM, not L2
    nb = max(2, int(400e6 // (N * K * 2)))
    bs = [torch.randn(N, K, device=dev).to(torch.bfloat16) for _ in range(nb)]
    a = torch.randn(M, K, device=dev).to(torch.bfloat16)
    c = torch.zeros(M, N, device=dev, dtype=torch.float32)
    res = []
    for bn in (0, 128, 4128):
        for sp in ((0,) if bn == 0 else (1, 2, 3, 4, 6, 8)):
            if bn and N % (bn % 1000):
                continue
            fl = 128 | 0x8000000 if bn == 4128 else bn
            flags = (fl | (sp << 20) | 0x20000 | 0x80000) if bn else 0x80000
            try:
                st = torch.cuda.Stream()
                with torch.cuda.stream(st):
                    for i in range(3):
                        L.check(L.lib.frag_kernel_gemm(a.data_ptr(), bs[i % nb].data_ptr(), c.data_ptr(), M, N, K,
                                                       2, flags, ctypes.c_void_p(st.cuda_stream)))
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=st):
                    for i in range(30):
                        L.check(L.lib.frag_kernel_gemm(a.data_ptr(), bs[i % nb].data_ptr(), c.data_ptr(), M, N, K,
                                                       2, flags, ctypes.c_void_p(st.cuda_stream)))
                g.replay()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) / 30 * 1e3
                nm = {4128: "bn128full_"}.get(bn, f"bn{bn or 'auto'}")
                res.append((f"{nm}s{sp}", round(us, 1), round(N * K * 2 / us / 1e3)))
            except Exception as ex:
                res.append((f"bn{bn}s{sp}", "err", str(ex)[:50]))
    res.sort(key=lambda x: x[1] if isinstance(x[1], float) else 1e9)
    print(M, name, f"ideal {N * K * 2 / 6.45e6:.1f}us", res[:10], flush=True)
