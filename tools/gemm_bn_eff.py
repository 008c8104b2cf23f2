import statistics, sys, torch
sys.path.insert(0, "/root/repo")
from paper_2601_12904_b200 import _lib as L
import sys as _s
# A (M x K bf16) must stay L2-resident, or the narrower tiles' extra A
# re-reads from DRAM confound the comparison: M = 2490 (20 MB of A)
M, N, K = 2490, 26880, 4096   # 26880 = 105*256 = 120*224 = 140*192 = 210*128
a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
c = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
for bn in (256, 224, 192, 128):
    ts = []
    for i in range(13):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        L.check(L.lib.frag_kernel_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, 0, bn | 0x40000, None))
        e1.record(); torch.cuda.synchronize()
        if i >= 3: ts.append(e0.elapsed_time(e1) * 1e3)
    us = statistics.median(ts)
    tiles = ((M + 255) // 256) * ((N + bn - 1) // bn)
    print(f"BN={bn}: {us:.1f} us {2.0*M*N*K/us/1e6:.0f} TFLOP/s, {tiles} tiles = {tiles/74:.2f} waves", flush=True)
