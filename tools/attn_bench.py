"""Time the sparse-Q attention kernel alone (CUDA events, 20 reps) at the 8B
sparse-pass shape: M query rows at sorted random positions of a T-key cache,
Hq=32/Hkv=8/dh=128; FLOP = 4*Hq*dh*sum(p_i). Optional argv: M T."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_12904_b200 import _lib as L  # noqa: E402

dev = torch.device("cuda")
M = int(sys.argv[1]) if len(sys.argv) > 1 else 2490
T = int(sys.argv[2]) if len(sys.argv) > 2 else 16416
Hq, Hkv, dh = 32, 8, 128
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(M, Hq, dh, device=dev, generator=g).to(torch.bfloat16)
k = torch.randn(T, Hkv, dh, device=dev, generator=g).to(torch.bfloat16)
v = torch.randn(T, Hkv, dh, device=dev, generator=g).to(torch.bfloat16)
rows = torch.sort(torch.randperm(T, device=dev, generator=g)[:M]).values.to(torch.int32)
out = torch.empty(M, Hq, dh, device=dev, dtype=torch.bfloat16)
flop = 4.0 * Hq * dh * float((rows.double() + 1).sum())


def run():
    L.check(L.lib.frag_kernel_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), rows.data_ptr(), out.data_ptr(),
                                        M, T, Hq, Hkv, dh, 0, None))


for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    run()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 20 * 1e3
print(f"attn M={M} T={T}: {us:.1f} us  {flop / us / 1e6:.0f} TFLOP/s")
