"""Ad-hoc attention correctness sweep (kernel vs fp64 torch) over GQA group,
splits and row counts; prints the max error per case."""
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from tests.test_kernels_gpu import _attn_ref  # noqa: E402
from paper_2601_12904_b200 import _lib as L  # noqa: E402

dev = torch.device("cuda")
for (Hq, Hkv, dh) in [(8, 1, 128), (32, 8, 128), (4, 4, 64), (16, 2, 128)]:
    for T, M in [(600, 64), (600, 20), (1000, 40), (300, 33)]:
        for split in [0, 128, 256]:
            g = torch.Generator(device="cuda").manual_seed(T + M + split)
            q = torch.randn(M, Hq, dh, device=dev, generator=g).to(torch.bfloat16)
            k = torch.randn(T, Hkv, dh, device=dev, generator=g).to(torch.bfloat16)
            v = torch.randn(T, Hkv, dh, device=dev, generator=g).to(torch.bfloat16)
            rows = torch.sort(torch.randperm(T, device=dev, generator=g)[:M]).values.to(torch.int32)
            out = torch.empty(M, Hq, dh, device=dev, dtype=torch.bfloat16)
            L.check(L.lib.frag_kernel_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), rows.data_ptr(),
                                                out.data_ptr(), M, T, Hq, Hkv, dh, split, None))
            ref = _attn_ref(q, k, v, rows.cpu(), 1.0 / math.sqrt(dh))
            err = (out.double() - ref).abs()
            bad = (err.amax(dim=(1, 2)) > 2e-2).nonzero().flatten().tolist()
            print(f"Hq={Hq} Hkv={Hkv} dh={dh} T={T} M={M} split={split}: max err {err.max().item():.4f} bad tokens {bad[:8]}")
