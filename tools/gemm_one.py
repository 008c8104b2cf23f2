"""Run one GEMM config a few times (for ncu): argv M N K flags [reps]."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_12904_b200 import _lib as L  # noqa: E402

M, N, K, flags = (int(x, 0) for x in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
c = torch.zeros(M, N, device="cuda", dtype=torch.float32)
for _ in range(reps):
    L.check(L.lib.frag_kernel_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, 2, flags, None))
torch.cuda.synchronize()
