"""compute-sanitizer driver for the round-2 GEMM paths (tools/sanitize.sh):
the one-M-tile split-K over strided k-blocks (the question pass's down
projection shape), a 224-wide CTA-pair tile with a partial last N tile, and
an 8B-width 2-layer reprocess whose question pass runs the GEMM chain with
split-major units and the strided down projection."""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2601_12904_b200 import _lib as L  # noqa: E402
from paper_2601_12904_b200 import fusion as F  # noqa: E402


def gemm(M, N, K, epi, flags):
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    c = torch.zeros(M, N, device="cuda", dtype=torch.float32)
    L.check(L.lib.frag_kernel_gemm(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, epi, flags, None))
    torch.cuda.synchronize()
    ref = a.float() @ b.float().T
    return float((c - ref).abs().max() / ref.abs().max())


print("strided split-K", gemm(32, 4096, 14336, 1, 0))
print("224-wide pair tiles", gemm(600, 1472, 512, 1, 224 | 0x40000))
cfg = F.preset("llama3-8b")
cfg.layers = 2
eng = F.Engine(cfg, seed=7)
store = F.ChunkKVStore(eng.cfg)
rng = np.random.default_rng(8)
ids = [eng.preprocess_isolated(store, rng.integers(0, cfg.vocab, 256).tolist()) for _ in range(2)]
res = F.Result(eng, 2 * 256 + 32)
eng.reprocess(store, rng.integers(0, cfg.vocab, 32).tolist(), ids, 0.15, res)
print("ok", res.logits()[0, :3])
