"""compute-sanitizer driver: the dh=128 sparse-Q attention kernel at two shapes (tools/sanitize.sh)."""
import sys, torch
sys.path.insert(0, '.')
from paper_2601_12904_b200 import _lib as L
dev = torch.device("cuda")
for (Hq, Hkv, dh, T, M) in [(32, 8, 128, 1500, 150), (32, 8, 128, 700, 20)]:
    g = torch.Generator(device="cuda").manual_seed(T + M)
    q = torch.randn(M, Hq, dh, device=dev, generator=g).to(torch.bfloat16)
    k = torch.randn(T, Hkv, dh, device=dev, generator=g).to(torch.bfloat16)
    v = torch.randn(T, Hkv, dh, device=dev, generator=g).to(torch.bfloat16)
    rows = torch.sort(torch.randperm(T, device=dev, generator=g)[:M]).values.to(torch.int32)
    out = torch.empty(M, Hq, dh, device=dev, dtype=torch.bfloat16)
    L.check(L.lib.frag_kernel_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), rows.data_ptr(), out.data_ptr(), M, T, Hq, Hkv, dh, 0, None))
    torch.cuda.synchronize()
print("ok")
