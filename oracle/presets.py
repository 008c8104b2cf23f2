"""Model shapes of the bench workloads as plain data.

TEST INFRASTRUCTURE: read by the oracle-side legs of bench.py (the
`--impl reference` arm and `cpu_baseline`) so that those legs never import
the product package (and thereby map libfrag.so into the reference process).
The product's own presets live in libfrag.so (`frag_model_preset`, capi.cpp);
tests/test_capi_cpu.py keeps the two tables equal.
"""
from __future__ import annotations

PRESETS = {
    # layers, d_model, n_heads, n_kv_heads, head_dim, ffn_dim, vocab, rope_base, norm_eps
    "tiny": dict(layers=2, d_model=256, n_heads=4, n_kv_heads=4, head_dim=64, ffn_dim=1024, vocab=256,
                 rope_base=1e4, norm_eps=1e-5),
    "llama3-8b": dict(layers=32, d_model=4096, n_heads=32, n_kv_heads=8, head_dim=128, ffn_dim=14336,
                      vocab=128256, rope_base=5e5, norm_eps=1e-5),
    "mistral-7b": dict(layers=32, d_model=4096, n_heads=32, n_kv_heads=8, head_dim=128, ffn_dim=14336,
                       vocab=32768, rope_base=1e6, norm_eps=1e-5),
    "llama3-70b": dict(layers=80, d_model=8192, n_heads=64, n_kv_heads=8, head_dim=128, ffn_dim=28672,
                       vocab=128256, rope_base=5e5, norm_eps=1e-5),
}


def preset(name: str) -> dict:
    return dict(PRESETS[name])
