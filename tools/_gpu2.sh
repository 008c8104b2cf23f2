for p in 0 4; do FRAG_ATTN_POLY=$p python tools/attn_bench.py; FRAG_ATTN_POLY=$p python tools/attn_bench.py 32 16416; done
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -k attention 2>&1 | tail -1
