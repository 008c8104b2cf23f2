timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k attention 2>&1 | tail -2
for i in 1 2; do timeout 60 python tools/attn_bench.py; done
FRAG_ATTN_POLY=4 timeout 60 python tools/attn_bench.py
timeout 60 python tools/attn_bench.py 32 16416
