FRAG_ATTN_PAIR=1 timeout 300 python -m pytest tests/test_kernels_gpu.py -k attention -x -q -p no:cacheprovider 2>&1 | tail -2
for i in 1 2; do FRAG_ATTN_PAIR=1 timeout 300 python tools/attn_bench.py; FRAG_ATTN_PAIR=0 timeout 300 python tools/attn_bench.py; done
FRAG_ATTN_PAIR=1 timeout 300 python tools/attn_trace.py 2>/dev/null | head -8
