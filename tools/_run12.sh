FRAG_ATTN_Q2=1 timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -p no:cacheprovider -k "attn or attention" 2>&1 | tail -3
for q in 0 1; do echo "Q2=$q"; FRAG_ATTN_Q2=$q timeout 300 python tools/attn_bench.py; FRAG_ATTN_Q2=$q timeout 300 python tools/attn_bench.py 4900 32800; done
