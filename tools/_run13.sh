for p in 0 2 3 4 8; do echo "PE=$p"; FRAG_ATTN_QTM_POLY=$p timeout 300 python tools/attn_bench.py; FRAG_ATTN_QTM_POLY=$p timeout 300 python tools/attn_bench.py 4900 32800; done
