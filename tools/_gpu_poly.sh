for p in 0 100 101; do echo "POLY=$p"; FRAG_ATTN_POLY=$p python tools/attn_trace.py 2>/dev/null | head -6; FRAG_ATTN_POLY=$p python tools/attn_bench.py; done
