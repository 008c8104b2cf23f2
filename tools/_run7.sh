FRAG_CHAIN_FLOW=0 timeout 300 python tools/chain_trace.py 2>&1 | tail -9
timeout 300 python tools/chain_trace.py 2>&1 | tail -9
