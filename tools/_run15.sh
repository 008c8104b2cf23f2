for fl in 1 0; do echo "flow $fl"; FRAG_CHAIN_FLOW=$fl timeout 300 python tools/r0_bench.py; done
