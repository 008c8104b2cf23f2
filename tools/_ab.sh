cd $GRAFT_REPO_ROOT
for rep in 1 2; do for v in 4 2 3 0; do echo -n "poly=$v "; FRAG_ATTN_QTM_POLY=$v timeout 300 python tools/attn_bench.py 2>&1 | tail -2 | tr '\n' ' '; echo; done; done
