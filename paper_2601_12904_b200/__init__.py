"""B200-native (sm_100a) FusionRAG online reprocessing: HBM chunk-KV store,
RoPE re-positioning, query-guided critical-token selection and selective
recompute prefill behind a C ABI (include/frag/frag_c.h).

`fusion` is the Python mirror of the reference's reprocessing surface.
"""
__version__ = "0.1.0"
