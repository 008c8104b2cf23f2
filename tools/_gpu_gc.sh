timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_pipeline_gpu.py tests/test_batch_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 300 python tools/gemm_trace.py 32 2>&1 | grep -E "^[a-z]|partial|end"
FRAG_GEMM_CLUSTER=0 timeout 300 python tools/gemm_trace.py 32 2>&1 | grep -E "^[a-z]"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --sweep "" --batch 0 > gpurun_out/bench_gc.log 2>&1; tail -1 gpurun_out/bench_gc.log | python -c "import json,sys; d=json.load(sys.stdin); print(d['ttft_ms'], d['stage_ms'], d['gemm_stream'], d['clocks'])"
