set -x
timeout 600 python -m pytest tests/test_kernels_gpu.py -k "attention" -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_pipeline_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 300 python tools/attn_bench.py 2>&1 | tail -5
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --sweep "" > gpurun_out/bench_attn.log 2>&1; tail -1 gpurun_out/bench_attn.log | python -c "import json,sys; d=json.load(sys.stdin); print(d['ttft_ms'], d['stage_ms'], d['attention'], d['kernels']['attention'], d['clocks'])"
