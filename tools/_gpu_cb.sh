set -x
timeout 600 python -m pytest tests/test_cacheblend_gpu.py -x -q -p no:cacheprovider > gpurun_out/pytest_cb.log 2>&1; tail -30 gpurun_out/pytest_cb.log
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cb.log 2>&1; tail -1 gpurun_out/bench_cb.log | python -c "import json,sys; d=json.load(sys.stdin); print(d['ttft_ms'], d['cacheblend'], d['stage_ms'])"
