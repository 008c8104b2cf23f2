timeout 600 python -m pytest tests/test_kernels_gpu.py -k attention -x -q 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --sweep "" --batch 0 > gpurun_out/bench_dual.log 2>&1; tail -1 gpurun_out/bench_dual.log | python -c "import json,sys; d=json.load(sys.stdin); print(d['ttft_ms'], d['stage_ms'], d['decode'], d['kernels']['attention'])"
