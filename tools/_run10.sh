timeout 900 python -m pytest tests/test_headline_gpu.py tests/test_parity_gpu.py tests/test_sharedv_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 900 python bench.py --steps 10 --warmup 3 --sweep "" --no-cpu-baseline > gpurun_out/bench_quick.log 2>&1; tail -1 gpurun_out/bench_quick.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('ttft', d['ttft_ms'], 'e2e', d['e2e']['ttft_ms'], 'clk', d['clocks']['sm_mhz'], 'stages', d['stage_ms'], {k: round(v['ms_per_step'],2) for k,v in d['kernels'].items()})"
