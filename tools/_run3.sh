timeout 600 python -m pytest tests/test_sharedv_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_sharedv.log 2>&1; tail -5 gpurun_out/pytest_sharedv.log
timeout 300 python tools/debug_sharedv.py 0.15 2>&1 | head -3
timeout 900 python bench.py --steps 10 --warmup 3 --sweep "" > gpurun_out/bench_quick.log 2>&1; tail -1 gpurun_out/bench_quick.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('ttft', d['ttft_ms'], 'e2e', d['e2e']['ttft_ms'])
for k in ['stage_ms','kernels','attention','stitch','decode','batched','clocks']: print(k, json.dumps(d.get(k))[:500])"
