timeout 600 python -m pytest tests -q -x -m gpu 2>&1 | tail -2
for i in 1 2; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]);print(round(d['ttft_ms'],2),d['stage_ms'],d['kernels']['norm'],d['clocks']['sm_mhz'])"; done
