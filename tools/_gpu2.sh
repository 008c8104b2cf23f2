timeout 600 python -m pytest tests -q -x -m gpu 2>&1 | tail -3
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]);print(d['ttft_ms'],d['stage_ms'],d['kernels']['select'])"
