set -x
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_q.log 2>&1; tail -1 gpurun_out/bench_q.log | python -c "import json,sys; d=json.load(sys.stdin); print(d['ttft_ms'], d['stage_ms'], d['decode'])"
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv python tools/profile_step.py > gpurun_out/ncu_q.csv 2>&1; python -c "import sys; sys.path.insert(0,'tools'); from pathlib import Path; import ncu_report as R; print(R.launch_table(Path('gpurun_out/ncu_q.csv'))[0])"
