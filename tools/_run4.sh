for side in 1 0; do
FRAG_VWIN_SIDE=$side timeout 900 python bench.py --steps 10 --warmup 3 --sweep "" --no-cpu-baseline > gpurun_out/bench_side$side.log 2>&1; tail -1 gpurun_out/bench_side$side.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('side $side ttft', d['ttft_ms'], 'e2e', d['e2e']['ttft_ms'], 'decode', d['decode']['ms_per_token'], 'clk', d['clocks']['sm_mhz'], 'sparse', d['stage_ms']['sparse_ms'])"
done
