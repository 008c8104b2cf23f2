for fl in 1 0; do
FRAG_CHAIN_FLOW=$fl timeout 900 python bench.py --steps 10 --warmup 3 --sweep "" --no-cpu-baseline > gpurun_out/bench_flow$fl.log 2>&1; tail -1 gpurun_out/bench_flow$fl.log | cut -c1-300; tail -1 gpurun_out/bench_flow$fl.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('flow $fl ttft', round(d['ttft_ms'],2), 'clk', d['clocks']['sm_mhz'], 'question', round(d['stage_ms']['question_ms'],3), 'decode', round(d['decode']['ms_per_token'],3))"
done
