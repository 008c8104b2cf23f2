out=gpurun_out/sanitizer_sync.log; : > $out
for prog in tools/sanitize_tiny.py tools/sanitize_attn.py; do
  echo "== synccheck $prog" >> $out
  timeout 600 compute-sanitizer --tool synccheck --print-limit 5 python $prog 2>&1 | grep -E "^ok|SUMMARY|rror|hazard" | head -8 >> $out
done
cat $out
timeout 600 python -m pytest tests/test_sharedv_gpu.py tests/test_kernels_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 900 python bench.py --steps 10 --warmup 3 --sweep "" --no-cpu-baseline > gpurun_out/bench_quick.log 2>&1; tail -1 gpurun_out/bench_quick.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('ttft', d['ttft_ms'], 'e2e', d['e2e']['ttft_ms'], 'clk', d['clocks']['sm_mhz'], 'attn', d['kernels']['attention'])"
