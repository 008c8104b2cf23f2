set -x
timeout 600 python -m pytest tests/test_kernels_gpu.py -k qg_score -x -q -p no:cacheprovider > gpurun_out/pytest_score.log 2>&1; tail -3 gpurun_out/pytest_score.log
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_pipeline_gpu.py tests/test_cacheblend_gpu.py -x -q -p no:cacheprovider > gpurun_out/pytest_par.log 2>&1; tail -3 gpurun_out/pytest_par.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_sc.log 2>&1; tail -1 gpurun_out/bench_sc.log | python -c "import json,sys; d=json.load(sys.stdin); print(d['ttft_ms'], d['stage_ms'], d['kernels']['select'])"
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"score|topk" python tools/profile_step.py > gpurun_out/ncu_score.csv 2>&1; grep -E "gpu__time" gpurun_out/ncu_score.csv | awk -F'","' '{print $5, $NF}' | cut -c1-200
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"score_tc_kernel|topk" -c 3 -o gpurun_out/score_r01 python tools/profile_step.py > /dev/null 2>&1; ls gpurun_out/
