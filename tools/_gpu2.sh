timeout 600 python bench.py --config mistral-7b-batch --warmup 3 --no-cpu-baseline > gpurun_out/m7.log 2>&1; tail -c 1500 gpurun_out/m7.log; echo
timeout 900 python bench.py --config llama3-70b --steps 5 --warmup 3 --full-steps 1 --no-cpu-baseline > gpurun_out/b70.log 2>&1; tail -c 1500 gpurun_out/b70.log
