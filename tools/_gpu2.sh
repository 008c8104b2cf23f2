timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "gemm" 2>&1 | tail -2
timeout 300 python tools/gemm_small.py 32 qkv,o,gu,down,lm > gpurun_out/gs.log 2>&1; cut -c1-300 gpurun_out/gs.log
timeout 300 python tools/gemm_small.py 1 qkv,o,gu,down > gpurun_out/gs1.log 2>&1; cut -c1-300 gpurun_out/gs1.log
