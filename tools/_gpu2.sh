timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k "stream_k or small_m" 2>&1 | tail -5
timeout 300 python tools/gemm_small.py 32 tiny,small,qkv,o,gu,down > gpurun_out/gs.log 2>&1; cut -c1-400 gpurun_out/gs.log
