timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "gemm" 2>&1 | tail -3
python tools/gemm_tune.py 2490,16416 2>&1 | tail -8
