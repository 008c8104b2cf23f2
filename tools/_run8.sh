timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_sharedv_gpu.py -q -x -p no:cacheprovider -k "rope or shared or stitch" 2>&1 | tail -2
timeout 300 python tools/stitch_bench.py
