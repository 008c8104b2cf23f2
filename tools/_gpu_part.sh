set -x
timeout 600 python -m pytest tests/test_partition_gpu.py -x -q -p no:cacheprovider > gpurun_out/pytest_part.log 2>&1; tail -30 gpurun_out/pytest_part.log
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
