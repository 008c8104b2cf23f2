# Round evidence run (one gpurun call): GPU tests, smoke, the default bench
# line, the reference arm, the other configs' bench lines and the ncu captures.
# Usage: bash tools/_gpu_final.sh <tag>
TAG=${1:-r02}
set -x
timeout 900 python -m pytest tests -q -x -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final.log 2>&1; tail -1 gpurun_out/bench_final.log | cut -c1-300
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-300
timeout 900 python bench.py --config mistral-7b-batch --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/bench_mistral.log 2>&1; tail -1 gpurun_out/bench_mistral.log | cut -c1-200
timeout 1200 python bench.py --config llama3-70b --steps 3 --warmup 3 --no-cpu-baseline --sweep "" > gpurun_out/bench_70b.log 2>&1; tail -1 gpurun_out/bench_70b.log | cut -c1-200
timeout 1500 bash tools/ncu_capture.sh $TAG > gpurun_out/cap.log 2>&1
timeout 1500 bash tools/sanitize.sh > /dev/null 2>&1; tail -5 gpurun_out/sanitizer.log
