set -x
python -c "import sys; sys.path.insert(0,'.'); import paper_2601_12904_b200" 
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; tail -c 3000 gpurun_out/bench.log
