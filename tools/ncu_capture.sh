#!/bin/bash
# One-request ncu evidence for profiles/: launch list (time per launch) and
# --set full captures of the dominant kernels of the sparse pass.
# Usage (on the GPU box): bash tools/ncu_capture.sh <tag>
set -x
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_$TAG.csv python tools/profile_step.py > /dev/null 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_full_$TAG.csv python tools/profile_step.py --full > /dev/null 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:gemm_tc -s 125 -c 4 -o $OUT/gemm_$TAG python tools/profile_step.py > /dev/null 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:attn_tc -s 31 -c 1 -o $OUT/attn_$TAG python tools/profile_step.py > /dev/null 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"rope_shift|score_kernel|topk|rmsnorm" -c 6 -o $OUT/mem_$TAG python tools/profile_step.py > /dev/null 2>&1
ls -la $OUT
