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
# sparse pass, layer 0: the four CTA-pair GEMMs (QKV, O, gate/up, down)
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:gemm_tc2 -s 0 -c 4 -o $OUT/gemm_$TAG python tools/profile_step.py > /dev/null 2>&1
# question pass, layer 0: the four weight-streaming GEMMs
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:gemm_tc_kernel -s 0 -c 4 -o $OUT/gemmq_$TAG python tools/profile_step.py > /dev/null 2>&1
# question pass, layer 0: the GEMM chain (combine pre-op + O, gate/up, down, next QKV)
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:gemm_chain -s 0 -c 1 -o $OUT/chain_$TAG python tools/profile_step.py > /dev/null 2>&1
# sparse pass, layer 0 attention (after the 32 question-pass launches) + one question-pass attention
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"attn_qtm|attn_tc" -s 32 -c 1 -o $OUT/attn_$TAG python tools/profile_step.py > /dev/null 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"attn_tc|attn_combine" -s 0 -c 2 -o $OUT/attnq_$TAG python tools/profile_step.py > /dev/null 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on \
    -k regex:"rope_shift|score_tc|score_split|topk|rmsnorm" -c 8 -o $OUT/mem_$TAG python tools/profile_step.py > /dev/null 2>&1
ls -la $OUT
