ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 2 -c 1 -o gpurun_out/attn_src2 timeout 120 python tools/attn_bench.py > gpurun_out/ncu_attn.log 2>&1
tail -2 gpurun_out/ncu_attn.log
