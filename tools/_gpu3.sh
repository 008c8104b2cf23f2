ncu --set full --clock-control none --import-source on -k regex:gemm_tc2 -s 2 -c 1 -o gpurun_out/gemm_tail python tools/gemm_one.py 2490 4096 4096 0x50100 > gpurun_out/ncu_g.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tc2 -s 2 -c 1 -o gpurun_out/gemm_notail python tools/gemm_one.py 2490 4096 4096 0x40100 >> gpurun_out/ncu_g.log 2>&1
tail -3 gpurun_out/ncu_g.log
