#!/bin/bash
# ncu --set full of the AlexNet conv kernel (gather producer) -> gpurun_out/prof_alex_gather.ncu-rep
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_fold -s 2 -c 1 -o gpurun_out/prof_alex_gather -f \
   python tools/prof_conv.py alex 512 0 0 3 > gpurun_out/ncu_alex_gather.log 2>&1
tail -3 gpurun_out/ncu_alex_gather.log
python tools/ncu_summary.py gpurun_out/prof_alex_gather.ncu-rep 40 > gpurun_out/ncu_alex_gather_summary.txt 2>&1
cat gpurun_out/ncu_alex_gather_summary.txt
