#!/bin/bash
# bandwidth ceilings + ncu full capture of the conv kernel (R50, n=2048)
mkdir -p gpurun_out
( timeout 120 ./tools/probes/wbw_probe; timeout 120 python tools/bw_probe.py ) > gpurun_out/bw.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_fold -s 2 -c 1 -o gpurun_out/prof_r50_n2048 -f \
   python tools/prof_conv.py r50 2048 0 0 3 > gpurun_out/ncu_full.log 2>&1
cat gpurun_out/bw.log
