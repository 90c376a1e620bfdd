#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_fold -s 2 -c 1 -o gpurun_out/prof_mnv2 -f \
   python tools/prof_conv.py mnv2 1024 0 0 3 > gpurun_out/ncu_mnv2.log 2>&1
tail -3 gpurun_out/ncu_mnv2.log
