#!/bin/bash
mkdir -p gpurun_out
( for fl in 0 0x1300 0x300; do timeout 60 python tools/prof_conv.py alex 2048 0 0 20 $fl; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"repitch|conv_fold" -c 6 python tools/prof_conv.py alex 2048 0 0 2 0 2>&1 | grep -E "repitch|conv_fold|gpu__time|dram__" | head -30
) > gpurun_out/alex2.log 2>&1
cat gpurun_out/alex2.log
