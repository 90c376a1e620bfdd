#!/bin/bash
mkdir -p gpurun_out
( timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for fl in 0 0x1300; do timeout 60 python tools/prof_conv.py alex 2048 0 0 20 $fl; done
timeout 60 python tools/prof_conv.py alex 512 0 0 20 0
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"repitch" -c 2 python tools/prof_conv.py alex 2048 0 0 2 0 2>&1 | grep -E "gpu__time|dram__" | head -6
) > gpurun_out/alex3.log 2>&1
cat gpurun_out/alex3.log
