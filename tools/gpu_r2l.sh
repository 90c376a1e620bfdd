#!/bin/bash
# round 2: AlexNet plan alternatives (fold factor / group size) at b512 and b2048
mkdir -p gpurun_out
( for a in "8 0" "8 2" "16 0" "16 2"; do set -- $a; for n in 512 2048; do timeout 120 python tools/prof_conv.py alex $n $1 $2 30 2>&1 | tail -1; done; done
  WF_CTA_PAIR=1 timeout 120 python tools/prof_conv.py alex 2048 8 2 30 2>&1 | tail -1
) > gpurun_out/r2l.log 2>&1
cat gpurun_out/r2l.log
