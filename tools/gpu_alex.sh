#!/bin/bash
mkdir -p gpurun_out
( for fl in 0 0x100 0x200 0x1000 0x300; do timeout 60 python tools/prof_conv.py alex 2048 0 0 20 $fl; done
timeout 60 python tools/prof_conv.py alex 2048 0 0 2 0x80000 2>&1 | grep -i "issuer" | head -4
for fl in 0 0x200; do WF_KPAIR=0 timeout 60 python tools/prof_conv.py alex 2048 0 0 20 $fl; done
) > gpurun_out/alex.log 2>&1
cat gpurun_out/alex.log
