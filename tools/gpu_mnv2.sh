#!/bin/bash
mkdir -p gpurun_out
( for c in mnv2 vgg; do for fl in 0 0x100 0x200 0x1000 0x300 0x1300; do timeout 60 python tools/prof_conv.py $c 1024 0 0 20 $fl; done; done
timeout 60 python tools/prof_conv.py mnv2 1024 0 0 2 0x80000 2>&1 | grep -i issuer | head -2
WF_KPAIR=0 timeout 60 python tools/prof_conv.py mnv2 1024 0 0 20 0
WF_TPS=1 timeout 60 python tools/prof_conv.py mnv2 1024 0 0 20 0
) > gpurun_out/mnv2.log 2>&1
cat gpurun_out/mnv2.log
