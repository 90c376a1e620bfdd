#!/bin/bash
mkdir -p gpurun_out
( timeout 120 python tools/cmp_modes.py
for fl in 0 0x1000 0x2000 0x2400 0x2100; do timeout 60 python tools/prof_conv.py r50 2048 0 0 20 $fl; done
for fl in 0 0x2000; do timeout 60 python tools/prof_conv.py r50 8192 0 0 10 $fl; done
for c in vgg mnv2; do for fl in 0 0x2000; do timeout 60 python tools/prof_conv.py $c 1024 0 0 10 $fl; done; done ) > gpurun_out/epi.log 2>&1
cat gpurun_out/epi.log
