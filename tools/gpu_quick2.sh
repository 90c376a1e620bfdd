#!/bin/bash
mkdir -p gpurun_out
( timeout 60 ./tools/probes/lbo_probe
for fl in 0 0x1000 0x1100 0x1200 0x1400 0x100 0x400; do timeout 60 python tools/prof_conv.py r50 2048 0 0 20 $fl; done ) > gpurun_out/quick2.log 2>&1
cat gpurun_out/quick2.log
