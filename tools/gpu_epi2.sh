#!/bin/bash
mkdir -p gpurun_out
( timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for c in mnv2 alex vgg; do timeout 60 python tools/prof_conv.py $c 1024 0 0 20 0; done
timeout 60 python tools/prof_conv.py r50 8192 0 0 20 0
timeout 60 python tools/prof_conv.py r50 2048 0 0 20 0x1100
) > gpurun_out/epi2.log 2>&1
cat gpurun_out/epi2.log
