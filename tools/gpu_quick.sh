#!/bin/bash
# quick loop: GPU parity tests + component timings (R50 conv1) + other configs
mkdir -p gpurun_out
( timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -15
for fl in 0 0x100 0x200 0x400 0x800; do timeout 60 python tools/prof_conv.py r50 2048 0 0 20 $fl; done
timeout 60 python tools/prof_conv.py r50 8192 0 0 10 0
for c in vgg mnv2; do timeout 60 python tools/prof_conv.py $c 1024 0 0 10 0; done ) > gpurun_out/quick.log 2>&1
cat gpurun_out/quick.log
