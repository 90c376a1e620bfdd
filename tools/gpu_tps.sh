#!/bin/bash
# two-tile stages: parity tests, then timings with and without (WF_TPS=1)
mkdir -p gpurun_out
( timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -25
for t in 2 1; do
  for c in "r50 2048" "r50 8192" "vgg 256" "mnv2 1024"; do
    if [ $t = 1 ]; then WF_TPS=1 timeout 60 python tools/prof_conv.py $c 0 0 10 0; else timeout 60 python tools/prof_conv.py $c 0 0 10 0; fi
  done
done ) > gpurun_out/tps.log 2>&1
cat gpurun_out/tps.log
