#!/bin/bash
# round 2: im2col transposer with warp-uniform realignment -- unfolded-variant parity + timing
mkdir -p gpurun_out
( timeout 600 python -m pytest tests -q -m gpu -x -k "unfolded or im2col or variant or sanit" 2>&1 | tail -3
  for cfg in "r50 2048" "alex 1024" "vgg 256" "mnv2 1024"; do timeout 120 python tools/prof_conv.py $cfg 0 0 5 0 unfolded; done
) > gpurun_out/r2ff.log 2>&1
cat gpurun_out/r2ff.log
