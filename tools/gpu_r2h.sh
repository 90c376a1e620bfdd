#!/bin/bash
# round 2: producer 6 (direct gather from x, L2 prefetch) -- parity + A/B against re-pitch+TMA and staged gather
mkdir -p gpurun_out
( timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -x -k "gather_producer" 2>&1 | tail -3
  for n in 512 2048; do for g in 0 1 2; do WF_GATHER=$g timeout 120 python tools/prof_conv.py alex $n 0 0 50 | sed "s/^/gather=$g /"; done; done
  WF_GATHER=2 WF_TPS=1 timeout 120 python tools/prof_conv.py alex 2048 0 0 50 | sed "s/^/gather=2 tps1 /"
) > gpurun_out/r2h.log 2>&1
cat gpurun_out/r2h.log
