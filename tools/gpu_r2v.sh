#!/bin/bash
# round 2: R50 b8192 knob A/B under the power cap (100 launches per sample, interleaved, 3 reps)
mkdir -p gpurun_out
( for rep in 1 2 3; do
    for env in "WF_X=0" "WF_TPS=1" "WF_TPS=4" "WF_KPAIR=0" "WF_EPI_PP=1"; do
      echo -n "r50 $env: "; env $env timeout 120 python tools/prof_conv.py r50 8192 0 0 100 2>&1 | tail -1 | awk '{print $7, $8}'
    done
  done
) > gpurun_out/r2v.log 2>&1
cat gpurun_out/r2v.log
