#!/bin/bash
# round 2: AlexNet b2048 knob A/B (interleaved, 3 reps)
mkdir -p gpurun_out
( for rep in 1 2 3; do
    for env in "WF_X=0" "WF_TPS=1" "WF_KPAIR=0" "WF_NACC=2" "WF_MCAST=1" "WF_PLANES=0"; do
      echo -n "alex $env: "; env $env timeout 120 python tools/prof_conv.py alex 2048 0 0 30 2>&1 | tail -1 | awk '{print $7, $8}'
    done
  done
) > gpurun_out/r2w.log 2>&1
cat gpurun_out/r2w.log
