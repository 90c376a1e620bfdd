#!/bin/bash
# round 2: interleaved A/B of the planner knobs that the sweep flagged (VGG multicast / tps, MNv2 ping-pong)
mkdir -p gpurun_out
( for rep in 1 2 3; do
    for env in "WF_X=0" "WF_MCAST=0" "WF_TPS=1" "WF_MCAST=0 WF_TPS=1"; do
      echo -n "vgg $env: "; env $env timeout 120 python tools/prof_conv.py vgg 256 0 0 100 2>&1 | tail -1 | awk '{print $7, $8}'
    done
    for env in "WF_X=0" "WF_EPI_PP=0"; do
      echo -n "mnv2 $env: "; env $env timeout 120 python tools/prof_conv.py mnv2 1024 0 0 100 2>&1 | tail -1 | awk '{print $7, $8}'
    done
    for env in "WF_X=0" "WF_MCAST=0"; do
      echo -n "alex $env: "; env $env timeout 120 python tools/prof_conv.py alex 2048 0 0 30 2>&1 | tail -1 | awk '{print $7, $8}'
    done
  done
) > gpurun_out/r2t.log 2>&1
cat gpurun_out/r2t.log
