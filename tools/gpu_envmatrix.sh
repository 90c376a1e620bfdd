#!/bin/bash
# config x planner/launch-knob timing matrix (short runs)
mkdir -p gpurun_out
( for env in "" "WF_TPS=1" "WF_TPS=4" "WF_KPAIR=0" "WF_KPAIR=1" "WF_NACC=2" "WF_EPI_PP=0" "WF_EPI_PP=1"; do
  echo "== $env"
  for c in "r50 4096" "alex 1024" "mnv2 1024" "vgg 512"; do
    set -- $c
    env $env timeout 60 python tools/prof_conv.py $1 $2 0 0 20 0 2>&1 | tail -1
  done
done ) > gpurun_out/envmatrix.log 2>&1
cat gpurun_out/envmatrix.log
