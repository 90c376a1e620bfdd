#!/bin/bash
# round 2: AlexNet direct-gather producer -- parity, A/B vs re-pitch, launch list
mkdir -p gpurun_out
( timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -m gpu -k "alexnet or random or gather or partial or multicast or zeros or non_finite" 2>&1 | tail -15
  timeout 300 python tools/ab_producer.py alex 512 "" "WF_REPITCH=1" 50
  timeout 300 python tools/ab_producer.py alex 2048 "" "WF_REPITCH=1" 20
  timeout 300 python tools/ab_producer.py alex 512 "WF_TPS=1" "WF_REPITCH=1,WF_TPS=1" 50
) > gpurun_out/r2_alex.log 2>&1
cat gpurun_out/r2_alex.log
