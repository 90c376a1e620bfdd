#!/bin/bash
# round 2: blocked unit order (each CTA streams a contiguous block of units) -- parity + A/B
mkdir -p gpurun_out
( WF_BLOCKED=1 timeout 600 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_fuzz.py -q -m gpu -x -k "steady or every_image or headline or random_geometry_exact" 2>&1 | tail -2
  for rep in 1 2 3; do
    for env in "WF_X=0" "WF_BLOCKED=1"; do
      echo -n "r50 $env: "; env $env timeout 120 python tools/prof_conv.py r50 8192 0 0 100 2>&1 | tail -1 | awk '{print $7, $8}'
      echo -n "vgg $env: "; env $env timeout 120 python tools/prof_conv.py vgg 256 0 0 100 2>&1 | tail -1 | awk '{print $7, $8}'
      echo -n "mnv2 $env: "; env $env timeout 120 python tools/prof_conv.py mnv2 1024 0 0 100 2>&1 | tail -1 | awk '{print $7, $8}'
      echo -n "alex $env: "; env $env timeout 120 python tools/prof_conv.py alex 2048 0 0 30 2>&1 | tail -1 | awk '{print $7, $8}'
    done
  done
) > gpurun_out/r2jj.log 2>&1
cat gpurun_out/r2jj.log
