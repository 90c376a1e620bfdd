#!/bin/bash
# round 2: single-pass A gather by the epilogue warps (cp.async) -- parity + batch-1 latency A/B
mkdir -p gpurun_out
( timeout 120 python tools/b1_components.py 0 | sed 's/^/gather_a: /'
  WF_GATHER_A=0 timeout 120 python tools/b1_components.py 0 | sed 's/^/tma: /'
  timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
  timeout 120 python tools/host_path_probe.py
  WF_GATHER_A=0 timeout 120 python tools/host_path_probe.py
) > gpurun_out/r2aa.log 2>&1
cat gpurun_out/r2aa.log
