#!/bin/bash
# round 2: single-pass launches with one stage set / one accumulator (2 CTAs per SM under PDL)
mkdir -p gpurun_out
( timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
  timeout 120 python tools/host_path_probe.py
  timeout 120 python tools/b1_components.py 0
  timeout 120 python tools/latency_b1.py
) > gpurun_out/r2p.log 2>&1
cat gpurun_out/r2p.log
