#!/bin/bash
# round 2: GPU suite, smoke, the default bench line, and the kernel launch list
mkdir -p gpurun_out
( timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -25
  timeout 300 python __graft_entry__.py --smoke-only 2>&1 | tail -3
  timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc $?"; tail -c 6000 gpurun_out/bench.log
) > gpurun_out/r2a.log 2>&1
cat gpurun_out/r2a.log | tail -60
