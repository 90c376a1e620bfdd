#!/bin/bash
# GPU tests, then the per-config bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
cat gpurun_out/pytest_gpu.log
timeout 900 python tools/bench_configs.py > gpurun_out/configs.log 2>&1
for fl in 0 0x4000; do timeout 60 python tools/prof_conv.py r50 2048 0 0 20 $fl; done >> gpurun_out/configs.log 2>&1
cat gpurun_out/configs.log
