#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/bench_configs.py > gpurun_out/configs.log 2>&1
for fl in 0 0x4000; do timeout 60 python tools/prof_conv.py r50 2048 0 0 20 $fl; done >> gpurun_out/configs.log 2>&1
cat gpurun_out/configs.log
