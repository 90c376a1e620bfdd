#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
( for fl in 0 0x4000 0x4100 0x4200 0x5000 0x5100; do timeout 60 python tools/prof_conv.py r50 2048 0 0 20 $fl; done ) > gpurun_out/rowprod.log 2>&1
timeout 900 python tools/bench_configs.py > gpurun_out/configs.log 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/rowprod.log gpurun_out/configs.log
