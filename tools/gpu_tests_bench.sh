#!/bin/bash
# GPU parity suite, then the default bench line (ours) and the per-config table
mkdir -p gpurun_out
( timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15
timeout 600 python bench.py --no-e2e > gpurun_out/bench_tb.log 2>&1; tail -c 1500 gpurun_out/bench_tb.log
timeout 600 python tools/bench_configs.py --out gpurun_out/configs.json > gpurun_out/configs.log 2>&1; tail -30 gpurun_out/configs.log
) > gpurun_out/tb.log 2>&1
cat gpurun_out/tb.log
