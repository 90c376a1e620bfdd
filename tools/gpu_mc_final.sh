#!/bin/bash
# Multicast N-tile cluster on by default: parity suite, smoke, multicast vs single-CTA, config table.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 200 python __graft_entry__.py --smoke-only > gpurun_out/smoke.log 2>&1
timeout 150 python tools/mc_check.py > gpurun_out/mc_check.log 2>&1
timeout 600 python tools/bench_configs.py --out gpurun_out/configs.json > gpurun_out/configs.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log; cat gpurun_out/mc_check.log; tail -12 gpurun_out/configs.log
