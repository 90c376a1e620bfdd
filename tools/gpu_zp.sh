#!/bin/bash
mkdir -p gpurun_out
( timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 600 python tools/bench_configs.py --only alexnet --out gpurun_out/alex_cfg.json 2>&1 | tail -3
) > gpurun_out/zp.log 2>&1
cat gpurun_out/zp.log
