#!/bin/bash
# round 2: run one GPU test file (default: the full-size parity file) with timings
mkdir -p gpurun_out
F=${1:-tests/test_gpu_fullsize.py}
timeout 1500 python -m pytest $F -q -m gpu --durations=30 -p no:cacheprovider > gpurun_out/r2_tests.log 2>&1
echo "rc $?" >> gpurun_out/r2_tests.log
tail -60 gpurun_out/r2_tests.log
