#!/bin/bash
# Final build evidence: compute-sanitizer over every producer (now incl. the
# multicast N-tile cluster), the bench line (both arms), the launch list.
mkdir -p gpurun_out
bash tools/gpu_sanitize.sh > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu --no-verify > gpurun_out/launches_bench.log 2>&1
grep -E "===|ERROR SUMMARY|normwise" gpurun_out/sanitize.log | head -30; tail -c 300 gpurun_out/bench.log
