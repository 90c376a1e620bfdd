#!/bin/bash
# Historical: the 0x2000 switch existed only for this experiment; it is a no-op on main.
# Issue path A/B: whole unrolled runs of the 21/28-entry schedules (default)
# vs rolled groups of 7 (profiling switch 0x2000); full kernel and MMA-only
# (0x1200), short runs, then the GPU parity suite and the sustained bench.
mkdir -p gpurun_out
( for rep in 1 2; do
  for c in "r50 4096" "alex 1024" "mnv2 1024" "vgg 512"; do
    set -- $c
    for fl in 0 0x2000 0x1200 0x3200; do
      timeout 60 python tools/prof_conv.py $1 $2 0 0 20 $fl 2>&1 | tail -1
    done
  done
done ) > gpurun_out/whole_runs.log 2>&1
cat gpurun_out/whole_runs.log
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 200 --warmup 5 --no-e2e --no-cpu --no-variants > gpurun_out/bench_quick.log 2>&1
tail -c 600 gpurun_out/bench_quick.log
