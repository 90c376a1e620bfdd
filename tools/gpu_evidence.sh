#!/bin/bash
# Evidence refresh on the final build: launch list of a short bench run, one
# ncu --set full capture of the conv kernel (R50 n=2048), DRAM bytes of the
# bench-sized launch.
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu --no-verify > gpurun_out/launches_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_fold -s 2 -c 1 -o gpurun_out/prof_r50_n2048 -f \
   python tools/prof_conv.py r50 2048 0 0 3 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:conv_fold -s 1 -c 1 --csv --log-file gpurun_out/traffic_r50_n8192.csv \
   python tools/prof_conv.py r50 8192 0 0 1 > gpurun_out/ncu_traffic.log 2>&1
ls -la gpurun_out | tail -8
