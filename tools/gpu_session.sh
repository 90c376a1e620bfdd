#!/bin/bash
# One gpurun session: GPU parity tests, smoke, the bench (both arms), the
# launch list and an ncu --set full capture of the conv kernel.
set -x
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/gpu.txt 2>&1
timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py --smoke-only > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu --no-verify > gpurun_out/launches_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_fold -s 2 -c 1 -o gpurun_out/prof_r50_n2048 -f \
   python tools/prof_conv.py r50 2048 0 0 3 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:conv_fold -s 1 -c 1 --csv --log-file gpurun_out/traffic_r50_n8192.csv \
   python tools/prof_conv.py r50 8192 0 0 1 > gpurun_out/ncu_traffic.log 2>&1
ls -la gpurun_out
WF_KPAIR=1 timeout 200 python tools/power_probe.py 8192 3 0,-1,0x1100,0x1200,0x300 > gpurun_out/power.log 2>&1
timeout 600 python tools/bench_configs.py --out gpurun_out/configs.json > gpurun_out/configs.log 2>&1
