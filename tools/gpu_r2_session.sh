#!/bin/bash
# round 2 evidence session: GPU suite, smoke, bench (both arms), launch list, ncu --set full of the
# R50 conv (n=2048) and of AlexNet (b512), DRAM bytes of the bench-sized launch, compute-sanitizer.
# Then: python tools/make_profiles.py r2x
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/gpu.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py --smoke-only > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu --no-verify --no-configs --no-variants > gpurun_out/launches_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_fold -s 2 -c 1 -o gpurun_out/prof_r50_n2048 -f \
   python tools/prof_conv.py r50 2048 0 0 3 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_fold -s 2 -c 1 -o gpurun_out/prof_vgg_b256 -f python tools/prof_conv.py vgg 256 0 0 3 > gpurun_out/ncu_full_vgg.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_fold -s 2 -c 1 -o gpurun_out/prof_alex_b512 -f \
   python tools/prof_conv.py alex 512 0 0 3 > gpurun_out/ncu_full_alex.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_fold -s 2 -c 1 -o gpurun_out/prof_mnv2_b1024 -f \
   python tools/prof_conv.py mnv2 1024 0 0 3 > gpurun_out/ncu_full_mnv2.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:conv_fold -s 1 -c 1 --csv --log-file gpurun_out/traffic_r50_n8192.csv \
   python tools/prof_conv.py r50 8192 0 0 1 > gpurun_out/ncu_traffic.log 2>&1
bash tools/gpu_sanitize.sh > /dev/null 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log | tail -1; grep -E "=== |ERROR SUMMARY" gpurun_out/sanitize.log
