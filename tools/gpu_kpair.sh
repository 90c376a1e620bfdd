#!/bin/bash
# A/B of the K-step schedules (WF_KPAIR=0: 32-byte covers, 1: cross-kh core-column pairs)
mkdir -p gpurun_out
( timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -15
for kp in 0 1; do
  export WF_KPAIR=$kp
  echo "== WF_KPAIR=$kp"
  for fl in 0 0x100 0x200 0x1000; do timeout 60 python tools/prof_conv.py r50 2048 0 0 20 $fl; done
  timeout 60 python tools/prof_conv.py r50 8192 0 0 20 0
  timeout 60 python tools/prof_conv.py alex 512 0 0 20 0
  timeout 60 python tools/prof_conv.py mnv2 1024 0 0 20 0
done
unset WF_KPAIR
timeout 300 python bench.py --no-e2e --no-cpu > gpurun_out/bench_kpair.log 2>&1; tail -c 600 gpurun_out/bench_kpair.log
) > gpurun_out/kpair.log 2>&1
cat gpurun_out/kpair.log
