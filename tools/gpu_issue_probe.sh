#!/bin/bash
# Issue-path bisection: issue_probe variants on the R50 kpair
# schedule (isolated, kernel-shaped launches), then the kernel's own CTA-0
# issuer counters (profiling 0x80000: cycles, globaltimer ns -> the SM clock
# the launch ran at, barrier waits) in MMA-only and full launches.
mkdir -p gpurun_out
python tools/sched_probe.py gpurun_out/sched_kpair.txt > /dev/null
timeout 120 tools/probes/issue_probe gpurun_out/sched_kpair.txt > gpurun_out/issue_probe_k.log 2>&1
( for c in "r50 4096" "alex 1024" "r50 8192"; do set -- $c
  for fl in 0x81200 0x281200 0x80000; do
    timeout 60 python tools/prof_conv.py $1 $2 0 0 5 $fl 2>&1 | grep -E "issuer cta0|flags=" | tail -2
  done
done ) >> gpurun_out/issue_probe_k.log 2>&1
cat gpurun_out/issue_probe_k.log
