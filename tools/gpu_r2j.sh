#!/bin/bash
# round 2: output-store energy probe (st.global vs TMA bulk store), the conv's own power, compute-sanitizer
# over every producer (incl. the unaligned-row gathers), then a PROFILE build: VGG/MNv2 component times
mkdir -p gpurun_out
( bash tools/gpu_sanitize.sh > /dev/null 2>&1; grep -E "=== |ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/sanitize.log
  grep -E "ring|gather" gpurun_out/sanitize.log | head -12
  timeout 300 python tools/store_probe.py 13.15 3
  timeout 300 python tools/power_probe.py 8192 3 0,-1
  rm -f paper_2601_11608_b200/csrc/build/*.o; make -C paper_2601_11608_b200/csrc PROFILE=1 PY=python -j32 > gpurun_out/r2j_build.log 2>&1; echo "profile build rc $?"
  for cfg in "vgg 256" "mnv2 1024"; do for fl in 0 0x100 0x1000 0x200 0x1100; do timeout 120 python tools/prof_conv.py $cfg 0 0 30 $fl; done; done
) > gpurun_out/r2j.log 2>&1
cat gpurun_out/r2j.log
