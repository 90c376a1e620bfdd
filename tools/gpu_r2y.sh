#!/bin/bash
# round 2: R50 b8192 energy per component under the 1000 W cap (PROFILE build, power.draw.instant)
mkdir -p gpurun_out
( rm -f paper_2601_11608_b200/csrc/build/*.o; make -C paper_2601_11608_b200/csrc PROFILE=1 PY=python -j32 > gpurun_out/r2y_build.log 2>&1; echo "profile build rc $?"
  timeout 600 python tools/power_probe.py 8192 4 0,0x100,0x200,0x1000,0x1100,0x300,0x1200,-1
) > gpurun_out/r2y.log 2>&1
cat gpurun_out/r2y.log
