#!/bin/bash
# round 2: where the unfolded Cin=3 variant (im2col row producer) spends its time -- CTA-0 counters (PROFILE build)
mkdir -p gpurun_out
( rm -f paper_2601_11608_b200/csrc/build/*.o; make -C paper_2601_11608_b200/csrc PROFILE=1 PY=python -j32 > gpurun_out/r2ee_build.log 2>&1; echo "profile build rc $?"
  timeout 120 python tools/prof_conv.py r50 512 0 0 1 0x88000 unfolded
  timeout 120 python tools/prof_conv.py r50 512 0 0 3 0 unfolded
  timeout 120 python tools/prof_conv.py r50 512 0 0 3 0x100 unfolded
  timeout 120 python tools/prof_conv.py r50 512 0 0 3 0x1000 unfolded
) > gpurun_out/r2ee.log 2>&1
cat gpurun_out/r2ee.log
