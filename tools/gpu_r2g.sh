#!/bin/bash
# round 2: producer 5 stage counters (PROFILE build, 0x80000: CTA 0 cycle counters of gather warp 0, the TMA producer, the MMA issuer)
mkdir -p gpurun_out
( rm -f paper_2601_11608_b200/csrc/build/*.o; make -C paper_2601_11608_b200/csrc PROFILE=1 PY=python -j32 > gpurun_out/r2g_build.log 2>&1; echo "profile build rc $?"
  timeout 120 python tools/prof_conv.py alex 2048 0 0 1 0x80000
  timeout 120 python tools/prof_conv.py alex 2048 0 0 1 0x80300
  WF_REPITCH=1 timeout 120 python tools/prof_conv.py alex 2048 0 0 1 0x80000
) > gpurun_out/r2g.log 2>&1
cat gpurun_out/r2g.log
