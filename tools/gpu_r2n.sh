#!/bin/bash
# round 2: batch-1 component times (PROFILE build), graph replay
mkdir -p gpurun_out
( timeout 120 python tools/b1_components.py 0
  rm -f paper_2601_11608_b200/csrc/build/*.o; make -C paper_2601_11608_b200/csrc PROFILE=1 PY=python -j32 > gpurun_out/r2n_build.log 2>&1; echo "profile build rc $?"
  timeout 300 python tools/b1_components.py 0,0x100,0x200,0x1000,0x1100,0x1300
) > gpurun_out/r2n.log 2>&1
cat gpurun_out/r2n.log
