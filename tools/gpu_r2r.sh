#!/bin/bash
mkdir -p gpurun_out
( rm -f paper_2601_11608_b200/csrc/build/*.o; make -C paper_2601_11608_b200/csrc PROFILE=1 PY=python -j32 > gpurun_out/r2r_build.log 2>&1; echo "profile build rc $?"
  timeout 60 python tools/b1_timeline.py tf32 1
  timeout 60 python tools/b1_timeline.py bf16 1
) > gpurun_out/r2r.log 2>&1
cat gpurun_out/r2r.log
