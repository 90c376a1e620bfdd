#!/bin/bash
# round 2: producer 5 diagnosis -- release timing, then a PROFILE build: no gather loads / no fence / no MMA / no epilogue
mkdir -p gpurun_out
( for n in 512 2048; do timeout 120 python tools/prof_conv.py alex $n 0 0 50; WF_REPITCH=1 timeout 120 python tools/prof_conv.py alex $n 0 0 50; done
  rm -f paper_2601_11608_b200/csrc/build/*.o; make -C paper_2601_11608_b200/csrc PROFILE=1 PY=python -j32 > gpurun_out/r2f_build.log 2>&1; echo "profile build rc $?"
  for fl in 0 0x8000 0x10000 0x18000 0x100 0x200 0x300 0x1000; do timeout 120 python tools/prof_conv.py alex 2048 0 0 30 $fl; done
  WF_REPITCH=1 timeout 120 python tools/prof_conv.py alex 2048 0 0 30 0x100
  WF_REPITCH=1 timeout 120 python tools/prof_conv.py alex 2048 0 0 30 0x200
) > gpurun_out/r2f.log 2>&1
cat gpurun_out/r2f.log
