#!/bin/bash
# round 2: does the epilogue's store stream slow the gather producer's global loads?
# PROFILE=1 build (profiling switches compiled in): 0x400 = epilogue skips its stores
cd paper_2601_11608_b200/csrc
rm -f build/*.o && make PY=python PROFILE=1 -j16 ../libwidthfold_b200.so > /dev/null 2>&1 || echo "build failed"
cd ../..
for fl in 0 0x400 0x200; do
  python tools/prof_conv.py alex 2048 0 0 20 $fl 2>&1 | tail -1
  WF_REPITCH=1 python tools/prof_conv.py alex 2048 0 0 20 $fl 2>&1 | tail -1
done
