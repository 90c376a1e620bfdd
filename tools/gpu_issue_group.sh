#!/bin/bash
# Rebuilds conv_prod0 with WFB_ISSUE_GROUP = 4 / 6 / 8 on the box and times the MMA-only and full kernels.
mkdir -p gpurun_out
( for g in 4 6 8; do
  echo "== group $g"
  touch paper_2601_11608_b200/csrc/conv_prod0.cu
  make -C paper_2601_11608_b200/csrc PY=$(which python) NVFLAGS="-std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xptxas -v -DWFB_ISSUE_GROUP=$g" > /dev/null 2>&1
  timeout 60 python tools/prof_conv.py r50 8192 0 0 10 0x201200
  timeout 60 python tools/prof_conv.py r50 8192 0 0 20 0
  timeout 60 python tools/prof_conv.py alex 1024 0 0 20 0
  timeout 60 python tools/prof_conv.py alex 1024 0 0 10 0x201200
done ) > gpurun_out/issue_group.log 2>&1
cat gpurun_out/issue_group.log
