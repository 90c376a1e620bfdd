#!/bin/bash
# ncu --set full of the conv kernel for AlexNet / VGG / MNv2 (R50 is in gpu_session.sh)
mkdir -p gpurun_out
for c in "alex 1024" "vgg 512" "mnv2 1024"; do
  set -- $c
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv_fold -s 2 -c 1 -o gpurun_out/prof_cfg_$1 -f \
     python tools/prof_conv.py $1 $2 0 0 3 > gpurun_out/ncu_cfg_$1.log 2>&1
  tail -1 gpurun_out/ncu_cfg_$1.log
done
