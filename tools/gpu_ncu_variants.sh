#!/bin/bash
# ncu --set full of the three variants of the same kernel on R50 conv1 (n=2048):
# fold (Cin 3, f=8), zero-padded Cin 3->8, unfolded Cin=3 (explicit im2col)
mkdir -p gpurun_out
for v in "fold r50 0" "zeropad r50zp 0" "unfolded r50 0"; do
  set -- $v
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_fold -s 1 -c 1 -o gpurun_out/prof_var_$1 -f \
     python tools/prof_conv.py $2 2048 $3 0 2 0 $( [ $1 = unfolded ] && echo unfolded || echo fold ) > gpurun_out/ncu_var_$1.log 2>&1
  tail -2 gpurun_out/ncu_var_$1.log
done
