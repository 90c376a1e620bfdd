mkdir -p gpurun_out
# Historical: the 0x2000 switch existed only for this experiment; it is a no-op on main.
( for rep in 1 2; do for c in "r50 4096" "alex 1024"; do set -- $c
  for fl in 0x1200 0x3200 0x201200 0x203200; do timeout 60 python tools/prof_conv.py $1 $2 0 0 20 $fl 2>&1 | tail -1; done; done; done ) > gpurun_out/opaddr.log 2>&1
cat gpurun_out/opaddr.log
