#!/bin/bash
mkdir -p gpurun_out
( timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for na in 4 2; do echo "== WF_NACC=$na"; export WF_NACC=$na
for c in mnv2 alex; do timeout 60 python tools/prof_conv.py $c 1024 0 0 20 0; done
timeout 60 python tools/prof_conv.py mnv2 1024 0 0 2 0x80000 2>&1 | grep -i issuer | head -1
done
unset WF_NACC
timeout 60 python tools/prof_conv.py r50 8192 0 0 20 0
) > gpurun_out/nacc.log 2>&1
cat gpurun_out/nacc.log
