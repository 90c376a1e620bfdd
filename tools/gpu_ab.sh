#!/bin/bash
# GPU parity + A/B timings: AlexNet CTA pair vs not, R50 default
mkdir -p gpurun_out
( timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -5
for pr in 0 1; do echo "== WF_CTA_PAIR=$pr"; WF_CTA_PAIR=$pr timeout 60 python tools/prof_conv.py alex 512 0 0 20 0; WF_CTA_PAIR=$pr timeout 60 python tools/prof_conv.py alex 2048 0 0 20 0; done
timeout 60 python tools/prof_conv.py r50 8192 0 0 20 0
) > gpurun_out/ab.log 2>&1
cat gpurun_out/ab.log
