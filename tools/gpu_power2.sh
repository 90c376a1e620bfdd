#!/bin/bash
mkdir -p gpurun_out
( echo "== default"; timeout 100 python tools/power_probe.py 8192 3 0,0x1300
echo "== WF_CTA_PAIR=1"; WF_CTA_PAIR=1 timeout 100 python tools/power_probe.py 8192 3 0
echo "== WF_TPS=1"; WF_TPS=1 timeout 100 python tools/power_probe.py 8192 3 0
nvidia-smi --query-gpu=power.draw,clocks.sm,temperature.gpu --format=csv
) > gpurun_out/power2.log 2>&1
cat gpurun_out/power2.log
