#!/bin/bash
mkdir -p gpurun_out
( WF_KPAIR=1 timeout 200 python tools/power_probe.py 8192 3 0,-1,0x1100,0x1200,0x200,0x100
) > gpurun_out/power.log 2>&1
cat gpurun_out/power.log
