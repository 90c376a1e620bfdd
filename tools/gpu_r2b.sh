#!/bin/bash
# round 2: batch-1 latency breakdown, PCIe ceiling of the e2e leg, e2e chunk sweep
mkdir -p gpurun_out
( timeout 120 python tools/latency_b1.py
  timeout 120 python tools/pcie_probe.py 822
  timeout 120 python tools/pcie_probe.py 154
  for c in 256 1024 2048; do timeout 400 python bench.py --steps 20 --warmup 3 --no-cpu --no-variants --no-configs --no-verify --e2e-chunk $c | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('chunk', $c, d['e2e']['value'], d['e2e']['ms_per_step'])"; done
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:conv_fold -s 30 -c 1 -o gpurun_out/r2b_b1_tf32 -f python tools/latency_b1.py > gpurun_out/r2b_ncu_b1.log 2>&1; echo "ncu rc $?"
) > gpurun_out/r2b.log 2>&1
cat gpurun_out/r2b.log
