#!/bin/bash
# R50 b8192 headline under the power cap (200-step bench runs) for planner
# knobs that trade A-operand traffic against MMA work: energy per image, not
# short-run speed, decides the sustained number.
# KNOBS="A=1,B=2" (comma-separated, the empty default first) overrides the set; TAG names the log.
mkdir -p gpurun_out
IFS=',' read -r -a knobs <<< "${KNOBS:-,WF_TPS=4,WF_KPAIR=0,WF_TPS=1}"
( for rep in 1 2; do
  for env in "${knobs[@]}"; do
    echo "== rep $rep env '$env'"
    env $env timeout 120 python bench.py --steps 200 --warmup 5 --no-e2e --no-cpu --no-variants --no-verify 2>&1 \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']), round(d['ms_per_step'],3), d['clocks'])"
  done
done ) > gpurun_out/sustained_knobs${TAG}.log 2>&1
cat gpurun_out/sustained_knobs${TAG}.log
