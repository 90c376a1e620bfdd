#!/bin/bash
# round 2: new planner defaults (no multicast, no ping-pong, one tile per stage at H stride 1) -- GPU suite + bench
mkdir -p gpurun_out
( timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
  timeout 900 python bench.py --steps 50 --warmup 5 --no-e2e --cpu-seconds 3 | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['value']), d['ms_per_step'], d['variants']['fold_speedup_vs_zeropad']); [print(k, round(v['fold']['ms'],4), round(v['fold']['images_per_s']), round(v['fold']['hbm_roofline_frac'],3), round(v['fold']['tensor_roofline_frac'],3), v.get('fold_speedup_vs_zeropad_cin8')) for k, v in d['configs'].items() if not k.startswith('_')]"
) > gpurun_out/r2u.log 2>&1
cat gpurun_out/r2u.log
