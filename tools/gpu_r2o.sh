#!/bin/bash
# round 2: B load before griddepcontrol.wait (operand epoch gates PDL) -- stream-order tests, batch-1 latency, bench sanity
mkdir -p gpurun_out
( timeout 600 python -m pytest tests/test_gpu_stream_order.py tests/test_gpu_run_host.py -q -m gpu 2>&1 | tail -3
  timeout 120 python tools/host_path_probe.py
  timeout 120 python tools/b1_components.py 0
  timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
  timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu --no-variants --no-e2e | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['value']), d['ms_per_step'], {k: (round(v['fold']['ms'],4), v.get('latency_us')) for k, v in d['configs'].items() if not k.startswith('_')})"
) > gpurun_out/r2o.log 2>&1
cat gpurun_out/r2o.log
