#!/bin/bash
# round 2: PDL + lean call path -- GPU suite, batch-1 host/device breakdown with and without PDL, bench A/B
mkdir -p gpurun_out
( timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
  timeout 300 python tools/host_path_probe.py
  WF_PDL=0 timeout 300 python tools/host_path_probe.py
  timeout 120 python tools/latency_b1.py
  for p in 1 0; do WF_PDL=$p timeout 400 python bench.py --steps 50 --warmup 5 --no-cpu --no-variants --no-e2e --no-verify > gpurun_out/r2c_bench_pdl$p.log 2>&1; python - <<PY
import json
d=json.loads([l for l in open("gpurun_out/r2c_bench_pdl$p.log") if l.startswith("{")][-1])
print("pdl $p", round(d["value"]), d["ms_per_step"], {k: (v["fold"]["ms"], round(v["fold"]["images_per_s"])) for k, v in d["configs"].items() if not k.startswith("_")})
PY
  done
) > gpurun_out/r2c.log 2>&1
cat gpurun_out/r2c.log
