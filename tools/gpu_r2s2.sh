#!/bin/bash
# round 2: core-column-plane workspace for the re-pitch producer -- parity + AlexNet A/B + split
mkdir -p gpurun_out
( timeout 300 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_stream_order.py tests/test_gpu_run_host.py -q -m gpu -x -k "alexnet or gather or repitch or partial or run_host or stream or order or tf32 or w71 or w50" 2>&1 | tail -3
  for n in 512 2048; do timeout 120 python tools/prof_conv.py alex $n 0 0 50; WF_PLANES=0 timeout 120 python tools/prof_conv.py alex $n 0 0 50; done
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"conv_fold|repitch" --csv --log-file gpurun_out/r2s2_alex.csv python tools/prof_conv.py alex 512 0 0 2 > /dev/null 2>&1; echo "ncu rc $?"
  python - <<'PY'
import csv
rows=list(csv.reader(open("gpurun_out/r2s2_alex.csv")))
h=[i for i,r in enumerate(rows) if r and r[0]=="ID"][0]; H=rows[h]
for r in rows[h+1:]:
    print(r[H.index("ID")], r[H.index("Kernel Name")][:40], r[H.index("Metric Name")], r[H.index("Metric Value")])
PY
) > gpurun_out/r2s2.log 2>&1
cat gpurun_out/r2s2.log
