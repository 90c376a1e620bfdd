#!/bin/bash
# round 2: stream-order tests under PDL; AlexNet time split (re-pitch pass vs conv) and DRAM bytes
mkdir -p gpurun_out
( timeout 600 python -m pytest tests/test_gpu_stream_order.py -q -m gpu 2>&1 | tail -3
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"conv_fold|repitch" --csv --log-file gpurun_out/r2d_alex_split.csv python tools/prof_conv.py alex 512 0 0 3 > /dev/null 2>&1; echo "ncu rc $?"
  python - <<'PY'
import csv
rows=list(csv.reader(open("gpurun_out/r2d_alex_split.csv")))
h=[i for i,r in enumerate(rows) if r and r[0]=="ID"][0]; H=rows[h]
for r in rows[h+1:]:
    print(r[H.index("ID")], r[H.index("Kernel Name")][:40], r[H.index("Metric Name")], r[H.index("Metric Value")])
PY
  for n in 512 2048; do timeout 120 python tools/prof_conv.py alex $n 0 0 50; WF_GATHER=1 timeout 120 python tools/prof_conv.py alex $n 0 0 50; done
) > gpurun_out/r2d.log 2>&1
cat gpurun_out/r2d.log
