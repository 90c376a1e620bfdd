#!/bin/bash
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  echo "=== $tool"
  timeout 900 compute-sanitizer --tool $tool --print-limit 10 python tools/sanitize.py 2>&1 | grep -v "^=========     \(Host Frame\|in \)" | head -60
done > gpurun_out/sanitize.log 2>&1
cat gpurun_out/sanitize.log
