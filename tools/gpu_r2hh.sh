#!/bin/bash
mkdir -p gpurun_out
for tool in memcheck synccheck; do
  echo "=== $tool"
  timeout 1200 compute-sanitizer --tool $tool --print-limit 10 python tools/sanitize_fuzz.py 40 2>&1 | grep -v "^=========     \(Host Frame\|in \)" | tail -15
done > gpurun_out/r2hh_sanitize_fuzz.log 2>&1
cat gpurun_out/r2hh_sanitize_fuzz.log
