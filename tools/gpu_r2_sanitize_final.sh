#!/bin/bash
# compute-sanitizer over the final build: memcheck / synccheck on 120 random geometries x knobs
# (tools/sanitize_fuzz.py), plus the fixed sanitizer set (tools/gpu_sanitize.sh: every producer).
mkdir -p gpurun_out
for tool in memcheck synccheck; do
  echo "=== $tool (sanitize_fuzz 120)"
  timeout 1500 compute-sanitizer --tool $tool --print-limit 10 python tools/sanitize_fuzz.py 120 2>&1 | grep -v "^=========     \(Host Frame\|in \)" | tail -8
done > gpurun_out/sanitize_fuzz_final.log 2>&1
bash tools/gpu_sanitize.sh > /dev/null 2>&1
grep -E "=== |ERROR SUMMARY|sanitize fuzz|Error|error" gpurun_out/sanitize_fuzz_final.log gpurun_out/sanitize.log | head -30
