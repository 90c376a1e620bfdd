#!/bin/bash
# device soak (tools/fuzz_soak.py) with a host-memory watchdog on its exact PID
mkdir -p gpurun_out
SECS=${1:-1200}; SEED=${2:-1000}; EXTRA=${3:-}
timeout $((SECS + 300)) python tools/fuzz_soak.py --seconds $SECS --seed $SEED $EXTRA > gpurun_out/soak_$SEED.log 2>&1 &
P=$!
while kill -0 $P 2>/dev/null; do
  avail=$(free -m | awk '/Mem/{print $7}')
  if [ "$avail" -lt 30000 ]; then echo "WATCHDOG: host memory low ($avail MB), killing $P" >> gpurun_out/soak_$SEED.log; kill -9 $P; fi
  sleep 1
done
wait $P; echo "rc=$?" >> gpurun_out/soak_$SEED.log
grep -E "^FAIL|WATCHDOG" gpurun_out/soak_$SEED.log | head -20; tail -2 gpurun_out/soak_$SEED.log | cut -c1-1500
