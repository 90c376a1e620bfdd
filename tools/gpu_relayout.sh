#!/bin/bash
mkdir -p gpurun_out
( timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for nr in 0 1; do echo "== no_relayout=$nr"; if [ $nr = 1 ]; then export WF_NO_RELAYOUT=1; fi
for fl in 0 0x300 0x200; do timeout 60 python tools/prof_conv.py alex 1024 0 0 20 $fl; done; done
unset WF_NO_RELAYOUT
for kp in 0; do WF_KPAIR=$kp timeout 60 python tools/prof_conv.py alex 1024 0 0 20 0; done
) > gpurun_out/relayout.log 2>&1
cat gpurun_out/relayout.log
