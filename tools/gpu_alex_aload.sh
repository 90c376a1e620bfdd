#!/bin/bash
# AlexNet A-producer sensitivity (DESIGN.md 9 item 1): full launch vs residue-0
# boxes only (0x40000, 1/4 of the TMA pieces) vs no A loads (0x1000), with the
# issuer's CTA-0 counters (0x80000).
mkdir -p gpurun_out
( for rep in 1 2; do for fl in 0x80000 0xC0000 0x81000; do
  timeout 60 python tools/prof_conv.py alex 1024 0 0 5 $fl 2>&1 | grep -E "issuer cta0|flags=" | tail -2
done; done ) > gpurun_out/alex_aload.log 2>&1
cat gpurun_out/alex_aload.log
