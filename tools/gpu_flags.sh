#!/bin/bash
# Component timing via the kernel's profiling switches (R50 conv1, n=2048):
# 0x100 skip MMA, 0x200 skip epilogue, 0x400 skip global store, 0x800 skip TMEM load, 0x1000 TMA-store epilogue
mkdir -p gpurun_out
for fl in 0 0x100 0x200 0x400 0x800 0x1000 0x1400 0x500; do timeout 60 python tools/prof_conv.py r50 2048 0 0 20 $fl; done > gpurun_out/flags.log 2>&1
for gs in 1 2 4; do timeout 60 python tools/prof_conv.py r50 2048 8 $gs 20 0; done >> gpurun_out/flags.log 2>&1
cat gpurun_out/flags.log
