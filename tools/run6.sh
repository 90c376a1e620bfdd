timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -3
timeout 120 python tools/cmp_modes.py
for fl in 0 0x100 0x200; do timeout 60 python tools/prof_conv.py r50 1024 0 0 20 $fl; done
timeout 60 python tools/prof_conv.py r50 8192 0 0 10 0
for c in vgg mnv2; do timeout 60 python tools/prof_conv.py $c 1024 0 0 10 0; done
