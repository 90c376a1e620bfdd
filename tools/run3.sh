timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
for fl in 0 0x100 0x200; do timeout 60 python tools/prof_conv.py r50 1024 0 0 20 $fl; done
timeout 60 python tools/prof_conv.py r50 8192 0 0 10
timeout 60 python tools/prof_conv.py vgg 256 0 0 20
timeout 60 python tools/prof_conv.py mnv2 1024 0 0 20
