timeout 120 python tools/cmp_modes.py
for fl in 0 0x1000 0x1100 0x1200; do timeout 60 python tools/prof_conv.py r50 1024 0 0 20 $fl; done
timeout 60 python tools/prof_conv.py r50 8192 0 0 10 0x1000
for c in vgg mnv2; do timeout 60 python tools/prof_conv.py $c 1024 0 0 10 0; timeout 60 python tools/prof_conv.py $c 1024 0 0 10 0x1000; done
