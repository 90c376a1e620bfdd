timeout 120 python tools/gpu_quick.py
for gs in 0 2 4; do for fl in 0 0x100 0x200; do timeout 60 python tools/prof_conv.py r50 1024 0 $gs 20 $fl; done; done
for gs in 0 2 4; do timeout 60 python tools/prof_conv.py vgg 256 0 $gs 20; done
for gs in 0 4 8; do timeout 60 python tools/prof_conv.py mnv2 1024 0 $gs 20; done
