for fl in 0 0x100 0x500 0x900 0xD00 0x200; do timeout 60 python tools/prof_conv.py r50 1024 0 0 20 $fl; done
