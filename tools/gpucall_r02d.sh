#!/bin/bash
# A/B: block-level first claims + load-aware claim order vs the previous build
python tools/gang_ab.py 4736 300 4 32:noparity:lib=build/variants/libmfsim_b200_prev.so 32 \
   32:noparity:lib=build/variants/libmfsim_b200_prev.so 32:noparity > gpurun_out/r02_ab10.log 2>&1
cat gpurun_out/r02_ab10.log
