#!/bin/bash
# two translation units: lone-warp latency (one-warp kernel with 128 registers)
# and the gang bench (unchanged kernel, re-checked)
for pol in karuna fs mfs; do timeout 600 python tools/phase_profile_budget.py build/libmfsim_b200_prof.so $pol 200000; done
python tools/gang_ab.py 4736 300 4 32 > gpurun_out/r02_ab13.log 2>&1
python tools/gang_ab.py 1184 300 4 1 > gpurun_out/r02_ab13b.log 2>&1
cat gpurun_out/r02_ab13.log gpurun_out/r02_ab13b.log
