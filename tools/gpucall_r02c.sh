#!/bin/bash
# one-warp latency of configs[2] Karuna (shared-memory slot demand + L1 carveout
# for sparse launches) and the gang bench with the same build
for pol in karuna fs mfs; do timeout 600 python tools/phase_profile_budget.py build/libmfsim_b200_prof.so $pol 200000; done
python tools/gang_ab.py 4736 300 4 32 1:noparity > gpurun_out/r02_ab9.log 2>&1
cat gpurun_out/r02_ab9.log
