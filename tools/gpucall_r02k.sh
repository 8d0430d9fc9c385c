#!/bin/bash
# A/B: a fourth gang barrier (between popping the event and its handler);
# ncu capture of the final gang kernel
python tools/gang_ab.py 4736 300 4 32:noparity:nomin 32:nomin:lib=build/variants/libmfsim_b200_split4.so 32:noparity:nomin > gpurun_out/r02_ab23.log 2>&1
cat gpurun_out/r02_ab23.log
python tools/profile_batch.py 4736 2000 200 > gpurun_out/r02k_prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:mfsim -c 1 \
  -o gpurun_out/r02k_gang python tools/profile_batch.py 4736 2000 200 > gpurun_out/r02k_prof_ncu.log 2>&1
echo "ncu_rc=$?"
tail -1 gpurun_out/r02k_prof_plain.log
