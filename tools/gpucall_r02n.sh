#!/bin/bash
# under the seed-grouped claim order: one 32-warp gang vs two 16-warp gangs per SM; ncu capture
python tools/gang_ab.py 4736 300 4 32:noparity:nomin 32:noparity:nomin:MFSIM_GANG_BLOCKS=1 32:noparity:nomin > gpurun_out/r02_ab28.log 2>&1
cat gpurun_out/r02_ab28.log
python tools/profile_batch.py 4736 2000 200 > gpurun_out/r02n_prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:mfsim -c 1 \
  -o gpurun_out/r02n_gang python tools/profile_batch.py 4736 2000 200 > gpurun_out/r02n_prof_ncu.log 2>&1
echo "ncu_rc=$?"
tail -1 gpurun_out/r02n_prof_plain.log
