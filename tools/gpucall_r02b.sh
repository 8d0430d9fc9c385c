#!/bin/bash
# A/B: Karuna cap-sorted prefix walk (register bitonic sort per class) vs the
# per-round cap scan, on the gang bench and on one warp (configs[2] Karuna)
python tools/gang_ab.py 4736 300 4 32:noparity 32:lib=build/variants/libmfsim_b200_capsort.so \
  1:noparity 1:noparity:lib=build/variants/libmfsim_b200_capsort.so > gpurun_out/r02_ab8.log 2>&1
cat gpurun_out/r02_ab8.log
for lib in build/libmfsim_b200_prof.so build/variants/libmfsim_b200_profcs.so; do
  timeout 600 python tools/phase_profile_budget.py $lib karuna 200000
done
