#!/bin/bash
# A/B: capped filling rounds settled from the last pass's two smallest caps (MF_CAP_TOP2)
python tools/gang_ab.py 4736 300 4 32:noparity:nomin 32:nomin:lib=build/variants/libmfsim_b200_top2.so 32:noparity:nomin 32:noparity:nomin:lib=build/variants/libmfsim_b200_top2.so > gpurun_out/r02_ab26.log 2>&1
cat gpurun_out/r02_ab26.log
for lib in build/libmfsim_b200_prof.so build/variants/libmfsim_b200_proft2.so; do
  timeout 600 python tools/phase_profile_budget.py $lib karuna 200000
done
