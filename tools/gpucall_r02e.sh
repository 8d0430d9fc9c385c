#!/bin/bash
# A/B: per-lane sorted cap lists (MF_LANE_CAPS) vs the per-round cap scan, on
# the gang bench, the one-warp kernel and a lone configs[2] Karuna warp
python tools/gang_ab.py 4736 300 4 32:noparity 32:lib=build/variants/libmfsim_b200_lanecaps.so \
  1:noparity 1:noparity:lib=build/variants/libmfsim_b200_lanecaps.so > gpurun_out/r02_ab11.log 2>&1
cat gpurun_out/r02_ab11.log
for lib in build/libmfsim_b200_prof.so build/variants/libmfsim_b200_proflc.so; do
  timeout 600 python tools/phase_profile_budget.py $lib karuna 200000
done
for v in gprof gproflc; do
  python tools/gang_ab.py 4736 300 4 32:noparity:lib=build/variants/libmfsim_b200_$v.so > gpurun_out/r02_ab11_$v.log 2>&1
  grep -v gangprof gpurun_out/r02_ab11_$v.log
  grep gangprof gpurun_out/r02_ab11_$v.log | tail -148 | python -c "
import sys,re
v=[float(re.search(r'busy share ([0-9.]+)',l).group(1)) for l in sys.stdin]
print('$v gang busy share over',len(v),'blocks: mean',round(sum(v)/len(v),3),'min',min(v),'max',max(v))"
done
# adaptive gang size for batches below 148 x 32 instances (2800 = a configs[3] rank on 4 GPUs)
python tools/gang_ab.py 2800 300 4 1:noparity 32:noparity:nomin > gpurun_out/r02_ab12.log 2>&1
cat gpurun_out/r02_ab12.log
