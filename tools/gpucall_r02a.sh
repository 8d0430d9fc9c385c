#!/bin/bash
# A/B: resumable filling units vs the event-level gang; gang busy share; the
# single-warp phase profile of BASELINE configs[2] Karuna (flow-by-flow vs
# bucketed demand)
python tools/gang_ab.py 4736 300 4 32 32:noparity:lib=build/variants/libmfsim_b200_evgang.so \
  32:noparity:lib=build/variants/libmfsim_b200_gprofu.so 1:noparity > gpurun_out/r02_ab7.log 2>&1
grep -v gangprof gpurun_out/r02_ab7.log
grep gangprof gpurun_out/r02_ab7.log | tail -160 | python -c "
import sys,re
v=[float(re.search(r'busy share ([0-9.]+)',l).group(1)) for l in sys.stdin]
print('units gang busy share over',len(v),'blocks: mean',sum(v)/len(v),'min',min(v),'max',max(v))"
for lib in build/libmfsim_b200_prof.so build/variants/libmfsim_b200_profkb.so; do
  timeout 600 python tools/phase_profile_budget.py $lib karuna 200000
done
timeout 300 python tools/phase_profile_budget.py build/libmfsim_b200_prof.so fs 200000
timeout 300 python tools/phase_profile_budget.py build/libmfsim_b200_prof.so mfs 200000
