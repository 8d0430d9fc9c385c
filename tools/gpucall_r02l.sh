#!/bin/bash
python tools/gang_ab.py 4736 300 4 32:noparity:nomin:lib=build/variants/libmfsim_b200_gprof.so > gpurun_out/r02_ab25.log 2>&1
grep -v gangprof gpurun_out/r02_ab25.log
grep gangprof gpurun_out/r02_ab25.log | tail -296 | python -c "
import sys,re
v=[float(re.search(r'busy share ([0-9.]+)',l).group(1)) for l in sys.stdin]
print('final gang busy share over',len(v),'blocks: mean',round(sum(v)/len(v),3),'min',min(v),'max',max(v))"
python tools/gang_ab.py 4736 300 4 32:noparity:nomin:MFSIM_GANG=10:MFSIM_GANG_BLOCKS=3:MFSIM_GANG_MINW=4 32:noparity:nomin
