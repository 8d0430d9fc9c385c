#!/bin/bash
# final-build validation (GPU tier, smoke, bench) + A/B of two 16-warp gangs per SM
python -m pytest tests -m gpu -q > gpurun_out/r02i_pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r02i_pytest_gpu.log
tail -2 gpurun_out/r02i_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02i_smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/r02i_smoke.log
cat gpurun_out/r02i_smoke.log
python bench.py > gpurun_out/r02i_bench.json 2> gpurun_out/r02i_bench.err; echo "bench_rc=$?"
cat gpurun_out/r02i_bench.json
python tools/gang_ab.py 4736 300 4 32:noparity 16:noparity:nomin:MFSIM_GANG_BLOCKS=2 32:noparity > gpurun_out/r02_ab19.log 2>&1
cat gpurun_out/r02_ab19.log
