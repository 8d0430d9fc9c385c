#!/bin/bash
python tools/gang_ab.py 4736 300 4 32:nomin 32:noparity:nomin > gpurun_out/r02_ab22.log 2>&1
python tools/gang_ab.py 2800 300 4 32:noparity:nomin >> gpurun_out/r02_ab22.log 2>&1
python tools/gang_ab.py 2000 300 4 32:noparity:nomin >> gpurun_out/r02_ab22.log 2>&1
cat gpurun_out/r02_ab22.log
python -m pytest tests/test_gpu_suspend.py tests/test_gpu_parity.py -q > gpurun_out/r02j_pytest.log 2>&1; tail -2 gpurun_out/r02j_pytest.log
python bench.py > gpurun_out/r02j_bench.json 2> gpurun_out/r02j_bench.err; cat gpurun_out/r02j_bench.json
