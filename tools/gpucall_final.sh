#!/bin/bash
# round-2 final build: GPU tier, smoke, bench, launch list
python -m pytest tests -m gpu -q > gpurun_out/final3_pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/final3_pytest_gpu.log
tail -2 gpurun_out/final3_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final3_smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/final3_smoke.log
cat gpurun_out/final3_smoke.log
python bench.py > gpurun_out/final3_bench.json 2> gpurun_out/final3_bench.err; echo "bench_rc=$?"
cat gpurun_out/final3_bench.json
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/final3_bench_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/final3_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/final3_ncu_launches.log 2>&1
echo "ncu_launches_rc=$?"
