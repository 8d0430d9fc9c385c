#!/bin/bash
# round-2 validation on one B200: GPU tier, smoke, bench, ncu launch list and
# one --set full capture of the gang kernel
python -m pytest tests -m gpu -q > gpurun_out/r02f_pytest_gpu.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r02f_pytest_gpu.log
tail -3 gpurun_out/r02f_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/r02f_smoke.log
cat gpurun_out/r02f_smoke.log
python bench.py > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err; echo "bench_rc=$?"
cat gpurun_out/r02f_bench.json
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02f_bench_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r02f_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02f_ncu_launches.log 2>&1
echo "ncu_launches_rc=$?"
python tools/profile_batch.py 4736 2000 200 > gpurun_out/r02f_prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:mfsim -c 1 \
  -o gpurun_out/r02f_gang python tools/profile_batch.py 4736 2000 200 > gpurun_out/r02f_prof_ncu.log 2>&1
echo "ncu_full_rc=$?"
tail -2 gpurun_out/r02f_prof_plain.log
