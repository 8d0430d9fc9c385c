# one GPU call: gpu tests, smoke, default bench, ncu launch list of a bench run, ncu --set full of the engine kernel
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench=$?"
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 600 $B > gpurun_out/bench_nocpu.json 2> gpurun_out/bench_nocpu.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1; echo "ncu_launch=$?"
timeout 300 python tools/profile_batch.py 1184 2000 200 > gpurun_out/pb_plain.log 2>&1 && \
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:mfsim_engine -c 1 -o gpurun_out/prof_engine python tools/profile_batch.py 1184 2000 200 > gpurun_out/ncu_full.log 2>&1; echo "ncu_full=$?"
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/bench.json
