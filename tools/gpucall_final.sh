# GPU call: final product -- gpu tests, smoke, default bench, ncu launch list + full capture
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --durations=4 > gpurun_out/pytest_final.log 2>&1; echo "pytest=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "smoke=$?"
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench=$?"
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 600 $B > gpurun_out/bench_final_nocpu.json 2> gpurun_out/bench_final_nocpu.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv $B > gpurun_out/ncu_launch_final.log 2>&1; echo "ncu_launch=$?"
timeout 300 python tools/profile_batch.py 4736 2000 200 > gpurun_out/pb_final_plain.log 2>&1 && \
timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:mfsim_engine -c 1 -o gpurun_out/prof_final_engine python tools/profile_batch.py 4736 2000 200 > gpurun_out/ncu_final_full.log 2>&1; echo "ncu_full=$?"
tail -4 gpurun_out/pytest_final.log; cat gpurun_out/smoke_final.log gpurun_out/bench_final.json gpurun_out/pb_final_plain.log
