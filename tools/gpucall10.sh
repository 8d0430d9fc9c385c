# GPU call: gpu tests, default bench, ncu launch list + full capture of the final engine,
# then BASELINE configs[2] + configs[4] parity (one launch, ~1.5 h)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --durations=4 > gpurun_out/pytest_gpu10.log 2>&1; echo "pytest=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke10.log 2>&1; echo "smoke=$?"
timeout 900 python bench.py > gpurun_out/bench10.json 2> gpurun_out/bench10.err; echo "bench=$?"
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 600 $B > gpurun_out/bench10_nocpu.json 2> gpurun_out/bench10_nocpu.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches10.csv $B > gpurun_out/ncu_launch10.log 2>&1; echo "ncu_launch=$?"
timeout 300 python tools/profile_batch.py 4144 2000 200 > gpurun_out/pb10_plain.log 2>&1 && \
timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:mfsim_engine -c 1 -o gpurun_out/prof10_engine python tools/profile_batch.py 4144 2000 200 > gpurun_out/ncu10_full.log 2>&1; echo "ncu_full=$?"
tail -4 gpurun_out/pytest_gpu10.log; cat gpurun_out/bench10.json gpurun_out/pb10_plain.log
MFSIM_FULL_PARITY=1 timeout 7000 python -m pytest tests/test_baseline_configs.py -m gpu -k "3_and_5" -x -q -s > gpurun_out/full_parity.log 2>&1; echo "full_parity=$?"
tail -25 gpurun_out/full_parity.log
