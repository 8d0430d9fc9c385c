# GPU call: gpu tests (lean/Aalo kernel variants), A/B, default bench, ncu launch list + full capture
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --durations=4 > gpurun_out/pytest_gpu7.log 2>&1; echo "pytest=$?"
P=paper_2603_17456_b200/libmfsim_b200.so
V=build/variants
timeout 600 python tools/ab_variants.py 3108 300 4 $V/libmfsim_b200_noaalo_nocapsort.so $P $V/libmfsim_b200_u1.so > gpurun_out/ab7.log 2>&1; echo "ab=$?"
timeout 900 python bench.py > gpurun_out/bench7.json 2> gpurun_out/bench7.err; echo "bench=$?"
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 600 $B > gpurun_out/bench7_nocpu.json 2> gpurun_out/bench7_nocpu.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches7.csv $B > gpurun_out/ncu_launch7.log 2>&1; echo "ncu_launch=$?"
timeout 300 python tools/profile_batch.py 3108 2000 200 > gpurun_out/pb7_plain.log 2>&1 && \
timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:mfsim_engine -c 1 -o gpurun_out/prof7_engine python tools/profile_batch.py 3108 2000 200 > gpurun_out/ncu7_full.log 2>&1; echo "ncu_full=$?"
tail -6 gpurun_out/pytest_gpu7.log; cat gpurun_out/ab7.log gpurun_out/bench7.json gpurun_out/pb7_plain.log
