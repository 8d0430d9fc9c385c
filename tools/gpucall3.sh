# GPU call: full gpu test tier on the product build, then an A/B of engine builds
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/pytest_gpu3.log 2>&1; echo "pytest=$?"
P=paper_2603_17456_b200/libmfsim_b200.so
V=build/variants
timeout 900 python tools/ab_variants.py 2368 300 4 $V/libmfsim_b200_old.so $P $V/libmfsim_b200_u1.so $V/libmfsim_b200_u2.so $P:3108 $V/libmfsim_b200_old.so:3108 $P:1184 > gpurun_out/ab3.log 2>&1; echo "ab=$?"
tail -12 gpurun_out/pytest_gpu3.log; cat gpurun_out/ab3.log
