# GPU call: gpu tests (topology-image key fix), A/B isolating the Aalo code and the cap sort
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --durations=6 > gpurun_out/pytest_gpu6.log 2>&1; echo "pytest=$?"
P=paper_2603_17456_b200/libmfsim_b200.so
V=build/variants
timeout 900 python tools/ab_variants.py 3108 300 4 $V/libmfsim_b200_u1.so $P $V/libmfsim_b200_nocapsort.so $V/libmfsim_b200_noaalo.so $V/libmfsim_b200_noaalo_nocapsort.so $V/libmfsim_b200_u1.so > gpurun_out/ab6.log 2>&1; echo "ab=$?"
tail -10 gpurun_out/pytest_gpu6.log; cat gpurun_out/ab6.log
