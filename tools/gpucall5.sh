# GPU call: gpu tests (cap-sorted walk, sequential Karuna demand), A/B vs the previous best, phases
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --durations=6 > gpurun_out/pytest_gpu5.log 2>&1; echo "pytest=$?"
P=paper_2603_17456_b200/libmfsim_b200.so
V=build/variants
timeout 600 python tools/ab_variants.py 2368 300 4 $V/libmfsim_b200_u1.so $P $V/libmfsim_b200_u1.so:3108 $P:3108 > gpurun_out/ab5.log 2>&1; echo "ab=$?"
timeout 600 python tools/phase_profile.py 300 fs,karuna,mfs 0.7 > gpurun_out/phase5.log 2>&1; echo "phase=$?"
tail -10 gpurun_out/pytest_gpu5.log; cat gpurun_out/ab5.log gpurun_out/phase5.log
