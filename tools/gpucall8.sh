# GPU call: gpu tests with the lazy cap minima, A/B against the previous product, phases
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --durations=4 > gpurun_out/pytest_gpu8.log 2>&1; echo "pytest=$?"
P=paper_2603_17456_b200/libmfsim_b200.so
V=build/variants
timeout 600 python tools/ab_variants.py 3108 300 4 $V/libmfsim_b200_noaalo_nocapsort.so $P > gpurun_out/ab8.log 2>&1; echo "ab=$?"
timeout 600 python tools/phase_profile.py 300 fs,sjf,edf,karuna,mfs 0.7 > gpurun_out/phase8.log 2>&1; echo "phase=$?"
tail -5 gpurun_out/pytest_gpu8.log; cat gpurun_out/ab8.log gpurun_out/phase8.log
