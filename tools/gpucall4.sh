# GPU call: gpu test tier (tiled filling, unroll 1), A/B of engine builds, per-phase cycle profile
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest=$?"
P=paper_2603_17456_b200/libmfsim_b200.so
V=build/variants
timeout 600 python tools/ab_variants.py 2368 300 4 $V/libmfsim_b200_u1.so $P $V/libmfsim_b200_tiled_u4.so $P:3108 $V/libmfsim_b200_u1.so:3108 > gpurun_out/ab4.log 2>&1; echo "ab=$?"
timeout 600 python tools/phase_profile.py 300 fs,sjf,edf,karuna,mfs 0.7 > gpurun_out/phase4.log 2>&1; echo "phase=$?"
tail -12 gpurun_out/pytest_gpu4.log; cat gpurun_out/ab4.log gpurun_out/phase4.log
