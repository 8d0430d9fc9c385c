# GPU call: A/B of route-count ILP and a smaller on-chip slot plan (more resident warps)
mkdir -p gpurun_out
V=build/variants
timeout 1500 python tools/ab_variants.py 3108 300 4 $V/libmfsim_b200_base8.so $V/libmfsim_b200_routeilp.so $V/libmfsim_b200_s128.so $V/libmfsim_b200_s128.so:4144 $V/libmfsim_b200_base8.so > gpurun_out/ab9.log 2>&1; echo "ab=$?"
cat gpurun_out/ab9.log
