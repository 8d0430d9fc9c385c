# GPU call: A/B of resident warps per SM (on-chip slot plan 128 / 112 / 96)
mkdir -p gpurun_out
V=build/variants
timeout 1500 python tools/ab_variants.py 4144 300 4 $V/libmfsim_b200_s128f.so $V/libmfsim_b200_s128f.so:4292 $V/libmfsim_b200_s112.so:4588 $V/libmfsim_b200_s96.so:4736 $V/libmfsim_b200_s96.so:4144 > gpurun_out/ab11.log 2>&1; echo "ab=$?"
cat gpurun_out/ab11.log
