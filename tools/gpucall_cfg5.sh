# GPU call: BASELINE configs[4] (4096-GPU fat-tree, heavy-tailed trace; mfs/fs) vs the reference's digests
mkdir -p gpurun_out
MFSIM_FULL_PARITY=1 timeout 3300 python -m pytest tests/test_baseline_configs.py -m gpu -k "config_5" -x -q -s > gpurun_out/parity_cfg5.log 2>&1; echo "cfg5=$?"
tail -8 gpurun_out/parity_cfg5.log
