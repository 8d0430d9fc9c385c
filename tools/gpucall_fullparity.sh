# GPU call: BASELINE configs[2] (ft128, 100k requests x 5 policies x 3 seeds) and configs[4]
# (4096-GPU fabric, heavy-tailed trace) against the reference's digests, one launch
mkdir -p gpurun_out
MFSIM_FULL_PARITY=1 timeout 7000 python -m pytest tests/test_baseline_configs.py -m gpu -k "3_and_5" -x -q -s > gpurun_out/full_parity.log 2>&1; echo "full_parity=$?"
tail -25 gpurun_out/full_parity.log
