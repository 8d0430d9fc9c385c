# GPU call: BASELINE configs[2] (ft128, 100k requests; fs/sjf/edf/mfs x 3 seeds) vs the reference's digests
mkdir -p gpurun_out
MFSIM_FULL_PARITY=1 timeout 3300 python -m pytest tests/test_baseline_configs.py -m gpu -k "config_3_bit_exact" -x -q -s > gpurun_out/parity_cfg3.log 2>&1; echo "cfg3=$?"
tail -16 gpurun_out/parity_cfg3.log
