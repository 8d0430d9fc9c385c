# GPU call: BASELINE-config parity (configs[0], [1], [4]), the sweep driver, single-instance latency
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_baseline_configs.py tests/test_sweep_run.py -m gpu -x -q --durations=5 > gpurun_out/pytest_baseline.log 2>&1; echo "pytest=$?"
timeout 900 python tools/dev_timing.py 2000 1,148 > gpurun_out/dev_timing.log 2>&1; echo "timing=$?"
tail -15 gpurun_out/pytest_baseline.log; cat gpurun_out/dev_timing.log
