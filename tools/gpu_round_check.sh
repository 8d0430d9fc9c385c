mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/s4_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s4_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s4_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s4_smoke.log
timeout 600 python bench.py > gpurun_out/s4_bench.json 2> gpurun_out/s4_bench.err; echo "bench rc=$?" >> gpurun_out/s4_bench.err
MFSIM_FULL_PARITY=1 timeout 2400 python -m pytest tests/test_baseline_configs.py -m gpu -k config_5 -x -q -s > gpurun_out/s4_parity_config5.log 2>&1; echo "cfg5 rc=$?" >> gpurun_out/s4_parity_config5.log
