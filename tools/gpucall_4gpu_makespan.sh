# 4-GPU call: configs[3] full grid again after the work-proportional SM map for
# run-to-completion launches (makespan), then the device parity tests
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29543"
S=$(date +%s.%N)
timeout 1300 $TR -m paper_2603_17456_b200.sweep_run --grid configs3 --no-reports --out /tmp/cfg3 > gpurun_out/cfg3_full_v2.log 2>&1; echo "cfg3=$?"
E=$(date +%s.%N)
echo "configs[3] full grid on 4 GPUs: wall $(python -c "print(round($E-$S,1))") s (torchrun start to exit)" | tee -a gpurun_out/cfg3_full_v2.log
mkdir -p gpurun_out/cfg3_full_v2 && cp /tmp/cfg3/sweep.csv gpurun_out/cfg3_full_v2/
python tools/check_sweep_sample.py extract /tmp/cfg3/ttft.npz gpurun_out/cfg3_full_v2/ttft_sample.npz
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_sweep_run.py tests/test_capi.py -m gpu -x -q > gpurun_out/pytest_v2.log 2>&1; echo "pytest=$?" >> gpurun_out/pytest_v2.log
tail -3 gpurun_out/pytest_v2.log; grep rank gpurun_out/cfg3_full_v2.log
