# 4-GPU call: bench weak scaling under torchrun, then BASELINE configs[3] run in full
# (11,200 cells, ft128, 2000 requests each) sharded over 4 ranks with the final NCCL gather
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541"
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv
timeout 900 $TR bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/bench_4gpu.json 2> gpurun_out/bench_4gpu.err; echo "bench4=$?"
cat gpurun_out/bench_4gpu.json
S=$(date +%s.%N)
timeout 2400 $TR -m paper_2603_17456_b200.sweep_run --grid configs3 --no-reports --out /tmp/cfg3 > gpurun_out/cfg3_full.log 2>&1; echo "cfg3=$?"
E=$(date +%s.%N)
echo "configs[3] full grid on 4 GPUs: wall $(python -c "print(round($E-$S,1))") s (torchrun start to exit)" | tee -a gpurun_out/cfg3_full.log
mkdir -p gpurun_out/cfg3_full && cp /tmp/cfg3/sweep.csv gpurun_out/cfg3_full/
python tools/check_sweep_sample.py extract /tmp/cfg3/ttft.npz gpurun_out/cfg3_full/ttft_sample.npz
tail -6 gpurun_out/cfg3_full.log
