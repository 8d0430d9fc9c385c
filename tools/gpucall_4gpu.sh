#!/bin/bash
# 4-GPU box call: weak-scaling bench, then BASELINE configs[3] in full (all
# 11,200 cells, sweep_run on 4 ranks, time-sliced run-to-completion batches),
# then the sample of per-request TTFTs the reference check reads here.
mkdir -p gpurun_out/cfg3_r02c
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm --format=csv
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 4 > gpurun_out/r02c_bench_4gpu.json 2> gpurun_out/r02c_bench_4gpu.err
echo bench4=$?
t0=$(date +%s.%N)
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 \
  -m paper_2603_17456_b200.sweep_run --grid configs3 --no-reports --out gpurun_out/cfg3_r02c \
  > gpurun_out/cfg3_r02c.log 2>&1
echo cfg3=$?
t1=$(date +%s.%N)
echo "configs[3] full grid on 4 GPUs: wall $(python -c "print(round($t1-$t0,1))") s (torchrun start to exit)" | tee -a gpurun_out/cfg3_r02c.log
python tools/check_sweep_sample.py extract gpurun_out/cfg3_r02c/ttft.npz gpurun_out/cfg3_r02c/ttft_sample.npz
rm -f gpurun_out/cfg3_r02c/ttft.npz
cmp gpurun_out/cfg3_r02c/sweep.csv profiles/r02_cfg3_full_4gpu/sweep.csv && echo "sweep.csv byte-identical to the first round-2 run"
cat gpurun_out/r02c_bench_4gpu.json
tail -8 gpurun_out/cfg3_r02c.log
