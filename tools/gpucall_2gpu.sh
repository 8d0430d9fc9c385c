# 2-GPU call: bench weak scaling under torchrun, and the sharded sweep driver with its NCCL gather
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533"
timeout 900 $TR bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_2gpu.json 2> gpurun_out/bench_2gpu.err; echo "bench2=$?"
printf 'workload.request_count = 300\n' > /tmp/extra.conf
cat tests/configs/cluster8.conf /tmp/extra.conf > /tmp/c8.conf
ARGS="--config /tmp/c8.conf --policies fs,sjf,edf,karuna,mfs,aalo --rates 6,10 --seeds 1,2"
timeout 900 $TR -m paper_2603_17456_b200.sweep_run $ARGS --out gpurun_out/sweep2 > gpurun_out/sweep2.log 2>&1; echo "sweep2=$?"
timeout 900 python -m paper_2603_17456_b200.sweep_run $ARGS --out gpurun_out/sweep1 > gpurun_out/sweep1.log 2>&1; echo "sweep1=$?"
cmp gpurun_out/sweep1/sweep.csv gpurun_out/sweep2/sweep.csv && echo "sweep.csv identical across 1 and 2 ranks"
rm -rf gpurun_out/sweep1/*/ gpurun_out/sweep2/*/
cat gpurun_out/bench_2gpu.json; tail -3 gpurun_out/bench_2gpu.err; head -5 gpurun_out/sweep2/sweep.csv
