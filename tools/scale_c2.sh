# C2 scaling lines (bench contract, weak scaling) on the GPUs of one box, then the
# multi-GPU tests; outputs under gpurun_out/
mkdir -p gpurun_out
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29$((600+N)) bench.py --gpus $N --steps 100 --warmup 10 > gpurun_out/scale_n$N.json 2> gpurun_out/scale_n$N.err
  tail -c 250 gpurun_out/scale_n$N.json
done
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_rgat.py -m gpu -q 2>&1 | tail -3
