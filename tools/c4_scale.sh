# C4 (MAG240M shape, 3 layers, 768-d fp16 paper features) at 1, 2, 4 GPUs: bench lines in gpurun_out/
mkdir -p gpurun_out
S=${C4_SCALE:-0.02}
timeout 900 python bench.py --workload c4 --scale $S --steps 50 --warmup 5 > gpurun_out/c4_n1.json 2> gpurun_out/c4_n1.err
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29$((800+N)) bench.py --workload c4 --scale $S --gpus $N --steps 50 --warmup 5 > gpurun_out/c4_n$N.json 2> gpurun_out/c4_n$N.err
done
