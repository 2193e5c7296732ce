# C5 (IGB-HET shape, 1024-d fp16 features on every type) at 1, 2, 4 GPUs: bench lines in gpurun_out/
mkdir -p gpurun_out
S=${C5_SCALE:-0.05}
timeout 900 python bench.py --workload c5 --scale $S --steps 50 --warmup 5 > gpurun_out/c5_n1.json 2> gpurun_out/c5_n1.err; tail -c 300 gpurun_out/c5_n1.json; tail -2 gpurun_out/c5_n1.err
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29$((700+N)) bench.py --workload c5 --scale $S --gpus $N --steps 50 --warmup 5 > gpurun_out/c5_n$N.json 2> gpurun_out/c5_n$N.err
  tail -c 200 gpurun_out/c5_n$N.json; grep -v "^\*\|OMP" gpurun_out/c5_n$N.err | tail -2
done
