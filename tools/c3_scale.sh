mkdir -p gpurun_out
python bench.py --model rgat --steps 50 --warmup 5 > gpurun_out/c3_n1.json 2> gpurun_out/c3_n1.err; tail -c 400 gpurun_out/c3_n1.json
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29$((500+N)) bench.py --model rgat --gpus $N --steps 50 --warmup 5 > gpurun_out/c3_n$N.json 2> gpurun_out/c3_n$N.err
  tail -c 300 gpurun_out/c3_n$N.json; tail -3 gpurun_out/c3_n$N.err
done
