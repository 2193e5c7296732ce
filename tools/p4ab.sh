run4() { python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 4 --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/p4_$1.json; python -c "import json; d=json.load(open('gpurun_out/p4_$1.json')); print('$1', round(d['value']/1e9,3), round(d['ms_per_step'],4), round(d['e2e']['value']/1e9,3), {k:v for k,v in d['kernel_us_per_step'].items() if k.startswith('replica_adam')})"; }
for i in 1 2; do
run4 r16
HETGPU_LIB=paper_2408_09697_b200/libhetgpu_r8.so run4 r8
done
