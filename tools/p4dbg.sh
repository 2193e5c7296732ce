run4() { python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 4 --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/p4_$1.json; python -c "import json; d=json.load(open('gpurun_out/p4_$1.json')); print('$1', round(d['value']/1e9,3), round(d['ms_per_step'],4)); print({k:v for k,v in d['kernel_us_per_step'].items() if k.startswith('replica')})"; }
run4 cur
HG_DBG_NOREMOTEW=1 run4 noremotew
