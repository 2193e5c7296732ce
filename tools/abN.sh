# A/B of library variants at N GPUs (torchrun, one rank per GPU): VARIANTS, N, ROUNDS
for r in $(seq ${ROUNDS:-1}); do
  for v in ${VARIANTS:-base}; do
    if [ "$v" = base ]; then export HETGPU_LIB=; else export HETGPU_LIB=$PWD/paper_2408_09697_b200/libhetgpu_$v.so; fi
    python -m torch.distributed.run --nnodes=1 --nproc-per-node ${N:-2} --master-addr 127.0.0.1 --master-port 29511 \
      bench.py --gpus ${N:-2} --steps ${STEPS:-100} --warmup 5 ${BENCH_ARGS:-} 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']/1e9,4), round(d['ms_per_step'],4), round(d['e2e']['value']/1e9,4), {k: v for k, v in d['kernel_us_per_step'].items() if k.startswith(('replica', 'agg'))})"
  done
done
