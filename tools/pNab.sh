runN() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus $1 --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('p=$1 $2', round(d['value']/1e9,3), round(d['ms_per_step'],4), round(d['e2e']['value']/1e9,3))"; }
for i in 1 2; do
  HETGPU_LIB=paper_2408_09697_b200/libhetgpu_prev.so runN 2 prev
  runN 2 new
  HETGPU_LIB=paper_2408_09697_b200/libhetgpu_prev.so runN 4 prev
  runN 4 new
done
