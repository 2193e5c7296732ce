one() { HETGPU_LIB=paper_2408_09697_b200/libhetgpu.so python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$HG_PRIO', round(d['value']/1e9,4), round(d['ms_per_step'],4), round(d['e2e']['value']/1e9,4))"; }
for i in 1 2; do
  for p in 0,0,0 1,1,0 0,1,0 1,1,1 0,1,1 1,0,1; do HG_PRIO=$p one; done
done
