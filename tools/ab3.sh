one() { HETGPU_LIB=$1 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']['kernels']; print('$2', round(d['value']/1e9,4), round(d['ms_per_step'],4), round(d['e2e']['value']/1e9,4), 'agg', round(r['aggregate']['frac'],3), 'csc', round(r['csc_gather']['frac'],3))"; }
for i in 1 2; do
  one paper_2408_09697_b200/libhetgpu.so w16
  one paper_2408_09697_b200/libhetgpu_w8.so w8
  one paper_2408_09697_b200/libhetgpu_w24.so w24
done
