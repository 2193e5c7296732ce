# A/B of the forward gather's neighbour batch (HG_GATHER_BATCH; 8, 5, 10 measured first, then 4, 5, 6), backward gather at 2 edges in flight
one() { HETGPU_LIB=$1 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernel_us_per_step']; r=d['roofline']['kernels']; print('$2', round(d['value']/1e9,4), round(d['ms_per_step'],4), round(d['e2e']['value']/1e9,4), 'agg', k['aggregate'], round(r['aggregate']['frac'],3), 'csc', k['csc_gather'], round(r['csc_gather']['frac'],3))"; }
for i in 1 2 3; do
  one paper_2408_09697_b200/libhetgpu_c2g4.so c2g4
  one paper_2408_09697_b200/libhetgpu_c2g5.so c2g5
  one paper_2408_09697_b200/libhetgpu_c2g6.so c2g6
done
