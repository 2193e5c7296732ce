# A/B of the gather grid sizes after the 5-row batch change (HG_GATHER_WAVES 16 vs 8 / 24 first; then 24 / 32; HG_CSC_WAVES 12)
one() { HETGPU_LIB=$1 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernel_us_per_step']; r=d['roofline']['kernels']; print('$2', round(d['value']/1e9,4), round(d['ms_per_step'],4), round(d['e2e']['value']/1e9,4), 'agg', k['aggregate'], round(r['aggregate']['frac'],3), 'csc', k['csc_gather'], round(r['csc_gather']['frac'],3))"; }
for i in 1 2 3; do
  one paper_2408_09697_b200/libhetgpu.so base
  one paper_2408_09697_b200/libhetgpu_gw32.so gw32
  one paper_2408_09697_b200/libhetgpu_gw24.so gw24
  one paper_2408_09697_b200/libhetgpu_gw24cw12.so gw24cw12
done
