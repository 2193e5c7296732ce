# A/B of the backward gather's edges in flight (HG_CSC_BATCH: 4, 2, 8 measured first; then 1, 2, 3)
one() { HETGPU_LIB=$1 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernel_us_per_step']; print('$2', round(d['value']/1e9,4), round(d['ms_per_step'],4), round(d['e2e']['value']/1e9,4), 'csc', k['csc_gather'], d['roofline']['kernels']['csc_gather']['frac'])"; }
for i in 1 2 3; do
  one paper_2408_09697_b200/libhetgpu.so csc4
  one paper_2408_09697_b200/libhetgpu_csc2.so csc2
  one paper_2408_09697_b200/libhetgpu_csc1.so csc1
  one paper_2408_09697_b200/libhetgpu_csc3.so csc3
done
