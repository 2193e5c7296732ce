# A/B re-check after the gather changes: relabel/transpose grid (HG_FRONT_WAVES 8) and weight-gradient chunk (HG_WCHUNK 256 / 1024)
one() { HETGPU_LIB=$1 python bench.py --steps 100 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernel_us_per_step']; print('$2', round(d['value']/1e9,4), round(d['ms_per_step'],4), round(d['e2e']['value']/1e9,4), 'front', k['frontier'], 'csc_build', k['csc_build'], 'wgrad', k['weight_grad'])"; }
for i in 1 2 3; do
  one paper_2408_09697_b200/libhetgpu.so base
  one paper_2408_09697_b200/libhetgpu_fw8.so fw8
  one paper_2408_09697_b200/libhetgpu_wc256.so wc256
  one paper_2408_09697_b200/libhetgpu_wc1024.so wc1024
done
