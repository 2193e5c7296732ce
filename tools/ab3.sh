one() { HETGPU_LIB=$1 python bench.py --steps 60 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernel_us_per_step']; print('$2', round(d['value']/1e9,4), round(d['ms_per_step'],4), round(d['e2e']['value']/1e9,4), 'sample', k['sample'], 'csc_build', k['csc_build'])"; }
HETGPU_LIB=paper_2408_09697_b200/libhetgpu_u8.so python -m pytest tests/test_gpu_sampling.py -x -q 2>&1 | tail -1
HETGPU_LIB=paper_2408_09697_b200/libhetgpu_sc1024.so python -m pytest tests/test_gpu_sampling.py tests/test_gpu_numerics.py -x -q 2>&1 | tail -1
for i in 1 2; do
  one paper_2408_09697_b200/libhetgpu.so base
  one paper_2408_09697_b200/libhetgpu_u8.so u8
  one paper_2408_09697_b200/libhetgpu_u2.so u2
  one paper_2408_09697_b200/libhetgpu_sc1024.so sc1024
done
