one() { HETGPU_LIB=$1 python bench.py --steps 60 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernel_us_per_step']; print('$2', round(d['value']/1e9,4), round(d['ms_per_step'],4), round(d['e2e']['value']/1e9,4), 'front', k['frontier'], 'csc_build', k['csc_build'])"; }
HETGPU_LIB=paper_2408_09697_b200/libhetgpu_f1.so python -m pytest tests/test_gpu_sampling.py tests/test_gpu_numerics.py -x -q 2>&1 | tail -1
for i in 1 2; do
  one paper_2408_09697_b200/libhetgpu.so f4
  one paper_2408_09697_b200/libhetgpu_f2.so f2
  one paper_2408_09697_b200/libhetgpu_f1.so f1
done
