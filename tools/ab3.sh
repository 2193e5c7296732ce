one() { HETGPU_LIB=$1 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernel_us_per_step']; print('$2', round(d['value']/1e9,4), round(d['ms_per_step'],4), round(d['e2e']['value']/1e9,4), 'proj', k['project'], 'dmean', k['mean_grad'], 'wgrad', k['weight_grad'])"; }
HETGPU_LIB=paper_2408_09697_b200/libhetgpu_s2.so python -m pytest tests/test_gpu_numerics.py -x -q 2>&1 | tail -1
for i in 1 2; do
  one paper_2408_09697_b200/libhetgpu.so s4
  one paper_2408_09697_b200/libhetgpu_s3.so s3
  one paper_2408_09697_b200/libhetgpu_s2.so s2
done
