one() { HETGPU_LIB=$1 python bench.py --steps 60 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernel_us_per_step']; print('$2', round(d['value']/1e9,4), round(d['ms_per_step'],4), round(d['e2e']['value']/1e9,4), 'proj', k['project'], k['project_top'])"; }
for i in 1 2; do
  one paper_2408_09697_b200/libhetgpu.so p64
  one paper_2408_09697_b200/libhetgpu_p128s2.so p128s2
  one paper_2408_09697_b200/libhetgpu_p128s3.so p128s3
  one paper_2408_09697_b200/libhetgpu_p32.so p32
done
