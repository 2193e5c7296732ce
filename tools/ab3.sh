one() { HETGPU_LIB=$1 python bench.py --steps 60 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$2', round(d['value']/1e9,4), round(d['ms_per_step'],4), round(d['e2e']['value']/1e9,4))"; }
for i in 1 2 3; do
  one paper_2408_09697_b200/libhetgpu_c4g8.so c4g8
  one paper_2408_09697_b200/libhetgpu_c8g8.so c8g8
  one paper_2408_09697_b200/libhetgpu_c4g16.so c4g16
  one paper_2408_09697_b200/libhetgpu.so c8g16
done
