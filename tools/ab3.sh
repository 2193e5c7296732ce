# A/B/C of library builds: prev (HEAD), alt, new (working tree)
for i in 1 2; do
  for lib in prev pdl1 ""; do
    f=paper_2408_09697_b200/libhetgpu${lib:+_$lib}.so
    HETGPU_LIB=$f python bench.py --steps 30 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$f', round(d['value']/1e9,4), round(d['ms_per_step'],4), round(d['e2e']['value']/1e9,4))"
  done
done
