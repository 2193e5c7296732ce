# A/B timing of library variants on one GPU: VARIANTS="base s3 ..." (base = libhetgpu.so),
# ROUNDS rounds, interleaved; prints value (G edges/s), ms/step, e2e and per-class us.
for r in $(seq ${ROUNDS:-2}); do
  for v in ${VARIANTS:-base}; do
    if [ "$v" = base ]; then export HETGPU_LIB=; else export HETGPU_LIB=$PWD/paper_2408_09697_b200/libhetgpu_$v.so; fi
    timeout 300 python bench.py --no-cpu-baseline ${BENCH_ARGS:-} 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']/1e9,4), round(d['ms_per_step'],4), round(d['e2e']['value']/1e9,4), d['kernel_us_per_step'])"
  done
done
