set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for i in 1 2; do
  HETGPU_LIB=paper_2408_09697_b200/libhetgpu_prev.so python bench.py --steps 30 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('prev', d['value'], d['ms_per_step'], d['e2e']['value'])"
  python bench.py --steps 30 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('new ', d['value'], d['ms_per_step'], d['e2e']['value'])"
done
