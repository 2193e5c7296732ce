for ph in "" sample serial "" sample serial; do
  HG_BENCH_PHASE=$ph python bench.py --steps 50 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('phase=[$ph]', d['ms_per_step'])"
done
