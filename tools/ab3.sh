one() { python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernel_us_per_step']; print('$HG_NT_CAP', round(d['value']/1e9,4), round(d['ms_per_step'],4), 'proj', k.get('project'), k.get('project_top'), 'dmean', k.get('mean_grad'), 'wgrad', k.get('weight_grad'))"; }
for i in 1 2; do
  for c in 128,128,128 64,128,128 32,128,128 128,32,128 128,128,64 64,32,64; do HG_NT_CAP=$c one; done
done
