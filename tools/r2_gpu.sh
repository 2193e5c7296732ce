# Round-2 GPU pass: gpu tests, smoke, bench, launch list and one full ncu capture
# of a bench step (every kernel class), all on one B200. The full report is
# reduced on the box (tools/traffic_json.py + ncu_summary.py) and deleted there:
# gpurun brings back at most 64 MiB.
set -x
mkdir -p gpurun_out
if [ -z "$NOTEST" ]; then
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo PYTEST_EXIT $? >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
fi
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -1 gpurun_out/bench.json | cut -c1-3000
if [ -n "$NCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 100 -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python tools/ncu_summary.py launches gpurun_out/launches.csv > gpurun_out/launches.md 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -s 124 -c 40 -f -o gpurun_out/prof_step python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
python tools/traffic_json.py gpurun_out/prof_step.ncu-rep "ncu --set full --clock-control none -s 124 -c 40 python bench.py --steps 10 --warmup 3 --no-cpu-baseline" > gpurun_out/traffic.json 2> gpurun_out/traffic.err
python tools/ncu_summary.py full gpurun_out/prof_step.ncu-rep > gpurun_out/prof_step.md 2>&1
ncu -i gpurun_out/prof_step.ncu-rep --page raw --csv > gpurun_out/prof_step_raw.csv 2>/dev/null
gzip -f gpurun_out/prof_step_raw.csv
rm -f gpurun_out/prof_step.ncu-rep
fi
ls -la gpurun_out/
