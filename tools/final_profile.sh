set -x
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
tail -1 gpurun_out/bench_final.json | cut -c1-400
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_final.json 2> gpurun_out/ref_final.err
tail -1 gpurun_out/ref_final.json | cut -c1-300
ncu --metrics gpu__time_duration.sum --clock-control none -s 100 -c 400 --csv --log-file gpurun_out/launches7.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu7.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:'k_gather_mean|k_csc_gather' -s 8 -c 4 -f -o gpurun_out/prof_gc python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_gc.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:'k_umma|k_sample_fused|k_cross_entropy' -s 20 -c 10 -f -o gpurun_out/prof_misc python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_misc.log 2>&1
ls -la gpurun_out/
