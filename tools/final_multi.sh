# Round-end multi-GPU record on one 4-GPU box: C2 scale lines (N = 2, 4) + multi-GPU tests,
# the reference arm, and the C4 x0.1 run (one GPU); outputs under gpurun_out/
bash tools/scale_c2.sh
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_arm.json 2> gpurun_out/ref_arm.err; tail -c 300 gpurun_out/ref_arm.json
timeout 1500 python tools/bench_c4.py --scale 0.1 --out gpurun_out/c4_x0.1.json > /dev/null 2> gpurun_out/c4.err; tail -c 400 gpurun_out/c4_x0.1.json
