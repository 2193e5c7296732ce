# Round-end record on one 4-GPU box: the 1-GPU bench line (against the committed traffic
# capture), C2 scale lines (N = 2, 4) + multi-GPU tests, the reference arm, C3 / C4 / C5 at
# 1, 2, 4 GPUs and the C4 x0.1 run (one GPU); outputs under gpurun_out/
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -c 300 gpurun_out/bench_final.json
bash tools/scale_c2.sh
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_arm.json 2> gpurun_out/ref_arm.err; tail -c 300 gpurun_out/ref_arm.json
bash tools/c4_scale.sh
bash tools/c5_scale.sh
bash tools/c3_scale.sh
timeout 1500 python tools/bench_c4.py --scale 0.1 --out gpurun_out/c4_x0.1.json > /dev/null 2> gpurun_out/c4.err; tail -c 400 gpurun_out/c4_x0.1.json
