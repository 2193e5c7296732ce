import sys, os, time
sys.path.insert(0, os.getcwd())
from paper_2408_09697_b200 import hetsim as H
g = H.gen_synthetic(H.ogbn_mag_spec(), 1)
eng = H.Engine.for_experiment(g, [25, 20], 64, 1, batch_cap=1024)
eng.presample_hotness(2, H.mix_seed(1, 0xCA11E), 512)  # warm
t = time.time(); hot = eng.presample_hotness(2, H.mix_seed(1, 0xCA11E), 512); dt = time.time() - t
n = sum(int(v.sum()) for v in hot.values())
print(f"presample_hotness ogbn-mag: 2 epochs x {(736389 + 511)//512} batches of 512 in {dt*1000:.1f} ms; {n} counted visits ({n/dt/1e9:.2f} G visits/s)")
