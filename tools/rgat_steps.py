"""A few C3 RGAT training steps (ncu launch lists of the RGAT kernels):
python tools/rgat_steps.py [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_09697_b200 import hetsim as H  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
g = H.gen_synthetic(H.ogbn_mag_spec(), 1)
batches = H.make_batches(g, 1024, steps, H.mix_seed(1, 0xBA7C))
eng = H.Engine.for_experiment(g, [25, 20], 64, 1, batch_cap=1024, model="rgat", heads=4)
eng.set_option("retain_grads", 0)
for i, b in enumerate(batches):
    print(eng.step(b, H.mix_seed(1, 0xB000 + i))["loss"])
