"""A few training steps of the hot path on mag-mini (sampling, forward, loss,
backward, Adam; graphs off so every kernel launches eagerly), for compute-sanitizer
(tests/test_gpu_sanitizer.py)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_09697_b200 import hetsim as H  # noqa: E402

g = H.gen_synthetic(H.bundled_spec("mag-mini"), 5)
eng = H.Engine.for_experiment(g, [25, 20], 32, 5, batch_cap=256)
eng.set_option("graphs", int(os.environ.get("HG_SANITIZE_GRAPHS", "0")))
batches = H.make_batches(g, 256, 3, H.mix_seed(5, 0xBA7C))
eng.prefetch(batches[0], H.mix_seed(5, 0xB000))
for i, b in enumerate(batches):
    if i + 1 < len(batches):
        eng.prefetch(batches[i + 1], H.mix_seed(5, 0xB000 + i + 1))
    rep = eng.step(b, H.mix_seed(5, 0xB000 + i), 0)
print("loss", rep["loss"])
