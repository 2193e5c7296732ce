"""presample_hotness (cache.cpp:39-63) on C2: one epoch of batch-1024 sampling passes with
the visit histogram on the device (one sampling-graph replay per batch), against the
reference's presample_hotness (oracle/_ref, one host thread) on the same graph, and the
counts compared bit for bit.  python tools/presample_bench.py"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_09697_b200 import hetsim as H  # noqa: E402
from oracle import ref  # noqa: E402  (the checker and the CPU reference arm only)

spec = H.ogbn_mag_spec()
g = H.gen_synthetic(spec, 1)
eng = H.Engine.for_experiment(g, [25, 20], 64, 1, batch_cap=1024)
eng.presample_hotness(1, 7, 1024)  # warm (graph capture)
t = time.time()
hot = eng.presample_hotness(1, H.mix_seed(1, 0xCA11E), 1024)
dev_s = time.time() - t
out = {"workload": "C2 presample_hotness, 1 epoch, batch 1024", "device_s": dev_s,
       "batches": int(np.ceil(spec["node_types"][0]["count"] / 1024))}
rg = ref.RefGraph.from_spec(spec, 1)
t = time.time()
want = rg.cache_sim(2, [25, 20], 1, H.mix_seed(1, 0xCA11E), 1024)
out["reference_cache_sim_s"] = time.time() - t
keys = [k for k in want if k.startswith("hot.")]
out["counts_bit_exact"] = bool(keys) and all(np.array_equal(np.asarray(hot[k]), np.asarray(want[k])) for k in keys)
out["speedup_vs_reference_1_thread"] = out["reference_cache_sim_s"] / dev_s
print(json.dumps(out))
