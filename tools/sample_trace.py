"""Diagnostics (not a test): per-tile timeline of the sampler on C2 (one batch).
Prints, per hop, the tiles sorted by start with their segment, SM, and the
scan / draw / gather durations (us, %globaltimer)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_09697_b200 import hetsim as H  # noqa: E402

g = H.gen_synthetic(H.ogbn_mag_spec(), 1)
eng = H.Engine.for_experiment(g, [25, 20], 64, 1, batch_cap=1024)
eng.set_option("trace_sampler", 1)
batches = H.make_batches(g, 1024, 4, H.mix_seed(1, 0xBA7C))
for i in range(3):
    eng.sample(batches[i], H.mix_seed(1, 0xB000 + i))
for h in (1, 2):
    tr = eng.read(f"trace.sample.h{h}")[f"trace.sample.h{h}"].astype(np.int64)
    live = tr[tr[:, 0] > 0]
    t0 = live[:, 0].min()
    print(f"hop {h}: {len(live)} live tiles, kernel span {(live[:, 3].max() - t0) / 1e3:.1f} us")
    segs = {}
    for r in live:
        s = segs.setdefault(int(r[4]), [])
        s.append(((r[0] - t0) / 1e3, (r[1] - r[0]) / 1e3, (r[2] - r[1]) / 1e3, (r[3] - r[2]) / 1e3, (r[3] - t0) / 1e3))
    rng = live[live[:, 6] > 0]
    if len(rng):
        print(f"  rng tiles (thread 0): seeding {np.median((rng[:,6]-rng[:,1])/1e3):.1f} us, outputs {np.median((rng[:,7]-rng[:,6])/1e3):.1f} us, resolve+rest {np.median((rng[:,2]-rng[:,7])/1e3):.1f} us")
    for sgi, v in sorted(segs.items()):
        v = np.array(v)
        print(f"  seg {sgi}: {len(v):4d} tiles start {v[:,0].min():6.1f}-{v[:,0].max():6.1f}  scan med {np.median(v[:,1]):5.1f} max {v[:,1].max():5.1f}"
              f"  draw med {np.median(v[:,2]):5.1f} max {v[:,2].max():5.1f}  gather med {np.median(v[:,3]):5.1f} max {v[:,3].max():5.1f}  end max {v[:,4].max():6.1f}")
