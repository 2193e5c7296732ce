"""Diagnostics (not a test): C2 at p ranks under torchrun; prints per rank the
leaf-frontier and replica-union sizes of one step and the eager per-class
device time of a few profiled steps."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_09697_b200 import hetsim as H  # noqa: E402

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
g = H.gen_synthetic(H.ogbn_mag_spec(), 1)
eng = H.Engine.for_experiment(g, [25, 20], 64, 1, batch_cap=1024 * world, p=world, rank=rank, device=local)
uid = [H.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(uid, src=0)
eng.attach_nccl(uid[0], world, rank)
handles = [None] * world
dist.all_gather_object(handles, eng.replica_handle())
eng.attach_replicas(handles)
batches = H.make_batches(g, 1024 * world, 8, H.mix_seed(1, 0xBA7C))
for i in range(3):
    eng.step(batches[i], H.mix_seed(1, 0xB000 + i), 0)
names = eng.tensor_names()
sizes = {n: len(v) for n, v in eng.read(*[n for n in names if n.endswith(".ids")]).items()}
unions = {}
for t in range(4):
    try:
        unions[t] = len(eng.read(f"merge.t{t}.union")[f"merge.t{t}.union"])
    except Exception:
        pass
eng.profile(True)
for i in range(3, 8):
    eng.step(batches[i], H.mix_seed(1, 0xB000 + i), 0)
prof = eng.profile_read()
us = {k.split(".")[1]: round(float(v[0]) * 1000 / 5, 1) for k, v in prof.items() if k.endswith(".ms")}
for r in range(world):
    if r == rank:
        print(f"rank {rank}: leaf ids {sizes} unions {unions}\n  us/step {us}", flush=True)
    dist.barrier()
dist.destroy_process_group()
