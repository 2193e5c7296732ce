"""Host side of the multi-GPU path on CPU with world_size 2 (gloo): every rank
builds the same meta-partition plan (metapartition.cpp:283-295) and takes its
own partition; across ranks the owned sub-metatrees cover the tree exactly once,
replicas split the batch rows i mod n_owners (raf.cpp:390-391) without overlap,
and the NCCL-id broadcast + max-over-ranks timing plumbing of bench.py works."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank(rank, world, port, spec_name, p, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2408_09697_b200 import hetsim as H
    g = H.gen_synthetic(H.bundled_spec(spec_name), 3)
    plan = H.meta_partition(g, 2, p)
    parts = {}
    for r in range(rank, p, world):  # this process's partitions
        parts[r] = {k.split(".", 1)[1]: plan[k] for k in plan if k.startswith(f"part{r}.")}
    got = [None] * world
    dist.all_gather_object(got, parts)
    # bench.py's plumbing: rank 0's id reaches every rank; the max over ranks
    uid = [b"id-from-rank-0" if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    import torch
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        merged = {}
        for d in got:
            merged.update(d)
        np.save(out, np.array([merged, plan, uid[0], float(t.item())], dtype=object), allow_pickle=True)
    dist.destroy_process_group()


@pytest.mark.parametrize("spec_name,p", [("mag-mini", 2), ("mag-mini", 4), ("igb-mini", 3)])
def test_partitions_cover_tree_across_ranks(tmp_path, spec_name, p):
    out = str(tmp_path / "res.npy")
    mp.spawn(_rank, args=(2, _free_port(), spec_name, p, out), nprocs=2, join=True)
    merged, plan, uid, tmax = np.load(out, allow_pickle=True)
    assert uid == b"id-from-rank-0" and tmax == 2.0
    assert sorted(merged) == list(range(p))
    n_subs = len(plan["subs.weight"])
    owners = {s: [] for s in range(n_subs)}
    for r, part in merged.items():
        for s in part["sub_ids"].tolist():
            owners[s].append(r)
    for s, own in owners.items():
        assert own, f"sub-metatree {s} unowned"
        reps = [tuple(merged[r]["replica"].tolist()) for r in own]
        if len(own) == 1:
            assert reps[0][0] == 0
        else:
            # replicas of one sub-metatree: indices 0..n-1, each row of the batch
            # belongs to exactly one of them (raf.cpp:390-391)
            assert sorted(x[1] for x in reps) == list(range(len(own)))
            assert all(x[2] == len(own) for x in reps)
            batch = np.arange(1000)
            shards = [batch[x[1]::x[2]] for x in reps]
            assert np.array_equal(np.sort(np.concatenate(shards)), batch)
