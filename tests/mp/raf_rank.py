"""One rank of a multi-GPU RAF run (one meta-partition per GPU, AGG_all over
NCCL). Launched by tests/test_gpu_multi.py as N processes; rank 0 publishes the
NCCL unique id through a file and writes the per-batch losses and active-row
counts (the PartialAgg row counts, raf.cpp:418-446) to an .npz."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


# fanouts (HG_FANOUTS="25,15,10": a three-layer model)
FANOUTS = [int(x) for x in os.environ.get("HG_FANOUTS", "25,20").split(",")]


def main():
    name, seed, p, rank, id_path, out_path, n_batches, bsz = sys.argv[1:9]
    seed, p, rank, n_batches, bsz = int(seed), int(p), int(rank), int(n_batches), int(bsz)
    from paper_2408_09697_b200 import hetsim as H
    if name.startswith("spec:"):  # a spec written by the test as JSON
        import json
        with open(name[len("spec:"):]) as f:
            spec = json.load(f)
    else:
        spec = H.bundled_spec(name)
    g = H.gen_synthetic(spec, seed)
    kw = {}
    if os.environ.get("HG_PLAN_WORK", "0") != "0":  # the work-aware plan (not the reference's)
        import numpy as _np
        sw = H.sub_work(g, FANOUTS, 4, bsz, seed, device=rank)
        kw["sub_work"] = _np.concatenate([sw["work"], sw["learn_rows"]])
    if os.environ.get("HG_MODEL", "rgcn") != "rgcn":  # the RGAT layer type (tests/test_rgat.py)
        kw["model"] = os.environ["HG_MODEL"]
    eng = H.Engine.for_experiment(g, FANOUTS, 32, seed, batch_cap=bsz, p=p, rank=rank, device=rank, **kw)
    if rank == 0:
        uid = H.nccl_unique_id()
        with open(id_path + ".tmp", "wb") as f:
            f.write(uid)
        os.replace(id_path + ".tmp", id_path)
    else:
        t0 = time.time()
        while not os.path.exists(id_path):
            if time.time() - t0 > 120:
                raise RuntimeError("no NCCL id from rank 0")
            time.sleep(0.05)
        uid = open(id_path, "rb").read()
    if os.environ.get("HG_NO_GRAPHS"):
        eng.set_option("graphs", 0)
    if os.environ.get("HG_SHARD_MERGE", "0") != "0":  # replica merge sharded by id (peer stores)
        eng.set_option("shard_merge", 1)
    print(f"rank {rank}: attaching", flush=True)
    eng.attach_nccl(uid, p, rank)
    print(f"rank {rank}: attached", flush=True)
    # replica groups: publish this rank's IPC handle, map the peers'
    hpath = f"{id_path}.h{rank}"
    with open(hpath + ".tmp", "wb") as f:
        f.write(eng.replica_handle())
    os.replace(hpath + ".tmp", hpath)
    t0 = time.time()
    while not all(os.path.exists(f"{id_path}.h{r}") for r in range(p)):
        if time.time() - t0 > 120:
            raise RuntimeError("missing replica handles")
        time.sleep(0.05)
    eng.attach_replicas([open(f"{id_path}.h{r}", "rb").read() for r in range(p)])
    budget = int(os.environ.get("HG_CACHE_BUDGET", "0"))
    if budget:  # run_experiment's cache (harness.cpp:373-437): plan from a whole-graph presample
        pe = H.Engine.for_experiment(g, FANOUTS, 32, seed, batch_cap=512, device=rank)
        hot = pe.presample_hotness(2, H.mix_seed(seed, 0xCA11E), 512)
        del pe
        n_types = len(g.export()["node_counts"])
        cplan = H.cache_plan(g, hot, n_types, budget)
        eng.set_cache([cplan[f"cached.t{t}"] for t in range(n_types)])
    batches = H.make_batches(g, bsz, n_batches, H.mix_seed(seed, 0xBA7C))
    losses, active, sync, lead, bound_ok, target_ok = [], [], [], [], [], []
    for i, b in enumerate(batches):
        rep = eng.step(b, H.mix_seed(seed, 0xB000 + i), i % p)
        if i == 0:
            g0 = eng.read(*[n for n in eng.tensor_names() if n.startswith(("grad.w.", "grad.f."))])
        print(f"rank {rank}: batch {i} loss {rep['loss']:.6f}", flush=True)
        losses.append(rep["loss"])
        active.append(rep["active_rows"])
        sync.append(rep["sync_bytes"])
        lead.append(int(rep["sync_leader"]))
        bound_ok.append(int(rep["message_bound_ok"]))
        target_ok.append(int(rep["target_only_ok"]))
        boundary = (rep["boundary_counts"], rep["boundary_cut_edges"])
    post = eng.read(*[n for n in eng.tensor_names()
                      if n.startswith(("post.r", "post.learn.t", "post.learn_step.t", "att."))])
    np.savez(out_path, losses=np.asarray(losses), active=np.asarray(active, np.int64),
             sync=np.asarray(sync, np.uint64), lead=np.asarray(lead), bound_ok=np.asarray(bound_ok),
             target_ok=np.asarray(target_ok), boundary=np.asarray(boundary[0], np.uint64),
             cut_edges=np.asarray([boundary[1]], np.uint64),
             **{"T:" + k: v for k, v in post.items()}, **{"G:" + k: v for k, v in g0.items()},
             **({"C:" + k: v for k, v in eng.cache_counters().items()} if budget else {}),
             **({"C:transfer_ns": cplan["profile.transfer_ns"]} if budget else {}))


if __name__ == "__main__":
    main()
