"""Multi-GPU RAF: one meta-partition per GPU, AGG_all as one
ncclAllReduce of the partial logits. Parity against the reference's
single-process RAF engine with the same p (raf.cpp:344-530, harness.cpp:403-423):
per-batch losses within 1e-3 and the PartialAgg message bytes of every batch
equal to the reference's CommStats (32 B header + rows x C x 4 B, raf.cpp:113-115)."""
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def n_gpus():
    from tests.util import gpu_count
    return gpu_count()


# one root relation: a single sub-metatree, so every rank is a replica of it
# (groups of 3 and 4 as at p = 8 on ogbn-mag), with learnable leaves to merge
SINGLE_ROOT = {
    "name": "single-root", "target": "paper", "num_classes": 6, "label_noise": 0.1,
    "node_types": [{"name": "paper", "count": 3000, "dim": 32, "storage": "dense"},
                   {"name": "author", "count": 4000, "dim": 16, "storage": "learnable"},
                   {"name": "field", "count": 600, "dim": 16, "storage": "learnable"}],
    "relations": [{"src": "author", "edge": "writes", "dst": "paper", "edges": 12000},
                  {"src": "field", "edge": "topic", "dst": "author", "edges": 6000}],
    "self_paired": []}


@pytest.mark.parametrize("name,p,shard", [("mag-mini", 2, 0), ("mag-mini", 4, 0), ("igb-mini", 4, 0),
                                          ("mag-mini", 4, 1), ("single-root", 3, 0), ("single-root", 4, 0),
                                          ("single-root", 3, 1)])
def test_raf_multi_gpu_matches_reference(ref, name, p, shard):
    # p = 4 > 3 sub-metatrees: one sub-metatree is replicated, its replicas split
    # the batch and synchronise weight gradients (NCCL) and learnable rows
    # (peer-mapped merge) before Adam
    if n_gpus() < p:
        pytest.skip(f"needs {p} GPUs")
    seed, n_batches, bsz = 5, 6, 64
    with tempfile.TemporaryDirectory() as td:
        idp = os.path.join(td, "nccl.id")
        arg = name
        if name == "single-root":
            import json
            arg = "spec:" + os.path.join(td, "spec.json")
            with open(arg[len("spec:"):], "w") as f:
                json.dump(SINGLE_ROOT, f)
        procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "mp", "raf_rank.py"), arg, str(seed), str(p),
                                   str(r), idp, os.path.join(td, f"r{r}.npz"), str(n_batches), str(bsz)],
                                  stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True,
                                  env=dict(os.environ, HG_SHARD_MERGE=str(shard))) for r in range(p)]
        outs = [pr.communicate(timeout=300)[0] for pr in procs]
        for pr, o in zip(procs, outs):
            assert pr.returncode == 0, o[-3000:]
        res = [np.load(os.path.join(td, f"r{r}.npz")) for r in range(p)]
    from paper_2408_09697_b200 import hetsim as H
    spec = SINGLE_ROOT if name == "single-root" else H.bundled_spec(name)
    g = H.gen_synthetic(spec, seed)
    batches = H.make_batches(g, bsz, n_batches, H.mix_seed(seed, 0xBA7C))
    rg = ref.RefGraph.from_spec(spec, seed) if name == "single-root" else ref.RefGraph.bundled(name, seed)
    want = rg.raf_train(2, 32, p, seed, [list(b) for b in batches], [25, 20])
    for r in range(p):  # every rank computes the same loss from the all-reduced logits
        np.testing.assert_allclose(res[r]["losses"], want["losses"], rtol=1e-3, atol=0)
    # final parameters: every partition's weight slots and learnable tables track
    # the reference's merged-gradient Adam; replicas hold bit-identical copies
    from tests.util import assert_adam_close, assert_close
    # first batch: weight gradients after the replica all-reduce equal the
    # reference's merged GradientSet (raf.cpp:468-494, hgnn.cpp:83-113)
    for r in range(p):
        for key in res[r].files:
            if key.startswith("G:grad.w."):
                assert_close(res[r][key], want["b0.grad." + key[len("G:grad."):]], 1e-3, f"rank {r}: {key}")
    seen = {}
    for r in range(p):
        for key in res[r].files:
            if not key.startswith("T:"):
                continue
            n, v = key[2:], res[r][key]
            if n in seen:
                assert np.array_equal(seen[n], v), f"replicas disagree on {n}"
            seen[n] = v
            if n.startswith("post.r"):
                assert_adam_close(v, want["final." + n[len("post."):]], None, max_flip_frac=5e-3, steps=n_batches,
                                  what=f"rank {r}: {n}")
            elif n.startswith("post.learn.t"):
                assert_adam_close(v, want["final.learn.t" + n.split(".t")[-1]], None, max_flip_frac=5e-3, steps=n_batches,
                                  what=f"rank {r}: {n}")
            elif n.startswith("post.learn_step.t"):
                assert int(v[0]) == int(want["final.learn_step.t" + n.split(".t")[-1]][0]), (r, n)
    # PartialAgg bytes: every bucket not owned by the designated worker sends
    # 32 + active_rows * C * 4 bytes; the PartialGrad mirror sends the same back
    C = int(np.asarray(rg.export()["num_classes"]).ravel()[0])
    act = res[0]["active"]
    for i in range(n_batches):
        got_bytes = H.agg_all_comm_bytes(act[i], i % p, C)["total_bytes"]
        assert got_bytes == int(want["bytes"][i]), (i, got_bytes, int(want["bytes"][i]))
    # ExecutionReport bookkeeping (raf.hpp:66-77): the ring-model sync bytes of
    # replicated slots and learnable rows (raf.cpp:496-510) summed over replica-group
    # leaders, structural boundaries and cut edges, and the check_comm_bounds verdicts
    for i in range(n_batches):
        got_sync = sum(int(res[r]["sync"][i]) for r in range(p) if res[r]["lead"][i])
        assert got_sync == int(want["sync_bytes"][i]), (i, got_sync, int(want["sync_bytes"][i]))
    for r in range(p):
        assert np.array_equal(res[r]["boundary"], want["boundary_counts"]), r
        assert int(res[r]["cut_edges"][0]) == int(want["boundary_cut_edges"][0])
        assert np.array_equal(res[r]["bound_ok"], want["message_bound_ok"].astype(res[r]["bound_ok"].dtype))
        assert np.array_equal(res[r]["target_ok"], want["target_only_ok"].astype(res[r]["target_ok"].dtype))


@pytest.mark.parametrize("name,p", [("mag-mini", 2), ("mag-mini", 4), ("igb-mini", 3)])
def test_work_aware_plan_matches_flat_reference(ref, name, p):
    # the work-aware plan (worker groups replicating sub-metatree sets, sized by the
    # measured sampled work and learnable rows) computes the flat pass's numbers: the
    # per-batch losses and the final parameters of the reference's p = 1 run
    if n_gpus() < p:
        pytest.skip(f"needs {p} GPUs")
    seed, n_batches, bsz = 5, 6, 64
    with tempfile.TemporaryDirectory() as td:
        idp = os.path.join(td, "nccl.id")
        procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "mp", "raf_rank.py"), name, str(seed), str(p),
                                   str(r), idp, os.path.join(td, f"r{r}.npz"), str(n_batches), str(bsz)],
                                  stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True,
                                  env=dict(os.environ, HG_PLAN_WORK="1")) for r in range(p)]
        outs = [pr.communicate(timeout=300)[0] for pr in procs]
        for pr, o in zip(procs, outs):
            assert pr.returncode == 0, o[-3000:]
        res = [np.load(os.path.join(td, f"r{r}.npz")) for r in range(p)]
    from paper_2408_09697_b200 import hetsim as H
    from tests.util import assert_adam_close
    g = H.gen_synthetic(H.bundled_spec(name), seed)
    batches = H.make_batches(g, bsz, n_batches, H.mix_seed(seed, 0xBA7C))
    want = ref.RefGraph.bundled(name, seed).raf_train(2, 32, 1, seed, [list(b) for b in batches], [25, 20])
    for r in range(p):
        np.testing.assert_allclose(res[r]["losses"], want["losses"], rtol=1e-3, atol=0)
    seen = {}
    for r in range(p):
        for key in res[r].files:
            if not key.startswith("T:"):
                continue
            n, v = key[2:], res[r][key]
            if n in seen:
                assert np.array_equal(seen[n], v), f"replicas disagree on {n}"
            seen[n] = v
            if n.startswith("post.r"):
                assert_adam_close(v, want["final." + n[len("post."):]], None, max_flip_frac=1e-2, steps=n_batches,
                                  what=f"rank {r}: {n}")
            elif n.startswith("post.learn.t"):
                assert_adam_close(v, want["final.learn.t" + n.split(".t")[-1]], None, max_flip_frac=1e-2,
                                  steps=n_batches, what=f"rank {r}: {n}")


@pytest.mark.parametrize("p", [2, 4])
def test_cache_counters_over_the_global_frontier(ref, p):
    """run_experiment's cache accounting at p > 1 looks up the whole batch's layer-0
    frontier (harness.cpp:425-437): every rank counts the union of the partitions'
    frontiers (an ncclMax all-reduce of 0/1 maps), equal to the reference's hits and misses."""
    if n_gpus() < p:
        pytest.skip(f"needs {p} GPUs")
    seed, n_batches, bsz, budget = 5, 4, 64, 1 << 18
    with tempfile.TemporaryDirectory() as td:
        idp = os.path.join(td, "nccl.id")
        procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "mp", "raf_rank.py"), "mag-mini", str(seed), str(p),
                                   str(r), idp, os.path.join(td, f"r{r}.npz"), str(n_batches), str(bsz)],
                                  stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True,
                                  env=dict(os.environ, HG_CACHE_BUDGET=str(budget))) for r in range(p)]
        outs = [pr.communicate(timeout=300)[0] for pr in procs]
        for pr, o in zip(procs, outs):
            assert pr.returncode == 0, o[-3000:]
        res = [np.load(os.path.join(td, f"r{r}.npz")) for r in range(p)]
    from paper_2408_09697_b200 import hetsim as H
    cfg = {"spec": "mag-mini", "partitioner": "meta", "p": p, "engine": "raf", "fanouts": [25, 20], "hidden": 32,
           "batch_size": bsz, "epochs": 1, "max_batches_per_epoch": n_batches, "seed": seed, "cache_budget": budget}
    stats, _, ok = ref.run_experiment(cfg)
    assert ok
    np.testing.assert_allclose(res[0]["losses"], [b["loss"] for b in stats["batches"]], rtol=1e-3, atol=0)
    e = H.gen_synthetic(H.bundled_spec("mag-mini"), seed).export()
    names = [t["name"] for t in H.bundled_spec("mag-mini")["node_types"]]
    for r in range(p):
        counters = {k[2:]: res[r][k] for k in res[r].files if k.startswith("C:cache.")}
        assert counters, "no cache counters"
        mine = {s["type"]: s for s in H.cache_stats(counters, e["kinds"], res[r]["C:transfer_ns"])}
        for want in stats["cache"]["per_type"]:
            got = mine[names.index(want["type"])]
            assert (got["hits"], got["misses"]) == (want["hits"], want["misses"]), (r, want["type"], got, want)


@pytest.mark.parametrize("p", [2, 4])
def test_three_layer_work_aware_plan_matches_flat_reference(ref, p):
    """A deep metatree (the C4 MAG240M schema at k = 3: relations recur at several depths):
    the work-aware planner only forms groups that share no weight slot or learnable leaf
    type, here the all-subs group replicated p times (data parallel with the replica
    merge); losses and the trained model match the reference's flat RAF run."""
    if n_gpus() < p:
        pytest.skip(f"needs {p} GPUs")
    import json
    from paper_2408_09697_b200 import hetsim as H
    seed, n_batches, bsz = 5, 4, 64
    spec = H.mag240m_spec(0.0005)
    with tempfile.TemporaryDirectory() as td:
        arg = "spec:" + os.path.join(td, "spec.json")
        with open(arg[len("spec:"):], "w") as f:
            json.dump(spec, f)
        idp = os.path.join(td, "nccl.id")
        procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "mp", "raf_rank.py"), arg, str(seed), str(p),
                                   str(r), idp, os.path.join(td, f"r{r}.npz"), str(n_batches), str(bsz)],
                                  stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True,
                                  env=dict(os.environ, HG_PLAN_WORK="1", HG_FANOUTS="25,15,10")) for r in range(p)]
        outs = [pr.communicate(timeout=300)[0] for pr in procs]
        for pr, o in zip(procs, outs):
            assert pr.returncode == 0, o[-3000:]
        res = [np.load(os.path.join(td, f"r{r}.npz")) for r in range(p)]
    g = H.gen_synthetic(spec, seed)
    batches = H.make_batches(g, bsz, n_batches, H.mix_seed(seed, 0xBA7C))
    want = ref.RefGraph.from_spec(spec, seed).raf_train(3, 32, 1, seed, [list(b) for b in batches], [25, 15, 10])
    from tests.util import assert_adam_close
    for r in range(p):
        np.testing.assert_allclose(res[r]["losses"], want["losses"], rtol=1e-3, atol=0)
        for key in res[r].files:
            if key.startswith("T:post.r"):
                n = key[len("T:post."):]
                assert_adam_close(res[r][key], want["final." + n], None, steps=n_batches, max_flip_frac=1e-2,
                                  what=f"p={p} rank {r}: {n}")
