"""Partition-aware feature cache on the GPU against the compiled reference
(SURVEY §8(a) a6-a10): the device presample_hotness counts (cache.cpp:39-63),
the cache plan built from them (cache.cpp:11-141), and the per-batch
lookup/update hit and miss accounting of run_experiment (harness.cpp:373-461)
together with the per-batch training losses of the same run."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,seed", [("mag-mini", 3), ("igb-mini", 5), ("freebase-mini", 7)])
def test_presample_hotness_on_device_matches_reference(H, ref, name, seed):
    rg = ref.RefGraph.bundled(name, seed)
    g = H.gen_synthetic(H.bundled_spec(name), seed)
    hs = H.mix_seed(seed, 0xCA11E)
    want = rg.cache_sim(2, [10, 10], 2, hs, 512)
    eng = H.Engine.for_experiment(g, [10, 10], 16, seed, batch_cap=512)
    got = eng.presample_hotness(2, hs, 512)
    n_types = len(g.export()["node_counts"])
    for t in range(n_types):
        assert np.array_equal(got[f"hot.t{t}"].astype(np.uint64), want[f"hot.t{t}"]), (name, t)


@pytest.mark.parametrize("budget", [1 << 16, 1 << 20])
def test_run_experiment_cache_counters_and_losses(H, ref, budget):
    seed, fanouts, hidden, bsz, nb = 3, [10, 10], 16, 256, 4
    cfg = {"spec": "mag-mini", "partitioner": "meta", "p": 1, "engine": "raf", "fanouts": fanouts,
           "hidden": hidden, "batch_size": bsz, "epochs": 1, "max_batches_per_epoch": nb, "seed": seed,
           "cache_budget": budget}
    stats, _, ok = ref.run_experiment(cfg)
    assert ok
    g = H.gen_synthetic(H.bundled_spec("mag-mini"), seed)
    e = g.export()
    n_types = len(e["node_counts"])
    eng = H.Engine.for_experiment(g, fanouts, hidden, seed, batch_cap=512)  # presample batches are 512
    hot = eng.presample_hotness(2, H.mix_seed(seed, 0xCA11E), 512)
    plan = H.cache_plan(g, hot, n_types, budget)
    eng.set_cache([plan[f"cached.t{t}"] for t in range(n_types)])
    batches = H.make_batches(g, bsz, nb, H.mix_seed(seed, 0xBA7C))
    losses = [eng.step(b, H.mix_seed(seed, 0xB000 + i), 0)["loss"] for i, b in enumerate(batches)]
    np.testing.assert_allclose(losses, [b["loss"] for b in stats["batches"]], rtol=1e-3, atol=0)
    mine = {s["type"]: s for s in H.cache_stats(eng.cache_counters(), e["kinds"], plan["profile.transfer_ns"])}
    names = list(H.bundled_spec("mag-mini")["node_types"])
    for want in stats["cache"]["per_type"]:
        t = [x["name"] for x in names].index(want["type"])
        got = mine[t]
        assert (got["hits"], got["misses"]) == (want["hits"], want["misses"]), (want["type"], got, want)
        assert got["penalty_ns"] == pytest.approx(want["penalty_ns"], rel=1e-12)
