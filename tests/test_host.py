"""CPU tests of the host layer (no GPU): bit-exact graphs, plans, batches and
cache planning against the compiled reference, the reference's own known-answer
tests for these paths, and the C-ABI surface of libhetgpu.so."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ---- C-ABI surface -------------------------------------------------------------------

def declared_symbols():
    text = open(os.path.join(ROOT, "include", "hetgpu.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    import ctypes
    from paper_2408_09697_b200 import _native
    lib = _native.lib()
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert isinstance(ctypes.CDLL(_native.LIB_PATH), ctypes.CDLL)


def test_library_built_for_sm100a_only():
    import subprocess
    from paper_2408_09697_b200 import _native
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


# ---- graphs ------------------------------------------------------------------------

def compare_exports(ours, ref_e):
    for key, want in ref_e.items():
        if key in ("type_names", "etype_names", "rel_etype"):
            continue
        got = ours[key]
        if key.startswith("feat."):
            want = want.astype(np.float32)  # the device stores fp32 (HGC1 also stores f32)
        assert got.shape == want.shape, key
        assert np.array_equal(got, want.astype(got.dtype)), key


@pytest.mark.parametrize("name", ["mag-mini", "freebase-mini", "donor-mini", "igb-mini"])
@pytest.mark.parametrize("seed", [1, 5])
def test_gen_synthetic_bit_exact(H, ref, name, seed):
    compare_exports(H.gen_synthetic(H.bundled_spec(name), seed).export(),
                    ref.RefGraph.bundled(name, seed).export())


@pytest.mark.parametrize("chunk", ["311", "4096", "100003"])
def test_gen_synthetic_jumped_feature_chunks_bit_exact(H, ref, chunk, monkeypatch):
    # feature streams cut into HG_FEAT_CHUNK-value chunks, each engine jumped ahead
    # (mt_jump.cpp), equal the reference's serial streams bit for bit
    monkeypatch.setenv("HG_FEAT_CHUNK", chunk)
    compare_exports(H.gen_synthetic(H.bundled_spec("mag-mini"), 1).export(),
                    ref.RefGraph.bundled("mag-mini", 1).export())


def test_mt64_jump_ahead_matches_serial_outputs(H):
    seed = H.mix_seed(7, 0xf0)
    serial = H.mt64_outputs(seed, 0, 400_000)  # start 0: the plain engine
    for start in [1, 311, 312, 313, 624, 19_937, 65_536, 123_457, 399_000]:
        got = H.mt64_outputs(seed, start, 1000)
        want = serial[start:start + 1000]
        assert np.array_equal(got[:len(want)], want), start


def test_gen_synthetic_spec_variants(H, ref):
    spec = H.toy_spec()
    for t in spec["node_types"]:
        t["count"] //= 20
    for r in spec["relations"]:
        r["edges"] //= 20
    spec["relations"][0]["degree"] = "powerlaw"
    spec["relations"][0]["alpha"] = 1.3
    spec["label_noise"] = 0.3
    compare_exports(H.gen_synthetic(spec, 9).export(), ref.RefGraph.from_spec(spec, 9).export())


def test_gen_synthetic_rejects_bad_specs(H, ref):
    bad = H.bundled_spec("mag-mini")
    bad["target"] = "nope"
    bad["relations"][1]["edges"] = 0
    with pytest.raises(ValueError) as ours:
        H.gen_synthetic(bad, 1)
    with pytest.raises(RuntimeError) as theirs:
        ref.RefGraph.from_spec(bad, 1)
    assert str(ours.value) == str(theirs.value)


def test_build_hetgraph_insertion_order(H):
    # test_hetgraph.cpp:39-50: CSR keeps insertion order inside each destination
    g = H.build_hetgraph([3, 3], [(1, 0)], [[(1, 0), (0, 1), (0, 0), (2, 1)]], 0, 2)
    e = g.export()
    assert list(e["rel0.indptr"]) == [0, 2, 4, 4]
    assert list(e["rel0.src"]) == [1, 0, 0, 2]


# ---- plans ---------------------------------------------------------------------------

def citation_graph(H):
    """A concrete graph whose metagraph is test_util.hpp:77-98's citation schema:
    vertex weights P1 A2 I3 F4, link weights 4,5,10,6,3,3,6."""
    counts = [1, 2, 3, 4]
    P, A, I, F = range(4)
    rels = [(A, P), (A, I), (P, P), (P, F), (P, A), (I, A), (F, P)]
    sizes = [4, 5, 10, 6, 3, 3, 6]
    edges = [[(0, 0)] * n for n in sizes]
    return H.build_hetgraph(counts, rels, edges, 0, 2)


def test_citation_replay_kats(H):
    # test_metapartition.cpp:47-100 and acceptance.cpp:119-138
    g = citation_graph(H)
    plan = H.meta_partition(g, 2, 2)
    assert sorted(plan["subs.weight"].tolist()) == [16, 17, 27]
    assert plan["subs.weight"].tolist() == [16, 27, 17]
    parts = [plan["part0.sub_ids"].tolist(), plan["part1.sub_ids"].tolist()]
    light = 0 if len(parts[0]) == 2 else 1
    assert parts[light] == [0, 2] and parts[1 - light] == [1]
    assert int(plan[f"part{light}.weight"][0]) == 33 and int(plan[f"part{1 - light}.weight"][0]) == 27
    assert sorted(plan[f"part{light}.relations"].tolist()) == [0, 3, 4, 5, 6]
    assert sorted(plan[f"part{1 - light}.relations"].tolist()) == [0, 2, 6]
    # cacheable types (test_cache.cpp:195-217)
    assert plan[f"part{light}.cacheable"].tolist() == [0, 2]
    assert plan[f"part{1 - light}.cacheable"].tolist() == [1, 3]
    solo = H.meta_partition(g, 2, 1)
    assert sorted(solo["part0.relations"].tolist()) == [0, 2, 3, 4, 5, 6]
    assert solo["part0.cacheable"].tolist() == [0, 2, 3]
    # hop relation sets (test_hgnn.cpp:189-198)
    assert solo["hop_rels1"].tolist() == [0, 2, 6]
    assert solo["hop_rels2"].tolist() == [0, 2, 3, 4, 5, 6]
    # replication beyond the sub count (test_metapartition.cpp:111-133)
    p5 = H.meta_partition(g, 2, 5)
    reps = [p5[f"part{i}.replica"].tolist() for i in range(5)]
    assert all(len(p5[f"part{i}.sub_ids"]) == 1 for i in range(5))
    assert sum(r[0] for r in reps) >= 2
    p3 = H.meta_partition(g, 2, 3)
    assert all(p3[f"part{i}.replica"][0] == 0 for i in range(3))


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 8])
def test_plans_match_reference(H, ref, p):
    for name in H.bundled_spec_names():
        want = ref.RefGraph.bundled(name, 5).meta_partition(2, p)
        got = H.meta_partition(H.gen_synthetic(H.bundled_spec(name), 5), 2, p)
        for key in set(want) & set(got):
            assert np.array_equal(want[key], got[key]), (name, p, key)
    for s in range(30):
        rg = ref.RefGraph.random(s)
        g = H.graph_from_export(rg.export())
        for k in (1, 2, 3):
            want = rg.meta_partition(k, p)
            got = H.meta_partition(g, k, p)
            for key in set(want) & set(got):
                assert np.array_equal(want[key], got[key]), (s, k, p, key)


@pytest.mark.parametrize("p", [1, 2, 4, 8])
def test_raf_bookkeeping_matches_reference(H, ref, p):
    # batch-invariant ExecutionReport fields computed once per plan (SURVEY 8(f)
    # item 3): structural_boundaries (raf.cpp:306-340) and boundary_cut_edges
    # (raf.cpp:521-528) equal what run_raf_batch reports for a real batch
    for name in H.bundled_spec_names():
        g = H.gen_synthetic(H.bundled_spec(name), 5)
        batch = H.make_batches(g, 32, 1, H.mix_seed(5, 0xBA7C))[0]
        want = ref.RefGraph.bundled(name, 5).raf_train(2, 16, p, 5, [list(batch)], [5, 5])
        got = H.meta_partition(g, 2, p)
        assert np.array_equal(got["raf.boundary_counts"], want["boundary_counts"]), (name, p)
        assert int(got["raf.boundary_cut_edges"][0]) == int(want["boundary_cut_edges"][0]), (name, p)
        assert int(want["message_bound_ok"][0]) == 1 and int(want["target_only_ok"][0]) == 1
        contrib = got["raf.slot_contributors"].reshape(-1, 3)
        assert contrib[:, 2].min() >= 1 and contrib[:, 2].max() <= p
        if p == 1:
            assert int(want["sync_bytes"][0]) == 0 and contrib[:, 2].max() == 1


def test_make_batches_matches_reference_shuffle(H, ref):
    g = H.gen_synthetic(H.bundled_spec("mag-mini"), 5)
    batches = H.make_batches(g, 256, 0, H.mix_seed(5, 0xBA7C))
    assert len(batches) == 32 and sum(len(b) for b in batches) == 8000
    order = np.concatenate(batches)
    assert sorted(order.tolist()) == list(range(8000))
    # the reference's own bench helper shuffles identically (mix_seed(seed, 0xba7c))
    assert H.mix_seed(5, 0xBA7C) == ref.mix_seed(5, 0xBA7C)


def test_mix_seed_matches_reference(H, ref):
    rng = np.random.default_rng(0)
    for a, b in rng.integers(0, 2**63, size=(50, 2), dtype=np.uint64):
        assert H.mix_seed(int(a), int(b)) == ref.mix_seed(int(a), int(b))


# ---- cache planning ------------------------------------------------------------------

def test_cache_plan_matches_reference(H, ref):
    seed = 3
    rg = ref.RefGraph.bundled("mag-mini", seed)
    g = H.gen_synthetic(H.bundled_spec("mag-mini"), seed)
    for budget in (1 << 16, 1 << 20, 1 << 23):
        want = rg.cache_sim(2, [10, 10], 2, 77, 512, budget)
        got = H.cache_plan(g, want, 4, budget)
        for key in ("profile.ratio", "profile.transfer_ns", "profile.record_bytes", "alloc.bytes", "alloc.capacity"):
            assert np.array_equal(got[key], want[key]), key
        for t in range(4):
            assert np.array_equal(got[f"cached.t{t}"], want[f"cached.t{t}"]), (budget, t)


@pytest.mark.parametrize("name,chunk", [("mag-mini", None), ("donor-mini", None), ("mag-mini", "4099")])
def test_init_model_and_learnable_match_reference(H, ref, name, chunk, monkeypatch):
    # hg_init_model / hg_init_learnable (the caller-owned model state of the drop-in
    # layer interface) are the reference's init_model / init_learnable bit for bit; the
    # learnable tables are generated in jumped-ahead chunks (HG_FEAT_CHUNK values each)
    if chunk:
        monkeypatch.setenv("HG_FEAT_CHUNK", chunk)
    rg = ref.RefGraph.bundled(name, 5)
    g = H.gen_synthetic(H.bundled_spec(name), 5)
    want = rg.flat_step(2, 16, 77, 88, [0, 1, 2], [3, 3], 1)
    model = H.init_model(g, 2, 16, 77)
    learn = H.init_learnable(g, 88)
    slots = [n for n in want if n.startswith("init.r")]
    assert slots and len(slots) == len([n for n in model if n.startswith("w.")])
    for n in slots:
        assert np.array_equal(model["w." + n[len("init."):]], want[n]), n
    for n in [x for x in want if x.startswith("init.learn.t")]:
        assert np.array_equal(learn["learn.t" + n.split(".t")[-1]], want[n]), n


def test_work_aware_plan_groups(H):
    # the work-aware plan (not the reference's policy) on the ogbn-mag schema with the
    # per-sub sampled edges of SURVEY §8(e) (S0 92k, S1 213k, S2 200k) and learnable leaf
    # rows (S0 institution ~6k, S1 author + field ~118k, S2 none): the sub with the big
    # learnable merge stays unreplicated, the others are replicated together
    g = H.gen_synthetic(H.bundled_spec("mag-mini"), 5)  # the same 3-sub metatree shape
    w = [92.0e3, 213.3e3, 200.2e3, 5.6e3, 118e3, 0.0]
    groups = lambda plan, p: [tuple(int(x) for x in plan[f"part{i}.sub_ids"]) for i in range(p)]
    assert groups(H.meta_partition_work_aware(g, 2, 4, w), 4) == [(0, 2), (0, 2), (0, 2), (1,)]
    plan = H.meta_partition_work_aware(g, 2, 4, w)
    assert [list(plan[f"part{i}.replica"]) for i in range(4)] == [[1, 0, 3], [1, 1, 3], [1, 2, 3], [0, 0, 1]]
    # without the merge term the objective alone replicates everything (pure data parallel)
    assert groups(H.meta_partition_work_aware(g, 2, 2, w[:3]), 2) == [(0, 1, 2), (0, 1, 2)]
    # p = 1: one group with every sub
    assert groups(H.meta_partition_work_aware(g, 2, 1, w), 1) == [(0, 1, 2)]
    with pytest.raises(ValueError):
        H.meta_partition_work_aware(g, 2, 2, [1.0, 2.0])
