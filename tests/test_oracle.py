"""Pins the oracle before trusting it (CPU, no GPU).

The oracle is two things: the compiled reference (oracle/_ref) and a pure
Python/numpy restatement (oracle/port.py). Here the restatement is checked
against the C++ standard's published mt19937_64 known answer, the reference's
own known-answer tests (test_hgnn.cpp, test_cache.cpp), the compiled reference,
and the committed golden fixtures (tests/golden/, made by make_golden.py)."""
import os

import numpy as np
import pytest

from oracle import port as P

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name):
    return dict(np.load(os.path.join(GOLDEN, name)))


def sub(d, prefix):
    return {k[len(prefix):]: v for k, v in d.items() if k.startswith(prefix)}


def test_mt19937_64_standard_known_answer():
    # [rand.predef]: the 10000th invocation of a default-constructed
    # mt19937_64 (seed 5489) yields 9981545732273789042
    eng = P.MT19937_64(5489)
    for _ in range(9999):
        eng()
    assert eng() == 9981545732273789042


def test_mix_seed_matches_reference(ref):
    rng = np.random.default_rng(1)
    for a, b in rng.integers(0, 2**63, size=(100, 2), dtype=np.uint64):
        assert P.mix_seed(int(a), int(b)) == ref.mix_seed(int(a), int(b))


def test_sample_neighbors_kats():
    # test_sampling.cpp:12-31
    assert P.sample_neighbors([0, 3], [7, 5, 9], 0, 3, 42, 1, 0) == [7, 5, 9]
    assert P.sample_neighbors([0, 3], [7, 5, 9], 0, 10, 42, 1, 0) == [7, 5, 9]
    s1 = P.sample_neighbors([0, 20], list(range(20)), 0, 8, 42, 1, 0)
    assert s1 == P.sample_neighbors([0, 20], list(range(20)), 0, 8, 42, 1, 0)
    assert len(set(s1)) == 8
    assert P.sample_neighbors([0, 20], list(range(20)), 0, 8, 43, 1, 0) != s1
    assert P.sample_neighbors([0, 20], list(range(20)), 0, 8, 42, 2, 0) != s1


def test_sample_rows_golden():
    g = golden("sample_rows.npz")
    for fanout in (8, 25, 160):
        for d in range(3):
            got = P.sample_neighbors(g["indptr"], g["src"], d, fanout, 42, 1, 0)
            assert got == g[f"f{fanout}.d{d}"].tolist(), (fanout, d)


@pytest.mark.parametrize("seed", [10, 11, 12, 13])
def test_sample_khop_golden(seed):
    g = golden(f"sample_random{seed}.npz")
    graph = P.Graph(sub(g, "graph."))
    hs = [g["hop_rels1"].tolist(), g["hop_rels2"].tolist()]
    b = P.sample_khop(graph, g["seeds"].tolist(), [3, 3], seed * 31 + 1, hs)
    want = sub(g, "sample.")
    for h, blocks in enumerate(b["hops"], start=1):
        assert [blk["rel"] for blk in blocks] == want[f"hop{h}.rels"].tolist()
        for blk in blocks:
            p = f"hop{h}.rel{blk['rel']}"
            assert blk["dst_ids"] == want[f"{p}.dst_ids"].tolist()
            assert blk["indptr"] == want[f"{p}.indptr"].tolist()
            assert blk["src_ids"] == want[f"{p}.src_ids"].tolist()
    for h in range(3):
        for t in range(graph.ntypes):
            assert b["frontier"][h][t] == want[f"frontier{h}.t{t}"].tolist()


@pytest.mark.parametrize("seed", range(20, 26))
def test_sample_khop_vs_reference(ref, seed):
    rg = ref.RefGraph.random(seed)
    g = P.Graph(rg.export())
    b = P.sample_khop(g, [0, 1, 2], [4, 2], 1234 + seed)
    want = rg.sample_khop([0, 1, 2], [4, 2], 1234 + seed)
    for h, blocks in enumerate(b["hops"], start=1):
        for blk in blocks:
            assert blk["src_ids"] == want[f"hop{h}.rel{blk['rel']}.src_ids"].tolist()


def test_flat_step_golden():
    g = golden("flat_step_random100.npz")
    graph = P.Graph(sub(g, "graph."))
    st = sub(g, "step.")
    tree = P.bfs_metatree(graph, 2)
    weights = {}
    for k, v in st.items():
        if k.startswith("init.r"):
            r, l = k[len("init.r"):].split(".l")
            weights[(int(r), int(l))] = v.copy()
    learn = {int(k.split(".t")[-1]): v.copy() for k, v in st.items() if k.startswith("init.learn.t")}
    batch = [0, 1, 2, 3]
    blocks = P.sample_khop(graph, batch, [3, 3], 105, P.hop_relation_sets(tree, 2))
    logits, H, tape = P.forward_flat(graph, tree, blocks, weights, learn, 5)
    np.testing.assert_allclose(logits, st["logits"], rtol=1e-10, atol=1e-12)
    loss, dz = P.cross_entropy(logits, blocks["frontier"][0][graph.target], batch, graph.labels, graph.num_classes)
    assert abs(loss - st["loss"][0]) < 1e-10
    np.testing.assert_allclose(dz, st["dlogits"], rtol=1e-9, atol=1e-12)
    wg, fg = P.backward_flat(graph, tree, blocks, H, tape, weights, dz)
    for (r, l), v in wg.items():
        np.testing.assert_allclose(v, st[f"grad.w.r{r}.l{l}"], rtol=1e-9, atol=1e-12)
    for t, (ids, rows) in fg.items():
        assert ids == st[f"grad.f.t{t}.ids"].tolist()
        np.testing.assert_allclose(rows, st[f"grad.f.t{t}.rows"], rtol=1e-9, atol=1e-12)
    # first Adam step (adam_update_model: step 1 for every slot with a gradient)
    for (r, l), w in weights.items():
        if (r, l) in wg:
            m, v = np.zeros_like(w), np.zeros_like(w)
            P.adam_step(w, m, v, wg[(r, l)], 1)
        np.testing.assert_allclose(w, st[f"post.r{r}.l{l}"], rtol=1e-9, atol=1e-12)


def test_cross_entropy_kat():
    # test_hgnn.cpp:76-92
    loss, d = P.cross_entropy(np.zeros((4, 3)), [0, 1, 2, 3], [1, 3], [0, 1, 2, 0], 3)
    assert abs(loss - np.log(3.0)) < 1e-12
    assert np.all(d[0] == 0)
    assert abs(d[1, 1] - (1 / 3 - 1) / 2) < 1e-12 and abs(d[1, 0] - (1 / 3) / 2) < 1e-12
    assert abs(d[1].sum()) < 1e-12


def test_adam_first_step_kat():
    # test_hgnn.cpp:151-175: a bias-corrected first step moves by lr * sign(g)
    w, m, v = np.array([-0.25]), np.zeros(1), np.zeros(1)
    P.adam_step(w, m, v, np.array([2.0]), 1)
    assert abs(w[0] - (-0.25 - 1e-2)) < 1e-8


def test_cache_golden_and_kats():
    g = golden("cache_magmini3.npz")
    hot = [g[f"hot.t{t}"] for t in range(4)]
    kinds = [1, 2, 2, 2]
    graph = type("G", (), {})()
    graph.ntypes, graph.kinds, graph.dims = 4, kinds, [128, 64, 64, 64]
    prof = P.profile_miss_penalty(graph)
    np.testing.assert_array_equal([p["ratio"] for p in prof], g["profile.ratio"])
    cap, nbytes = P.allocate_cache(1 << 20, hot, prof)
    assert cap == g["alloc.capacity"].tolist() and nbytes == g["alloc.bytes"].tolist()
    for t, c in enumerate(P.fill_and_serve(cap, hot)):
        assert c.tolist() == g[f"cached.t{t}"].tolist()
    # test_cache.cpp:112-134 top-k {1,2,4}; :136-165 hits/misses/penalty
    assert P.fill_and_serve([3], [[5, 9, 9, 1, 9]])[0].tolist() == [1, 2, 4]
    st = P.cache_lookups([0, 1], np.array([0]), True, 100.0)
    assert st == dict(hits=2, misses=2, penalty_ns=200.0)


def test_presample_hotness_vs_reference(ref):
    rg = ref.RefGraph.random(7)
    g = P.Graph(rg.export())
    tree = P.bfs_metatree(g, 2)
    got = P.presample_hotness(g, tree, [3, 3], 2, 99, 4)
    want = rg.cache_sim(2, [3, 3], 2, 99, 4)
    for t in range(g.ntypes):
        assert got[t].tolist() == want[f"hot.t{t}"].tolist()
