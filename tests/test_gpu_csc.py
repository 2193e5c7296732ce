"""The backward scatter of a hub source (hgnn.cpp:344-353): a power-law graph's hub
collects thousands of sampled edges in one transposed (CSC) segment. The segment is
sorted by a whole warp (bitonic in shared memory, merged runs beyond 1024 entries),
so its gradient is summed in the same (block, row) order every run: bit-identical
across fresh engines, and within 1e-3 of the reference."""
import numpy as np
import pytest

from tests.util import assert_close, csr_from_pairs

pytestmark = pytest.mark.gpu


def hub_graph(H, ref, n_dst, n_src=12, dim=8, seed=0):
    # every destination row has the hub (source 0) plus two others
    pairs = []
    for d in range(n_dst):
        for s in (0, 1 + d % (n_src - 1), 1 + (d * 7 + 3) % (n_src - 1)):
            pairs.append((s, d))
    rng = np.random.default_rng(seed)
    feat0 = rng.uniform(-1, 1, (n_dst, dim)).astype(np.float32)
    labels = (np.arange(n_dst) % 3).astype(np.int32)
    indptr, src = csr_from_pairs(n_dst, pairs)
    e = {"node_counts": np.array([n_dst, n_src], np.uint64), "rel_src": np.array([1], np.int32),
         "rel_dst": np.array([0], np.int32), "rel_reverse": np.array([0], np.int32),
         "rel0.indptr": indptr, "rel0.src": src, "kinds": np.array([1, 2], np.int32),
         "dims": np.array([dim, dim], np.int32), "feat.t0": feat0, "labels": labels,
         "target": np.array([0]), "num_classes": np.array([3])}
    g = H.graph_from_export(e)
    rg = ref.RefGraph.build([n_dst, n_src], [(1, 0)], [pairs], 0, 3, labels, [1, 2], [dim, dim],
                            [feat0.astype(np.float64)])
    return g, rg


@pytest.mark.parametrize("n_dst", [700, 3000])
def test_hub_segment_gradient_deterministic_and_exact(H, ref, n_dst):
    g, rg = hub_graph(H, ref, n_dst)
    batch = list(range(n_dst))
    want = rg.flat_step(1, 6, 3, 4, batch, [5], 17)
    rows = []
    for _ in range(2):
        eng = H.Engine(g, [5], hidden=6, batch_cap=n_dst, model_seed=3, learn_seed=4)
        eng.step(batch, 17, 0, train=True)
        got = eng.read("grad.f.t1.ids", "grad.f.t1.rows")
        assert np.array_equal(got["grad.f.t1.ids"], want["grad.f.t1.ids"])
        assert_close(got["grad.f.t1.rows"], want["grad.f.t1.rows"], 1e-3, "hub gradient rows")
        rows.append(got["grad.f.t1.rows"])
    assert np.array_equal(rows[0], rows[1]), "hub gradient not bit-reproducible"
