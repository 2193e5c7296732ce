"""Half-precision feature tables and the host-resident table with an HBM cache
(BASELINE configs[3] / SURVEY §8(d) C4: fp16 paper features that exceed HBM).

Parity mode: the reference's features rounded to fp16 / bf16 values
(oracle ref_graph_round_features) travel losslessly through a half-precision device
table, so one training step matches the f64 reference within 1e-3 and the layer-0
inputs exactly. A table kept in pinned host memory (read over PCIe) with an HBM copy
of the cached rows computes bit-identical steps to the same table in HBM."""
import numpy as np
import pytest

from tests.util import assert_adam_close, assert_close

pytestmark = pytest.mark.gpu
TOL = 1e-3


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
def test_half_feature_table_step_matches_reference(H, ref, dtype):
    rg = ref.RefGraph.bundled("mag-mini", 5)
    rg.round_features(dtype)
    g = H.gen_synthetic(H.bundled_spec("mag-mini"), 5)
    batch = list(range(0, 1024, 4))
    want = rg.flat_step(2, 32, 77, 88, batch, [25, 20], 11)
    eng = H.Engine(g, [25, 20], hidden=32, batch_cap=256, model_seed=77, learn_seed=88, feat_dtype=dtype)
    names = eng.tensor_names()
    rep = eng.step(batch, 11, 0, train=True)
    got = eng.read(*[n for n in names if not n.startswith("post.learn")])
    # layer-0 dense inputs are the rounded reference values exactly
    assert np.array_equal(got["H2.t0"], want["H2.t0"]), "paper features in the half table"
    assert abs(rep["loss"] - float(want["loss"][0])) <= TOL * abs(float(want["loss"][0]))
    for n in want:
        if n.startswith(("logits", "dlogits", "mean.", "grad.w.", "H1.")):
            assert_close(got[n], want[n], TOL, f"{dtype}: {n}")
        elif n.startswith("grad.f.") and n.endswith(".rows"):
            assert_close(got[n], want[n], TOL, f"{dtype}: {n}")
        elif n.startswith("post.r"):
            assert_adam_close(got[n], want[n], None, steps=1, what=f"{dtype}: {n}")


@pytest.mark.parametrize("dtype", ["f32", "f16"])
def test_host_resident_table_with_hbm_cache_is_bit_identical(H, dtype):
    g = H.gen_synthetic(H.bundled_spec("mag-mini"), 5)
    batches = H.make_batches(g, 128, 4, H.mix_seed(5, 0xBA7C))
    seeds = [H.mix_seed(5, 0xB000 + i) for i in range(len(batches))]
    dev = H.Engine.for_experiment(g, [25, 20], 32, 5, batch_cap=128, feat_dtype=dtype)
    host = H.Engine.for_experiment(g, [25, 20], 32, 5, batch_cap=128, feat_dtype=dtype, feat_host=True)
    # half of the paper rows (and a third of the fields) cached in HBM, the rest read from
    # pinned host memory; the first two steps run before the cache exists
    cached = [np.arange(0, 8000, 2, dtype=np.uint32), np.zeros(0, np.uint32), np.zeros(0, np.uint32),
              np.arange(0, 1000, 3, dtype=np.uint32)]
    for i, (b, s) in enumerate(zip(batches, seeds)):
        if i == 2:
            dev.set_cache(cached)
            host.set_cache(cached)
        a, c = dev.step(b, s), host.step(b, s)
        assert a["loss"] == c["loss"], (i, a["loss"], c["loss"])
    names = [n for n in dev.tensor_names() if n.startswith(("logits", "grad.", "post.r", "H"))]
    x, y = dev.read(*names), host.read(*names)
    for n in names:
        assert np.array_equal(x[n], y[n]), n
    assert {k: v.tolist() for k, v in dev.cache_counters().items()} == \
           {k: v.tolist() for k, v in host.cache_counters().items()}


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
def test_ragged_width_half_tables_match_reference(H, ref, dtype):
    """Dense widths that are not multiples of the 8-feature lanes (100 and 36: the last
    lane of a row's chunk is partly padding) and an fp32 learnable type in the same
    half-precision gather launch, against the f64 reference on the rounded features."""
    spec = dict(name="ragged", target="paper", num_classes=7, label_noise=0.1,
                node_types=[dict(name="paper", count=3000, dim=100, storage="dense"),
                            dict(name="venue", count=400, dim=36, storage="dense"),
                            dict(name="author", count=2500, dim=20, storage="learnable")],
                relations=[dict(src="paper", edge="cites", dst="paper", edges=24000),
                           dict(src="venue", edge="hosts", dst="paper", edges=3000),
                           dict(src="author", edge="writes", dst="paper", edges=9000),
                           dict(src="paper", edge="in", dst="venue", edges=3000)],
                self_paired=["cites"])
    g = H.gen_synthetic(spec, 9)
    rg = ref.RefGraph.from_spec(spec, 9)
    rg.round_features(dtype)
    batch = list(range(0, 2048, 8))
    want = rg.flat_step(2, 32, 3, 4, batch, [25, 20], 13)
    eng = H.Engine(g, [25, 20], hidden=32, batch_cap=256, model_seed=3, learn_seed=4, feat_dtype=dtype)
    names = eng.tensor_names()
    rep = eng.step(batch, 13, 0, train=True)
    got = eng.read(*[n for n in names if not n.startswith("post.learn")])
    assert abs(rep["loss"] - float(want["loss"][0])) <= TOL * abs(float(want["loss"][0]))
    checked = 0
    for n in want:
        if n.startswith(("logits", "dlogits", "mean.", "grad.w.", "H1.")):
            assert_close(got[n], want[n], TOL, f"{dtype}: {n}")
            checked += 1
        elif n.startswith("grad.f.") and n.endswith(".rows"):
            assert_close(got[n], want[n], TOL, f"{dtype}: {n}")
            checked += 1
    assert checked > 10
