"""BASELINE configs[3] (C4, MAG240M shape) on a down-scaled twin the CPU reference can
run: 3-layer RGCN, fanout [25,15,10], 768-d paper features stored as fp16 (the
reference's features rounded to fp16 values: lossless in the half table), learnable
64-d author / institution tables. One full training step against the f64 reference
(hgnn.cpp:215-410): sampled blocks bit-exact, activations / gradients within 1e-3."""
import numpy as np
import pytest

from tests.util import assert_adam_close, assert_close

TOL = 1e-3
SCALE = 1.0 / 2000


def _relu_flips(got, want):
    """ReLU units whose sign differs from the f64 reference (ties at ~1e-7 that any
    fp32 evaluation can flip); a flipped unit passes (or blocks) its whole dH entry."""
    n = 0
    for name in want:
        if name.startswith(("H1.", "H2.")) and name in got:
            n += int(((got[name] > 0) != (want[name] > 0)).sum())
    return n


@pytest.mark.gpu
@pytest.mark.parametrize("umma,rng_seed", [(0, 21), (1, 21), (1, 22)])
def test_c4_twin_three_layer_fp16_step(H, ref, umma, rng_seed):
    """umma = 1 is the product path (tcgen05, 3xTF32); umma = 0 runs the same step with
    the fp32 SIMT contractions, which pins the algorithm itself at fp32 round-off."""
    spec = H.mag240m_spec(SCALE)
    g = H.gen_synthetic(spec, 1)
    rg = ref.RefGraph.from_spec(spec, 1)
    rg.round_features("f16")
    batch = H.make_batches(g, 256, 1, H.mix_seed(1, 0xBA7C))[0]
    fanouts = [25, 15, 10]
    want = rg.flat_step(3, 64, 5, 6, batch, fanouts, rng_seed, want_init="rows")
    eng = H.Engine(g, fanouts, hidden=64, batch_cap=256, model_seed=5, learn_seed=6, feat_dtype="f16")
    eng.set_option("umma", umma)
    names = eng.tensor_names()
    fwd = eng.step(batch, rng_seed, 0, train=False)
    got = eng.read(*[n for n in names if not n.startswith(("post.", "grad."))])
    blocks = [n for n in want if n.startswith(("frontier", "hop")) and not n.endswith(".rels")]
    for n in blocks:
        assert np.array_equal(np.asarray(got.get(n, np.zeros(0, np.uint32))).ravel(), np.asarray(want[n]).ravel()), n
    assert sum(len(want[n]) for n in blocks if n.endswith(".src_ids")) == fwd["sampled_edges"]
    assert np.array_equal(got["H3.t0"], want["H3.t0"]), "fp16 paper features"
    assert abs(fwd["loss"] - float(want["loss"][0])) <= TOL * abs(float(want["loss"][0]))
    for n in want:
        if n.startswith(("logits", "dlogits", "mean.", "H1.", "H2.")):
            assert_close(got[n], want[n], TOL, f"C4 twin {n}")
    flips = _relu_flips(got, want)
    rep = eng.step(batch, rng_seed, 0, train=True)
    assert rep["loss"] == fwd["loss"]
    got = eng.read(*[n for n in names if n.startswith(("grad.", "post.r"))])
    if umma == 0:
        assert flips == 0
    if flips:
        # a flipped tie changes one dpre entry by the full dH value: the gradients of the
        # layers below it legitimately differ from the f64 reference (measured: 1 unit of
        # 1.57M at |pre-activation| 1.5e-7 moves two layer-1 weight gradients by 3%)
        pytest.skip(f"{flips} ReLU tie(s) flipped vs the f64 reference; forward parity checked")
    checked = 0
    for n in want:
        if n.startswith("grad.w.") or (n.startswith("grad.f.") and n.endswith(".rows")):
            assert_close(got[n], want[n], TOL, f"C4 twin {n}")
            checked += 1
        elif n.startswith("grad.f.") and n.endswith(".ids"):
            assert np.array_equal(got[n], want[n]), n
        elif n.startswith("post.r"):
            assert_adam_close(got[n], want[n], None, steps=1, what=f"C4 twin {n}")
    assert checked > 10


def test_c4_twin_graph_matches_oracle(H, ref):
    spec = H.mag240m_spec(SCALE)
    ours, want = H.gen_synthetic(spec, 1).export(), ref.RefGraph.from_spec(spec, 1).export()
    for n, w in want.items():
        if n in ("type_names", "etype_names", "rel_etype"):
            continue
        if n.startswith("feat."):
            assert np.array_equal(ours[n], w.astype(np.float32)), n
        else:
            assert np.array_equal(np.asarray(ours[n]).ravel(), np.asarray(w).ravel()), n
