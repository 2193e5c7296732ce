"""GPU numerics parity against the compiled reference: forward tape, logits,
loss, dlogits, gradients and the first Adam step (hgnn.cpp:215-410), plus a
multi-batch RAF training trajectory (raf.cpp:344-530, harness.cpp:400-423).
Tolerance: 1e-3 relative per tensor (max|diff| / max|ref|), BASELINE north_star."""
import numpy as np
import pytest

from tests.util import assert_adam_close, assert_close

pytestmark = pytest.mark.gpu

TOL = 1e-3


def check_flat_step(H, ref, rg, g, k, fanouts, hidden, batch, rng_seed, what):
    want = rg.flat_step(k, hidden, 77, 88, batch, fanouts, rng_seed)
    eng = H.Engine(g, fanouts, hidden=hidden, batch_cap=max(8, len(batch)), model_seed=77, learn_seed=88)
    # initial parameters are bit-identical to the reference's init (f64 -> f32)
    names = eng.tensor_names()
    for n in [x for x in want if x.startswith("init.r")]:
        got_w = eng.read("post." + n[len("init."):])["post." + n[len("init."):]]
        assert np.array_equal(got_w, want[n].astype(np.float32).astype(np.float64)), f"{what}: init {n}"
    # forward + loss only first: the tape and layer-0 inputs before any update
    fwd = eng.step(batch, rng_seed, 0, train=False)
    got = eng.read(*[n for n in names if not n.startswith(("post.", "grad."))])
    assert abs(fwd["loss"] - float(want["loss"][0])) <= TOL * max(1.0, abs(float(want["loss"][0]))), what
    assert_close(got["logits"], want["logits"], TOL, f"{what}: logits")
    assert_close(got["dlogits"], want["dlogits"], TOL, f"{what}: dlogits")
    for n in want:
        if (n.startswith("H") or n.startswith("mean.")) and n in got:
            assert_close(got[n], want[n], TOL, f"{what}: {n}")
    # the same batch again, now with backward and Adam
    rep = eng.step(batch, rng_seed, 0, train=True)
    assert rep["loss"] == fwd["loss"], what
    got = eng.read(*names)
    for n in want:
        if n.startswith("grad.w."):
            assert_close(got[n], want[n], TOL, f"{what}: {n}")
        if n.startswith("grad.f.") and n.endswith(".ids"):
            assert np.array_equal(got[n], want[n]), f"{what}: {n}"
        if n.startswith("grad.f.") and n.endswith(".rows"):
            assert_close(got[n], want[n], TOL, f"{what}: {n}")
    for n in want:
        if n.startswith("post.r"):
            init = want["init." + n[len("post."):]]
            assert_adam_close(got[n], want[n], init, what=f"{what}: {n}")
        if n.startswith("post.learn.t"):
            t = n.split(".t")[-1]
            if n in got:
                assert_adam_close(got[n], want[n], want[f"init.learn.t{t}"], what=f"{what}: {n}")
            else:
                # not a layer-0 type of this tree: never read, never updated
                assert np.array_equal(want[n], want[f"init.learn.t{t}"]), f"{what}: {n}"


@pytest.mark.parametrize("seed", list(range(100, 112)))
def test_flat_step_random_graphs(H, ref, seed):
    rg = ref.RefGraph.random(seed, 4, 5, 60)
    ex = rg.export()
    g = H.graph_from_export(ex)
    n_target = int(ex["node_counts"][0])
    batch = list(range(min(4, n_target)))
    check_flat_step(H, ref, rg, g, 2, [3, 3], 5, batch, 5 + seed, f"random {seed}")


def test_flat_step_duplicate_seeds(H, ref):
    rg = ref.RefGraph.random(3)
    g = H.graph_from_export(rg.export())
    check_flat_step(H, ref, rg, g, 2, [3, 2], 6, [0, 1, 2, 1, 1], 99, "duplicates")


@pytest.mark.parametrize("name", ["mag-mini", "igb-mini", "freebase-mini", "donor-mini"])
def test_flat_step_bundled(H, ref, name):
    rg = ref.RefGraph.bundled(name, 5)
    g = H.gen_synthetic(H.bundled_spec(name), 5)
    batch = list(range(0, 2048, 3))[:256]
    check_flat_step(H, ref, rg, g, 2, [25, 20], 32, batch, 11, name)


def test_flat_step_three_layers(H, ref):
    rg = ref.RefGraph.bundled("mag-mini", 5)
    g = H.gen_synthetic(H.bundled_spec("mag-mini"), 5)
    check_flat_step(H, ref, rg, g, 3, [10, 10, 5], 16, list(range(128)), 3, "mag-mini k=3")


@pytest.mark.parametrize("name", ["mag-mini", "freebase-mini"])
def test_raf_training_trajectory(H, ref, name):
    """Several consecutive batches through run_raf_batch + Adam (harness.cpp:403-423):
    per-batch losses and the final parameters track the f64 reference."""
    seed = 5
    rg = ref.RefGraph.bundled(name, seed)
    g = H.gen_synthetic(H.bundled_spec(name), seed)
    batches = H.make_batches(g, 64, 6, H.mix_seed(seed, 0xBA7C))
    want = rg.raf_train(2, 32, 1, seed, [list(b) for b in batches], [25, 20])
    eng = H.Engine.for_experiment(g, [25, 20], 32, seed, batch_cap=64)
    losses = []
    for i, b in enumerate(batches):
        losses.append(eng.step(b, H.mix_seed(seed, 0xB000 + i), i % 1)["loss"])
    np.testing.assert_allclose(losses, want["losses"], rtol=TOL, atol=0)
    got = eng.read(*eng.tensor_names())
    for n in want:
        if n.startswith("final.r"):
            key = "post." + n[len("final."):]
            assert_adam_close(got[key], want[n], None, max_flip_frac=5e-3, steps=len(batches),
                              what=f"{name}: {key}")
        if n.startswith("final.learn_step.t"):
            t = n.split(".t")[-1]
            mine = int(got[f"post.learn_step.t{t}"][0]) if f"post.learn_step.t{t}" in got else 0
            assert mine == int(want[n][0]), f"{name}: step of type {t}"
        if n.startswith("final.learn.t") and "post.learn.t" + n.split(".t")[-1] in got:
            key = "post.learn.t" + n.split(".t")[-1]
            assert_adam_close(got[key], want[n], None, max_flip_frac=5e-3, steps=len(batches),
                              what=f"{name}: {key}")


@pytest.mark.parametrize("name", ["mag-mini", "donor-mini"])
def test_tensor_core_contractions_match_fp32_tiles(H, name):
    # The tcgen05 (3xTF32) projection / weight-grad / mean-grad kernels against
    # the SIMT fp32 tile kernels on identical inputs: fp32-level agreement
    # (tf32 split error ~2^-21), far inside the 1e-3 parity budget.
    g = H.gen_synthetic(H.bundled_spec(name), 4)
    batch = list(range(0, 600, 2))
    outs = []
    for umma in (0, 1):
        eng = H.Engine(g, [10, 5], hidden=32, batch_cap=512, model_seed=5, learn_seed=6)
        eng.set_option("umma", umma)
        eng.step(batch, 99, 0, train=True)
        # H2.* (layer-0 learnable rows) and post.* are read after Adam, whose
        # +-lr steps flip for gradients at rounding level: compared separately
        names = [n for n in eng.tensor_names()
                 if n.startswith(("H0", "H1", "logits", "dlogits", "grad.w.", "grad.f."))]
        outs.append(eng.read(*names))
    simt, tc = outs
    for n in simt:
        if n.endswith(".ids"):
            assert np.array_equal(simt[n], tc[n]), n
        else:
            assert_close(tc[n], simt[n], 2e-5, f"{name}: {n} (tcgen05 vs fp32 tiles)")


def test_tensor_core_tile_shapes():
    # every tile width (32/64/128 columns, multi-tile 349), partial row tiles,
    # K chunk counts (din not a multiple of 4 / 32), 1-3 relations per group,
    # split-K chunk edges (255/256/257 rows): tcgen05 vs fp32 tiles
    import ctypes as C
    from paper_2408_09697_b200 import _native as N
    cases = []
    for rows in (1, 7, 128, 257, 1000):
        for nrel, din, dout in ((1, 2, 3), (2, 5, 8), (3, 17, 33), (1, 32, 64), (2, 64, 64), (3, 128, 64),
                                (1, 64, 349), (2, 100, 100), (1, 128, 128), (3, 64, 349)):
            cases.append((rows, nrel, din, dout))
    arr = np.asarray(cases, np.int32).ravel()
    err = N.take(N.lib().hg_selftest_contractions(N.ptr(arr), len(cases), 0))["err"]
    bad = [(cases[i], err[i].tolist()) for i in range(len(cases)) if not np.all(err[i] < 2e-5)]
    assert not bad, bad[:8]


def test_toy_config_run_experiment(H, ref):
    # BASELINE configs[0]: 4 types x 128-d dense, 5 uniform
    # relations without reverses, fanout [10,10], hidden 64, batch 1024: the
    # per-batch losses of the reference's run_experiment, batch by batch
    spec = H.toy_spec()
    seed, nb = 1, 3
    cfg = {"spec": spec, "partitioner": "meta", "p": 1, "engine": "raf", "fanouts": [10, 10], "hidden": 64,
           "batch_size": 1024, "epochs": 1, "max_batches_per_epoch": nb, "seed": seed}
    stats, _, ok = ref.run_experiment(cfg)
    assert ok
    g = H.gen_synthetic(spec, seed)
    eng = H.Engine.for_experiment(g, [10, 10], 64, seed, batch_cap=1024)
    batches = H.make_batches(g, 1024, nb, H.mix_seed(seed, 0xBA7C))
    reps = [eng.step(b, H.mix_seed(seed, 0xB000 + i), 0) for i, b in enumerate(batches)]
    np.testing.assert_allclose([r["loss"] for r in reps], [b["loss"] for b in stats["batches"]], rtol=1e-3, atol=0)
    # the per-batch stats entry of run_experiment (harness.cpp:410-446)
    for r, want in zip(reps, stats["batches"]):
        assert r["boundary_counts"] == want["boundary_counts"]
        assert r["sync_bytes"] == want["sync_bytes"] and r["sync_leader"]
        assert r["message_bound_ok"] == want["message_bound_ok"]
        assert r["target_only_ok"] == want["target_only_ok"]


def test_prefetch_pipeline_is_bit_identical(H):
    # sampling batch i+1 (second sample slot, sampling stream) while batch i
    # trains must not change a single bit of the training trajectory
    g = H.gen_synthetic(H.bundled_spec("mag-mini"), 5)
    batches = H.make_batches(g, 128, 6, H.mix_seed(5, 0xBA7C))
    seeds = [H.mix_seed(5, 0xB000 + i) for i in range(len(batches))]
    plain = H.Engine.for_experiment(g, [25, 20], 32, 5, batch_cap=128)
    ref_losses = [plain.step(b, s)["loss"] for b, s in zip(batches, seeds)]
    piped = H.Engine.for_experiment(g, [25, 20], 32, 5, batch_cap=128)
    piped.prefetch(batches[0], seeds[0])
    losses = []
    for i, (b, s) in enumerate(zip(batches, seeds)):
        if i + 1 < len(batches):
            piped.prefetch(batches[i + 1], seeds[i + 1])
        losses.append(piped.step(b, s)["loss"])
    assert losses == ref_losses
    names = [n for n in plain.tensor_names() if n.startswith("post.")]
    a, b = plain.read(*names), piped.read(*names)
    for n in names:
        assert np.array_equal(a[n], b[n]), n
    # a step whose batch was not prefetched still samples it (stale prefetch dropped)
    piped.prefetch(batches[1], seeds[1])
    r = piped.step(batches[2], seeds[2])
    assert np.isfinite(r["loss"])
