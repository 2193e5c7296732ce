"""RGAT layer type (BASELINE configs[2]).

The reference has no attention layer, so the checker is the framework's own f64
restatement, oracle/rgat.py. It is pinned here by central finite differences of its
loss (CPU), then the device path (tcgen05 projections + the attention kernels of
csrc/rgat_kernels.cu) is compared with it on the same sampled blocks (GPU):
forward activations, logits, loss, weight / attention / learnable-row gradients
within 1e-3 relative, and the post-Adam model within the one-flip bound."""
import numpy as np
import pytest

from oracle import port
from oracle import rgat as R
from tests.util import assert_adam_close, assert_close

TOL = 1e-3
FANOUTS = [10, 8]
HIDDEN = 32
HEADS = 4
BATCH = list(range(0, 512, 4))
RNG_SEED = 11


def blocks_from(arrays, k, ntypes, nrels):
    """port-style SampledBlocks from exported arrays (frontier{h}.t{t}, hop{h}.rel{r}.*)."""
    frontier = [[[int(x) for x in np.asarray(arrays.get(f"frontier{h}.t{t}", []))] for t in range(ntypes)]
                for h in range(k + 1)]
    hops = []
    for h in range(1, k + 1):
        blks = []
        for r in range(nrels):
            key = f"hop{h}.rel{r}"
            if key + ".indptr" not in arrays:
                continue
            blks.append(dict(rel=r, dst_ids=[int(x) for x in arrays[key + ".dst_ids"]],
                             indptr=[int(x) for x in arrays[key + ".indptr"]],
                             src_ids=[int(x) for x in arrays[key + ".src_ids"]]))
        hops.append(blks)
    return dict(k=k, hops=hops, frontier=frontier)


@pytest.fixture(scope="module")
def mini(ref):
    rg = ref.RefGraph.bundled("mag-mini", 5)
    g = port.Graph(rg.export())
    tree = port.bfs_metatree(g, 2)
    sampled = rg.sample_khop(BATCH, FANOUTS, RNG_SEED, port.hop_relation_sets(tree, 2))
    return rg, g, tree, blocks_from(sampled, 2, g.ntypes, g.nrels)


def random_params(g, tree, seed):
    rng = np.random.default_rng(seed)
    weights, att = {}, {}
    for (_, depth, _, r) in tree:
        if r < 0:
            continue
        layer = 2 - depth + 1
        din = g.dims[g.rel_src[r]] if layer == 1 else HIDDEN
        dout = g.num_classes if layer == 2 else HIDDEN
        weights[(r, layer)] = rng.normal(0, 0.3, (din, dout))
        att[(r, layer)] = rng.normal(0, 0.5, dout)
    learn = {t: rng.normal(0, 0.5, (g.counts[t], g.dims[t])) for t in range(g.ntypes) if g.kinds[t] == 2}
    return weights, att, learn


def test_oracle_gradients_match_finite_differences(mini):
    _, g, tree, blocks = mini
    weights, att, learn = random_params(g, tree, 3)
    loss, _, _, _, wg, ag, fg = R.step(g, tree, blocks, weights, att, learn, HIDDEN, HEADS, BATCH)

    def loss_of():
        return R.step(g, tree, blocks, weights, att, learn, HIDDEN, HEADS, BATCH)[0]

    rng = np.random.default_rng(7)
    eps = 1e-6
    checked = 0
    for table, grads in ((weights, wg), (att, ag)):
        for key in sorted(grads)[:6]:
            arr = table[key]
            for _ in range(2):
                idx = tuple(int(rng.integers(0, n)) for n in arr.shape)
                old = arr[idx]
                arr[idx] = old + eps
                lp = loss_of()
                arr[idx] = old - eps
                lm = loss_of()
                arr[idx] = old
                num = (lp - lm) / (2 * eps)
                ana = grads[key][idx]
                assert abs(num - ana) <= 1e-5 * max(1.0, abs(ana)) + 1e-7, (key, idx, num, ana)
                checked += 1
    for t, (ids, rows) in fg.items():
        for q in rng.integers(0, len(ids), 3):
            c = int(rng.integers(0, rows.shape[1]))
            old = learn[t][ids[q], c]
            learn[t][ids[q], c] = old + eps
            lp = loss_of()
            learn[t][ids[q], c] = old - eps
            lm = loss_of()
            learn[t][ids[q], c] = old
            assert abs((lp - lm) / (2 * eps) - rows[q, c]) <= 1e-5 * max(1.0, abs(rows[q, c])) + 1e-7
            checked += 1
    assert checked >= 20 and np.isfinite(loss)


def _relu_flips(got, H_want, blocks, g):
    n = 0
    for t in range(g.ntypes):
        if t in H_want[1] and f"H1.t{t}" in got:
            n += int(((got[f"H1.t{t}"] > 0) != (H_want[1][t] > 0)).sum())
    return n


@pytest.mark.gpu
@pytest.mark.parametrize("umma", [1, 0])
def test_rgat_step_matches_oracle(H, mini, umma):
    rg, g, tree, blocks = mini
    gd = H.gen_synthetic(H.bundled_spec("mag-mini"), 5)
    eng = H.Engine(gd, FANOUTS, hidden=HIDDEN, batch_cap=len(BATCH), model_seed=77, learn_seed=88, model="rgat",
                   heads=HEADS)
    eng.set_option("umma", umma)
    names = eng.tensor_names()
    init = eng.read(*[n for n in names if n.startswith(("post.r", "att.", "post.learn.t"))])
    weights = {(int(n.split(".")[1][1:]), int(n.split(".")[2][1:])): init[n] for n in init if n.startswith("post.r")}
    att = {(int(n.split(".")[1][1:]), int(n.split(".")[2][1:])): init[n].ravel() for n in init if n.startswith("att.")}
    learn = {int(n.split(".t")[-1]): init[n] for n in init if n.startswith("post.learn.t")}
    assert len(weights) == len(att) >= 6 and learn
    loss, logits, Hw, dl, wg, ag, fg = R.step(g, tree, blocks, weights, att, learn, HIDDEN, HEADS, BATCH)

    fwd = eng.step(BATCH, RNG_SEED, 0, train=False)
    got = eng.read(*[n for n in names if n.startswith(("frontier", "hop", "H1.", "logits", "dlogits"))
                     and not n.endswith(".col")])
    # the device sampler's blocks are the reference's (model-independent)
    mine = blocks_from(got, 2, g.ntypes, g.nrels)
    assert mine["frontier"] == blocks["frontier"] and mine["hops"] == blocks["hops"]
    assert abs(fwd["loss"] - loss) <= TOL * abs(loss)
    assert_close(got["logits"], logits, TOL, "RGAT logits")
    assert_close(got["dlogits"], dl, TOL, "RGAT dlogits")
    for t in range(g.ntypes):
        if t in Hw[1]:
            assert_close(got[f"H1.t{t}"], Hw[1][t], TOL, f"RGAT H1.t{t}")
    flips = _relu_flips(got, Hw, blocks, g)

    rep = eng.step(BATCH, RNG_SEED, 0, train=True)
    assert rep["loss"] == fwd["loss"]
    got = eng.read(*[n for n in names if n.startswith(("grad.", "post.r", "att."))])
    if flips:
        pytest.skip(f"{flips} ReLU tie(s) flipped vs the f64 oracle; forward parity checked")
    for key, want in wg.items():
        r, l = key
        assert_close(got[f"grad.w.r{r}.l{l}"], want, TOL, f"RGAT grad.w.r{r}.l{l}")
        assert_close(got[f"grad.att.r{r}.l{l}"].ravel(), ag[key], TOL, f"RGAT grad.att.r{r}.l{l}")
    for t, (ids, rows) in fg.items():
        gids = eng.read(f"grad.f.t{t}.ids", f"grad.f.t{t}.rows")
        assert [int(x) for x in gids[f"grad.f.t{t}.ids"]] == ids
        assert_close(gids[f"grad.f.t{t}.rows"], rows, TOL, f"RGAT grad.f.t{t}")
    # one Adam step of the model (hgnn.cpp:364-390 semantics) from the oracle's gradients
    for key, want in wg.items():
        r, l = key
        for name, w0, gr in ((f"post.r{r}.l{l}", weights[key], want), (f"att.r{r}.l{l}", att[key], ag[key])):
            w, m, v = w0.copy(), np.zeros_like(w0), np.zeros_like(w0)
            port.adam_step(w, m, v, gr, 1)
            assert_adam_close(got[name].reshape(w.shape), w, None, steps=1, what=f"RGAT {name}")
    # learnable rows after their sparse Adam
    post = eng.read(*[f"post.learn.t{t}" for t in fg])
    for t, (ids, rows) in fg.items():
        w, m, v = learn[t][ids].copy(), np.zeros_like(rows), np.zeros_like(rows)
        port.adam_step(w, m, v, rows, 1)
        assert_adam_close(post[f"post.learn.t{t}"][ids], w, None, steps=1, what=f"RGAT learn t{t}")


@pytest.mark.gpu
def test_rgat_steps_are_bit_reproducible(H):
    gd = H.gen_synthetic(H.bundled_spec("mag-mini"), 5)
    batches = H.make_batches(gd, 128, 3, H.mix_seed(5, 0xBA7C))
    runs = []
    for _ in range(2):
        eng = H.Engine(gd, FANOUTS, hidden=HIDDEN, batch_cap=128, model_seed=77, learn_seed=88, model="rgat",
                       heads=HEADS)
        losses = [eng.step(b, H.mix_seed(5, 0xB000 + i))["loss"] for i, b in enumerate(batches)]
        # the same batch again and again: the loss falls
        losses += [eng.step(batches[0], 9)["loss"] for _ in range(6)]
        runs.append((losses, eng.read("post.r0.l1")["post.r0.l1"]))
    assert runs[0][0] == runs[1][0]
    assert np.array_equal(runs[0][1], runs[1][1])
    assert runs[0][0][-1] < runs[0][0][3]


@pytest.mark.gpu
def test_rgat_c2_step_matches_oracle(H, ref):
    """The C3 configuration itself: C2's graph and batch (1024, fanout [25,20]), hidden 64,
    4 heads; one training step against the f64 restatement on the reference's blocks."""
    spec = H.ogbn_mag_spec()
    rg = ref.RefGraph.from_spec(spec, 1)
    g = port.Graph(rg.export())
    tree = port.bfs_metatree(g, 2)
    gd = H.gen_synthetic(spec, 1)
    batch = [int(x) for x in H.make_batches(gd, 1024, 1, H.mix_seed(1, 0xBA7C))[0]]
    seed = H.mix_seed(1, 0xB000)
    blocks = blocks_from(rg.sample_khop(batch, [25, 20], seed, port.hop_relation_sets(tree, 2)), 2, g.ntypes,
                         g.nrels)
    eng = H.Engine.for_experiment(gd, [25, 20], 64, 1, batch_cap=1024, model="rgat", heads=4)
    names = eng.tensor_names()
    init = eng.read(*[n for n in names if n.startswith(("post.r", "att.", "post.learn.t"))])
    weights = {(int(n.split(".")[1][1:]), int(n.split(".")[2][1:])): init[n] for n in init if n.startswith("post.r")}
    att = {(int(n.split(".")[1][1:]), int(n.split(".")[2][1:])): init[n].ravel() for n in init if n.startswith("att.")}
    learn = {int(n.split(".t")[-1]): init[n] for n in init if n.startswith("post.learn.t")}
    loss, logits, Hw, dl, wg, ag, fg = R.step(g, tree, blocks, weights, att, learn, 64, 4, batch)
    rep = eng.step(batch, seed, 0, train=True)
    got = eng.read(*[n for n in names if n.startswith(("H1.", "logits", "grad."))])
    assert abs(rep["loss"] - loss) <= TOL * abs(loss)
    assert_close(got["logits"], logits, TOL, "C3 logits")
    for t in range(g.ntypes):
        if t in Hw[1]:
            assert_close(got[f"H1.t{t}"], Hw[1][t], TOL, f"C3 H1.t{t}")
    if _relu_flips(got, Hw, blocks, g):
        pytest.skip("ReLU tie flipped vs the f64 oracle; forward parity checked")
    for key, want in wg.items():
        r, l = key
        assert_close(got[f"grad.w.r{r}.l{l}"], want, TOL, f"C3 grad.w.r{r}.l{l}")
        assert_close(got[f"grad.att.r{r}.l{l}"].ravel(), ag[key], TOL, f"C3 grad.att.r{r}.l{l}")
    for t, (ids, rows) in fg.items():
        assert [int(x) for x in got[f"grad.f.t{t}.ids"]] == ids
        assert_close(got[f"grad.f.t{t}.rows"], rows, TOL, f"C3 grad.f.t{t}")


@pytest.mark.gpu
@pytest.mark.parametrize("p", [2, 4])
def test_rgat_multi_gpu_matches_one_gpu(H, p):
    """C3 at p GPUs (BASELINE configs[2] runs RGAT on 4): one meta-partition per GPU, AGG_all
    of the partial logits over NCCL; at p = 4 one sub-metatree is replicated (its replicas
    split the batch and merge weight, attention and learnable-row gradients). Every
    batch's loss and the trained model match the single-GPU RGAT engine."""
    import os
    import subprocess
    import sys
    import tempfile

    from tests.util import gpu_count
    if gpu_count() < p:
        pytest.skip(f"needs {p} GPUs")
    here = os.path.dirname(os.path.abspath(__file__))
    seed, n_batches, bsz = 5, 6, 64
    with tempfile.TemporaryDirectory() as td:
        idp = os.path.join(td, "nccl.id")
        procs = [subprocess.Popen([sys.executable, os.path.join(here, "mp", "raf_rank.py"), "mag-mini", str(seed), str(p),
                                   str(r), idp, os.path.join(td, f"r{r}.npz"), str(n_batches), str(bsz)],
                                  stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True,
                                  env=dict(os.environ, HG_MODEL="rgat")) for r in range(p)]
        outs = [pr.communicate(timeout=300)[0] for pr in procs]
        for pr, o in zip(procs, outs):
            assert pr.returncode == 0, o[-3000:]
        res = [np.load(os.path.join(td, f"r{r}.npz")) for r in range(p)]
    g = H.gen_synthetic(H.bundled_spec("mag-mini"), seed)
    batches = H.make_batches(g, bsz, n_batches, H.mix_seed(seed, 0xBA7C))
    one = H.Engine.for_experiment(g, [25, 20], 32, seed, batch_cap=bsz, model="rgat", heads=4)
    losses = [one.step(b, H.mix_seed(seed, 0xB000 + i))["loss"] for i, b in enumerate(batches)]
    want = one.read(*[n for n in one.tensor_names() if n.startswith(("post.r", "att."))])
    for r in range(p):
        np.testing.assert_allclose(res[r]["losses"], losses, rtol=1e-3, atol=0)
    seen = {}
    for r in range(p):
        for key in res[r].files:
            if not key.startswith("T:"):
                continue
            n, v = key[2:], res[r][key]
            if n in seen:
                assert np.array_equal(seen[n], v), f"replicas disagree on {n}"
            seen[n] = v
            if n in want:
                assert_adam_close(v, want[n], None, steps=n_batches, max_flip_frac=1e-2, what=f"p={p} rank {r}: {n}")
    assert any(n.startswith("att.") for n in seen)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f16", "bf16"])
def test_rgat_half_tables_match_oracle(H, ref, dtype):
    """Layer-1 attention reads fp16 / bf16 feature rows (k_att_leaf_*'s 8-byte loads): the
    reference's features rounded to that type make the same step as the f64 restatement."""
    rg = ref.RefGraph.bundled("mag-mini", 5)
    rg.round_features(dtype)
    g = port.Graph(rg.export())
    tree = port.bfs_metatree(g, 2)
    blocks = blocks_from(rg.sample_khop(BATCH, FANOUTS, RNG_SEED, port.hop_relation_sets(tree, 2)), 2, g.ntypes,
                         g.nrels)
    gd = H.gen_synthetic(H.bundled_spec("mag-mini"), 5)
    eng = H.Engine(gd, FANOUTS, hidden=HIDDEN, batch_cap=len(BATCH), model_seed=77, learn_seed=88, model="rgat",
                   heads=HEADS, feat_dtype=dtype)
    names = eng.tensor_names()
    init = eng.read(*[n for n in names if n.startswith(("post.r", "att.", "post.learn.t"))])
    weights = {(int(n.split(".")[1][1:]), int(n.split(".")[2][1:])): init[n] for n in init if n.startswith("post.r")}
    att = {(int(n.split(".")[1][1:]), int(n.split(".")[2][1:])): init[n].ravel() for n in init if n.startswith("att.")}
    learn = {int(n.split(".t")[-1]): init[n] for n in init if n.startswith("post.learn.t")}
    loss, logits, Hw, dl, wg, ag, fg = R.step(g, tree, blocks, weights, att, learn, HIDDEN, HEADS, BATCH)
    rep = eng.step(BATCH, RNG_SEED, 0, train=True)
    got = eng.read(*[n for n in names if n.startswith(("H1.", "logits", "grad.w.", "grad.att."))])
    assert abs(rep["loss"] - loss) <= TOL * abs(loss)
    assert_close(got["logits"], logits, TOL, f"RGAT {dtype} logits")
    for t in range(g.ntypes):
        if t in Hw[1]:
            assert_close(got[f"H1.t{t}"], Hw[1][t], TOL, f"RGAT {dtype} H1.t{t}")
    if _relu_flips(got, Hw, blocks, g):
        pytest.skip("ReLU tie flipped vs the f64 oracle; forward parity checked")
    for (r, l), want in wg.items():
        assert_close(got[f"grad.w.r{r}.l{l}"], want, TOL, f"RGAT {dtype} grad.w.r{r}.l{l}")
        assert_close(got[f"grad.att.r{r}.l{l}"].ravel(), ag[(r, l)], TOL, f"RGAT {dtype} grad.att.r{r}.l{l}")


@pytest.mark.gpu
@pytest.mark.parametrize("k,heads", [(3, 4), (2, 1), (2, 8)])
def test_rgat_depths_and_heads_match_oracle(H, ref, k, heads):
    """Three layers (two aggregate-first inner layers over the previous layer's rows) and
    the 1- and 8-head kernel instantiations against the f64 restatement."""
    fanouts = [6, 5, 4][:k]
    rg = ref.RefGraph.bundled("mag-mini", 5)
    g = port.Graph(rg.export())
    tree = port.bfs_metatree(g, k)
    batch = list(range(0, 256, 4))
    blocks = blocks_from(rg.sample_khop(batch, fanouts, RNG_SEED, port.hop_relation_sets(tree, k)), k, g.ntypes,
                         g.nrels)
    gd = H.gen_synthetic(H.bundled_spec("mag-mini"), 5)
    eng = H.Engine(gd, fanouts, hidden=HIDDEN, batch_cap=len(batch), model_seed=77, learn_seed=88, model="rgat",
                   heads=heads)
    names = eng.tensor_names()
    init = eng.read(*[n for n in names if n.startswith(("post.r", "att.", "post.learn.t"))])
    weights = {(int(n.split(".")[1][1:]), int(n.split(".")[2][1:])): init[n] for n in init if n.startswith("post.r")}
    att = {(int(n.split(".")[1][1:]), int(n.split(".")[2][1:])): init[n].ravel() for n in init if n.startswith("att.")}
    learn = {int(n.split(".t")[-1]): init[n] for n in init if n.startswith("post.learn.t")}
    loss, logits, Hw, dl, wg, ag, fg = R.step(g, tree, blocks, weights, att, learn, HIDDEN, heads, batch)
    rep = eng.step(batch, RNG_SEED, 0, train=True)
    got = eng.read(*[n for n in names if n.startswith(("H", "logits", "grad.w.", "grad.att."))])
    assert abs(rep["loss"] - loss) <= TOL * abs(loss)
    assert_close(got["logits"], logits, TOL, "logits")
    flips = 0
    for d in range(1, k):
        for t in range(g.ntypes):
            if t in Hw[d] and f"H{d}.t{t}" in got:
                assert_close(got[f"H{d}.t{t}"], Hw[d][t], TOL, f"H{d}.t{t}")
                flips += int(((got[f"H{d}.t{t}"] > 0) != (Hw[d][t] > 0)).sum())
    if flips:
        pytest.skip("ReLU tie flipped vs the f64 oracle; forward parity checked")
    for (r, l), want in wg.items():
        assert_close(got[f"grad.w.r{r}.l{l}"], want, TOL, f"grad.w.r{r}.l{l}")
        assert_close(got[f"grad.att.r{r}.l{l}"].ravel(), ag[(r, l)], TOL, f"grad.att.r{r}.l{l}")
