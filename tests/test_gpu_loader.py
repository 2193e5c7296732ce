"""Streaming HGC1 loader (reference container.cpp:92-154): an engine
built straight from a container file (pairs and feature rows through pinned buffers
into the device CSR and tables) trains bit-identically to an engine built from the
host graph of the same file — for f32 / f16 feature tables and host-resident tables,
the reference's own container bytes included — and malformed files fail loudly."""
import numpy as np
import pytest

from paper_2408_09697_b200._native import HetGpuError

pytestmark = pytest.mark.gpu


def _steps(eng, H, g, n=3, bsz=128):
    batches = H.make_batches(g, bsz, n, H.mix_seed(5, 0xBA7C))
    losses = [eng.step(b, H.mix_seed(5, 0xB000 + i))["loss"] for i, b in enumerate(batches)]
    names = [x for x in eng.tensor_names() if x.startswith(("logits", "grad.", "post.r", "H"))]
    return losses, eng.read(*names)


@pytest.mark.parametrize("name,dtype,host", [("mag-mini", "f32", False), ("mag-mini", "f16", False),
                                             ("mag-mini", "bf16", True), ("igb-mini", "f32", False)])
def test_streamed_engine_equals_host_graph_engine(H, tmp_path, name, dtype, host):
    g = H.gen_synthetic(H.bundled_spec(name), 5)
    path = str(tmp_path / "g.hgc")
    H.save_container(g, path)
    kw = dict(batch_cap=128, model_seed=7, learn_seed=8, feat_dtype=dtype, feat_host=host)
    a = H.Engine(H.load_container(path), [25, 20], 32, **kw)
    b = H.Engine.from_container(path, [25, 20], 32, **kw)
    la, ta = _steps(a, H, g)
    lb, tb = _steps(b, H, g)
    assert la == lb
    assert set(ta) == set(tb)
    for k in ta:
        assert np.array_equal(ta[k], tb[k]), k


def test_streamed_engine_reads_reference_container(H, ref, tmp_path):
    rg = ref.RefGraph.bundled("mag-mini", 3)
    path = str(tmp_path / "ref.hgc")
    rg.save(path)  # the reference's own writer
    g = H.load_container(path)
    a = H.Engine(g, [25, 20], 32, batch_cap=128, model_seed=1, learn_seed=2)
    b = H.Engine.from_container(path, [25, 20], 32, batch_cap=128, model_seed=1, learn_seed=2)
    assert _steps(a, H, g)[0] == _steps(b, H, g)[0]


def test_streamed_rgat_engine(H, tmp_path):
    g = H.gen_synthetic(H.bundled_spec("mag-mini"), 5)
    path = str(tmp_path / "g.hgc")
    H.save_container(g, path)
    kw = dict(batch_cap=128, model_seed=7, learn_seed=8, model="rgat", heads=4)
    assert _steps(H.Engine(g, [25, 20], 32, **kw), H, g)[0] == _steps(H.Engine.from_container(path, [25, 20], 32, **kw), H, g)[0]


def test_malformed_containers_fail(H, tmp_path):
    g = H.gen_synthetic(H.bundled_spec("mag-mini"), 5)
    path = str(tmp_path / "g.hgc")
    H.save_container(g, path)
    raw = bytearray(open(path, "rb").read())
    hlen = int.from_bytes(raw[4:8], "little")
    first_pair = 8 + hlen
    # truncated body
    bad = str(tmp_path / "trunc.hgc")
    open(bad, "wb").write(bytes(raw[: first_pair + 100]))
    with pytest.raises(HetGpuError, match="truncated"):
        H.Engine.from_container(bad, [25, 20], 32, batch_cap=64)
    # an endpoint out of range (src of the first pair)
    oob = bytearray(raw)
    oob[first_pair:first_pair + 4] = (0xFFFFFFF0).to_bytes(4, "little")
    bad = str(tmp_path / "oob.hgc")
    open(bad, "wb").write(bytes(oob))
    with pytest.raises(ValueError, match="out of range in relation 0"):
        H.Engine.from_container(bad, [25, 20], 32, batch_cap=64)
    # destinations not ascending: swap the dst of the first pair with a large one
    order = bytearray(raw)
    order[first_pair + 4:first_pair + 8] = (50).to_bytes(4, "little")
    bad = str(tmp_path / "order.hgc")
    open(bad, "wb").write(bytes(order))
    with pytest.raises(HetGpuError, match="dst-major"):
        H.Engine.from_container(bad, [25, 20], 32, batch_cap=64)
