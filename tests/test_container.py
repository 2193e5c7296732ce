"""HGC1 container (reference container.cpp:47-154, tests
test_container.cpp:62-70 "bit-exact round trip"): our writer produces the
reference's exact bytes, each side loads the other's file, and malformed files
fail with the reference's runtime_error messages. Host code only (CPU)."""
import os

import numpy as np
import pytest

from paper_2408_09697_b200._native import HetGpuError


def _same_export(a, b):
    keys = set(a) & set(b)
    assert {"node_counts", "labels", "rel_src", "rel_dst", "kinds", "dims"} <= keys
    assert any(k.startswith("rel0.") for k in keys)
    for k in keys:
        x, y = np.asarray(a[k]), np.asarray(b[k])
        # HGC1 stores features as f32 (the reference keeps its generated f64 in memory)
        dt = np.float32 if k.startswith("feat.") else np.float64
        assert x.shape == y.shape and np.array_equal(x.astype(dt), y.astype(dt)), k


@pytest.mark.parametrize("name,seed", [("mag-mini", 3), ("donor-mini", 1), ("freebase-mini", 2)])
def test_container_bytes_and_round_trip(H, ref, tmp_path, name, seed):
    g = H.gen_synthetic(H.bundled_spec(name), seed)
    rg = ref.RefGraph.bundled(name, seed)
    ours, theirs = str(tmp_path / "ours.hgc"), str(tmp_path / "ref.hgc")
    H.save_container(g, ours)
    rg.save(theirs)
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    _same_export(H.load_container(theirs).export(), rg.export())
    _same_export(ref.RefGraph.load(ours).export(), g.export())


def test_container_random_graph_with_learnable_and_absent(H, ref, tmp_path):
    rg = ref.RefGraph.random(17)
    theirs = str(tmp_path / "ref.hgc")
    rg.save(theirs)
    g = H.load_container(theirs)
    ours = str(tmp_path / "ours.hgc")
    H.save_container(g, ours)
    assert open(ours, "rb").read() == open(theirs, "rb").read()


def test_container_errors(H, tmp_path):
    bad = tmp_path / "bad.hgc"
    bad.write_bytes(b"XXXX\x00\x00\x00\x00")
    with pytest.raises(HetGpuError, match="bad container magic"):
        H.load_container(str(bad))
    g = H.gen_synthetic(H.bundled_spec("mag-mini"), 3)
    good = str(tmp_path / "good.hgc")
    H.save_container(g, good)
    cut = tmp_path / "cut.hgc"
    cut.write_bytes(open(good, "rb").read()[: os.path.getsize(good) // 2])
    with pytest.raises(HetGpuError, match="truncated"):
        H.load_container(str(cut))
    with pytest.raises(HetGpuError, match="cannot open"):
        H.load_container(str(tmp_path / "missing.hgc"))
