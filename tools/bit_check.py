"""Bit-identity of two builds of the library (A/B variants that must not change any
result): run once per build (HETGPU_LIB=... selects a variant; each run writes an npz of
two steps' logits, gradients and layer outputs on eight graphs: f32 / f16 / bf16 tables,
C2, C4 and C5 shapes), then compare.
    HETGPU_LIB=... python tools/bit_check.py OUT.npz  /  python tools/bit_check.py --cmp A B"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(out):
    from paper_2408_09697_b200 import hetsim as H
    res = {}
    cases = [("mag-mini", "f32", H.bundled_spec("mag-mini"), [25, 20]), ("mag-mini-f16", "f16", H.bundled_spec("mag-mini"), [25, 20]),
             ("mag-mini-bf16", "bf16", H.bundled_spec("mag-mini"), [25, 20]), ("igb-mini", "f32", H.bundled_spec("igb-mini"), [25, 20]),
             ("c2", "f32", H.ogbn_mag_spec(), [25, 20]), ("c5", "f16", H.igb_het_spec(0.01), [25, 20]),
             ("c5f32", "f32", H.igb_het_spec(0.002), [25, 20]), ("c4", "f16", H.mag240m_spec(0.002), [25, 15, 10])]
    for name, dt, spec, fan in cases:
        g = H.gen_synthetic(spec, 3)
        eng = H.Engine(g, fan, 64, batch_cap=1024, model_seed=1, learn_seed=2, feat_dtype=dt)
        batches = H.make_batches(g, 1024, 2, H.mix_seed(3, 0xBA7C))
        for i, b in enumerate(batches):
            res[f"{name}.loss{i}"] = np.array([eng.step(b, H.mix_seed(3, 0xB000 + i))["loss"]])
        names = [x for x in eng.tensor_names() if x.startswith(("logits", "grad.", "post.r", "H", "mean"))]
        for k, v in eng.read(*names).items():
            res[f"{name}.{k}"] = v
        print(name, "ok", flush=True)
    np.savez(out, **res)


def cmp(a, b):
    A, B = np.load(a), np.load(b)
    assert set(A.files) == set(B.files), set(A.files) ^ set(B.files)
    bad = [k for k in A.files if not np.array_equal(A[k], B[k])]
    print(len(A.files), "tensors;", "identical" if not bad else f"DIFFER: {bad[:20]}")
    return 1 if bad else 0


if __name__ == "__main__":
    if sys.argv[1] == "--cmp":
        sys.exit(cmp(sys.argv[2], sys.argv[3]))
    run(sys.argv[1])
