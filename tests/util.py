"""Shared helpers for the parity tests (product vs oracle)."""
from __future__ import annotations

import numpy as np


def rel_err(ours: np.ndarray, ref: np.ndarray, floor: float = 1e-6) -> float:
    """max|ours - ref| / max(max|ref|, floor): the per-tensor relative error the
    north_star's "within 1e-3 relative" is measured with."""
    ours = np.asarray(ours, np.float64)
    ref = np.asarray(ref, np.float64)
    assert ours.shape == ref.shape, (ours.shape, ref.shape)
    if ref.size == 0:
        return 0.0
    return float(np.max(np.abs(ours - ref)) / max(float(np.max(np.abs(ref))), floor))


def assert_close(ours, ref, tol=1e-3, what=""):
    e = rel_err(ours, ref)
    assert e <= tol, f"{what}: relative error {e:.3e} > {tol:.1e}"


def assert_adam_close(w_ours, w_ref, w_before, lr=1e-2, tol=1e-3, max_flip_frac=2e-3, steps=1, what=""):
    """Post-Adam parameters after `steps` Adam updates. An element whose gradient
    is at fp32 rounding level may get the opposite sign of Adam's step, which moves
    it by lr*|m_hat|/sqrt(v_hat) <= ~lr per step (hgnn.cpp:364-377); a flipped
    element may therefore differ by at most 2*lr per step taken. At most
    `max_flip_frac` of the tensor may be outside the relative tolerance."""
    w_ours = np.asarray(w_ours, np.float64)
    w_ref = np.asarray(w_ref, np.float64)
    d = np.abs(w_ours - w_ref)
    scale = max(float(np.max(np.abs(w_ref))), 1e-6)
    bad = d > tol * scale
    frac = float(bad.mean()) if bad.size else 0.0
    assert frac <= max_flip_frac, f"{what}: {bad.sum()} of {bad.size} elements differ (max {d.max():.3e})"
    # the tensor as a whole stays within the relative tolerance (Frobenius norm)
    fro = float(np.linalg.norm(w_ours - w_ref) / max(np.linalg.norm(w_ref), 1e-30))
    assert fro <= tol, f"{what}: relative Frobenius error {fro:.3e} > {tol:.1e}"
    if bad.any():
        bound = 2 * lr * steps * 1.01
        assert float(d[bad].max()) <= bound, f"{what}: a flip of {d[bad].max():.3e} > {bound:.3e} ({steps} steps)"


def csr_from_pairs(n_dst, pairs):
    """dst-major CSR keeping insertion order (hetgraph.cpp:126-156)."""
    indptr = np.zeros(n_dst + 1, np.uint64)
    for _, d in pairs:
        indptr[d + 1] += 1
    indptr = np.cumsum(indptr).astype(np.uint64)
    fill = indptr[:-1].copy()
    src = np.zeros(len(pairs), np.uint32)
    for s, d in pairs:
        src[fill[d]] = s
        fill[d] += 1
    return indptr, src


def single_relation_graph(H, deg_list, n_src=None, dim=4, seed=0):
    """Target type 0 with len(deg_list) nodes; relation 0 from type 1 into it with
    the given in-degrees (sources 0..deg-1 in order, shifted per row)."""
    n_dst = len(deg_list)
    n_src = n_src or max(1, max(deg_list))
    pairs = []
    for d, deg in enumerate(deg_list):
        for j in range(deg):
            pairs.append(((j + d) % n_src, d))
    indptr, src = csr_from_pairs(n_dst, pairs)
    rng = np.random.default_rng(seed)
    e = {
        "node_counts": np.array([n_dst, n_src], np.uint64),
        "rel_src": np.array([1], np.int32), "rel_dst": np.array([0], np.int32),
        "rel_reverse": np.array([0], np.int32),
        "rel0.indptr": indptr, "rel0.src": src,
        "kinds": np.array([1, 1], np.int32), "dims": np.array([dim, dim], np.int32),
        "feat.t0": rng.uniform(-1, 1, (n_dst, dim)).astype(np.float32),
        "feat.t1": rng.uniform(-1, 1, (n_src, dim)).astype(np.float32),
        "labels": np.zeros(n_dst, np.int32), "target": np.array([0]), "num_classes": np.array([2]),
    }
    return e


def gpu_count() -> int:
    """Visible GPUs, without importing torch (torch's bundled NCCL clashes with the system
    libnccl that libhetgpu.so links once the product library is loaded)."""
    import subprocess
    try:
        out = subprocess.run(["nvidia-smi", "-L"], capture_output=True, text=True, timeout=60).stdout
    except Exception:
        return 0
    return sum(1 for line in out.splitlines() if line.startswith("GPU "))
