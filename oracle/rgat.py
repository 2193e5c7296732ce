"""TEST INFRASTRUCTURE ONLY — CPU restatement (numpy, f64) of the RGAT layer type.

The reference has no attention layer (BASELINE.md
configs[2] "no oracle"), so this module *defines* the framework's RGAT and is the
checker of the device path (paper_2408_09697_b200/csrc/rgat.cu, rgat_kernels.cu).
Parity is pinned by finite differences of this restatement
(tests/test_rgat.py::test_oracle_gradients_match_finite_differences), not by the
reference. Structure (metatree, blocks, relation order, ReLU, loss) follows the
reference's RGCN path restated in oracle/port.py (hgnn.cpp:215-362); only the
per-relation aggregation differs:

    z_j       = h_j W_r                                   (source rows of the block)
    t_j^h     = a_r^h . z_j^(h)                           (head h: columns [hF, (h+1)F))
    alpha_e^h = softmax over the edges e of dst i of LeakyReLU_0.2(t_src(e)^h)
    out_i     = sum_r concat_h sum_e alpha_e^h z_src(e)^(h)      (+ReLU below the top)

H heads below the top layer, one head at the top (F = d_out / H).
"""
from __future__ import annotations

from typing import Dict, Tuple

import numpy as np

from . import port

SLOPE = 0.2


def _lrelu(x):
    return np.where(x > 0, x, SLOPE * x)


def _segments(blk):
    ip = np.asarray(blk["indptr"], np.int64)
    n = len(ip) - 1
    return np.repeat(np.arange(n), np.diff(ip)), n


def attend(blk, h_src, src_front, w, a, heads):
    """One relation's block: returns (out [n_dst x d_out], cache for backward)."""
    seg, n = _segments(blk)
    col = np.searchsorted(np.asarray(src_front, np.int64), np.asarray(blk["src_ids"], np.int64))
    z = h_src @ w
    dout = w.shape[1]
    F = dout // heads
    hc = np.arange(dout) // F
    t = (z * a[None, :]).reshape(len(z), heads, F).sum(-1)
    x = _lrelu(t[col])  # [E, H]
    m = np.full((n, heads), -np.inf)
    np.maximum.at(m, seg, x)
    ex = np.exp(x - m[seg])
    s = np.zeros((n, heads))
    np.add.at(s, seg, ex)
    alpha = ex / s[seg]
    out = np.zeros((n, dout))
    np.add.at(out, seg, alpha[:, hc] * z[col])
    return out, dict(seg=seg, col=col, z=z, t=t, alpha=alpha, hc=hc, heads=heads, F=F)


def attend_backward(c, dout_rows, h_src, w, a):
    """Gradients of one relation's block given d out: (dW, da, dH_src)."""
    seg, col, z, t, alpha, hc = c["seg"], c["col"], c["z"], c["t"], c["alpha"], c["hc"]
    H, F = c["heads"], c["F"]
    g = dout_rows[seg]  # [E, d_out]
    dalpha = (g * z[col]).reshape(len(seg), H, F).sum(-1)
    csum = np.zeros((dout_rows.shape[0], H))
    np.add.at(csum, seg, alpha * dalpha)
    dt = alpha * (dalpha - csum[seg]) * np.where(t[col] > 0, 1.0, SLOPE)
    dz = np.zeros_like(z)
    np.add.at(dz, col, alpha[:, hc] * g)
    tsum = np.zeros((len(z), H))
    np.add.at(tsum, col, dt)
    dz += tsum[:, hc] * a[None, :]
    da = (tsum[:, hc] * z).sum(0)
    return h_src.T @ dz, da, dz @ w.T


def forward(g: port.Graph, tree, blocks: dict, weights: Dict[Tuple[int, int], np.ndarray],
            att: Dict[Tuple[int, int], np.ndarray], learn: Dict[int, np.ndarray], hidden: int, heads: int):
    """forward_flat (hgnn.cpp:215-279 structure) with attention per relation."""
    k = blocks["k"]
    H = [dict() for _ in range(k + 1)]
    for t in range(g.ntypes):
        front = blocks["frontier"][k][t]
        if not front:
            continue
        H[k][t] = g.dense[t][front] if g.kinds[t] == 1 else learn[t][front]
    tape = []
    for l in range(1, k + 1):
        d = k - l + 1
        rels = port.rels_by_dst_at_depth(tree, d)
        dout = g.num_classes if l == k else hidden
        nh = 1 if l == k else heads
        for t in range(g.ntypes):
            front = blocks["frontier"][d - 1][t]
            if not front:
                continue
            out = np.zeros((len(front), dout))
            for r in rels.get(t, []):
                blk = next((b for b in blocks["hops"][d - 1] if b["rel"] == r), None)
                if blk is None:
                    continue
                s = g.rel_src[r]
                if s not in H[d]:  # no sampled sources: a zero contribution
                    continue
                part, cache = attend(blk, H[d][s], blocks["frontier"][d][s], weights[(r, l)], att[(r, l)], nh)
                out += part
                tape.append(dict(layer=l, rel=r, depth=d, dst=t, src=s, cache=cache))
            if l < k:
                out = np.maximum(out, 0.0)
            H[d - 1][t] = out
    return H[0][g.target], H, tape


def backward(g: port.Graph, blocks, H, tape, weights, att, dlogits):
    """backward_flat (hgnn.cpp:309-362 structure): weight, attention and leaf-row gradients."""
    k = blocks["k"]
    dH = [dict() for _ in range(k + 1)]
    dH[0][g.target] = dlogits
    wgrads, agrads, fgrads = {}, {}, {}
    for l in range(k, 0, -1):
        d = k - l + 1
        for e in tape:
            if e["layer"] != l or e["dst"] not in dH[d - 1]:
                continue
            dpre = dH[d - 1][e["dst"]].copy()
            if l < k:
                dpre[H[d - 1][e["dst"]] <= 0.0] = 0.0
            key = (e["rel"], l)
            s = e["src"]
            dw, da, dh = attend_backward(e["cache"], dpre, H[d][s], weights[key], att[key])
            wgrads[key] = wgrads.get(key, 0.0) + dw
            agrads[key] = agrads.get(key, 0.0) + da
            dH[d][s] = dH[d].get(s, 0.0) + dh
    for t, m in dH[k].items():
        if g.kinds[t] == 2:
            fgrads[t] = (list(blocks["frontier"][k][t]), m)
    return wgrads, agrads, fgrads


def step(g: port.Graph, tree, blocks, weights, att, learn, hidden, heads, batch):
    """One flat step: (loss, logits, H, dlogits, wgrads, agrads, fgrads)."""
    logits, H, tape = forward(g, tree, blocks, weights, att, learn, hidden, heads)
    loss, dl = port.cross_entropy(logits, blocks["frontier"][0][g.target], batch, g.labels, g.num_classes)
    wg, ag, fg = backward(g, blocks, H, tape, weights, att, dl)
    return loss, logits, H, dl, wg, ag, fg
