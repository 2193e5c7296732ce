"""TEST INFRASTRUCTURE ONLY — a CPU restatement of the reference's hot path.

Pure Python / numpy restatement of the reference algorithms on the Heta
mini-batch path (reference: /root/reference/proj, file:line cited per
function). It is pinned by tests/test_oracle.py against the compiled reference
(oracle/_ref) and the committed golden fixtures (tests/golden/), and is only
ever used as a checker: tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline leg. Small cases only (the sampler is pure Python).

Third-party arithmetic restated here: libstdc++ 13's std::mt19937_64
(bits/random.tcc:328-466) and std::uniform_int_distribution<uint64_t>
(bits/uniform_int_dist.h:255-320, Lemire's nearly-divisionless method).
"""
from __future__ import annotations

from typing import Dict, List, Optional, Sequence

import numpy as np

M64 = (1 << 64) - 1


# ---- sampling.cpp:9-15 -------------------------------------------------------------------
def mix_seed(a: int, b: int) -> int:
    z = (a + 0x9E3779B97F4A7C15 * (b + 1)) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


class MT19937_64:
    """std::mt19937_64 (random.tcc:328-466)."""

    N, M = 312, 156
    UPPER, LOWER = 0xFFFFFFFF80000000, 0x7FFFFFFF

    def __init__(self, seed: int):
        x = [0] * self.N
        x[0] = seed & M64
        for i in range(1, self.N):
            x[i] = (6364136223846793005 * (x[i - 1] ^ (x[i - 1] >> 62)) + i) & M64
        self.x, self.p = x, self.N

    def _twist(self):
        x, n, m = self.x, self.N, self.M
        for k in range(n):
            y = (x[k] & self.UPPER) | (x[(k + 1) % n] & self.LOWER)
            x[k] = x[(k + m) % n] ^ (y >> 1) ^ (0xB5026F5AA96619E9 if y & 1 else 0)
        self.p = 0

    def __call__(self) -> int:
        if self.p >= self.N:
            self._twist()
        z = self.x[self.p]
        self.p += 1
        z ^= (z >> 29) & 0x5555555555555555
        z ^= (z << 17) & 0x71D67FFFEDA60000
        z ^= (z << 37) & 0xFFF7EEE000000000
        z ^= z >> 43
        return z & M64


def uniform_u64(eng: MT19937_64, lo: int, hi: int) -> int:
    """uniform_int_distribution<uint64_t>(lo, hi) (uniform_int_dist.h:255-320)."""
    rng = hi - lo + 1
    p = eng() * rng
    low = p & M64
    if low < rng:
        thr = ((1 << 64) - rng) % rng
        while low < thr:
            p = eng() * rng
            low = p & M64
    return lo + (p >> 64)


# ---- sampling.cpp:17-39 ------------------------------------------------------------------
def sample_neighbors(indptr, src, dst: int, fanout: int, rng_seed: int, hop: int, rel: int) -> List[int]:
    lo, hi = int(indptr[dst]), int(indptr[dst + 1])
    deg = hi - lo
    if deg <= fanout:
        return [int(x) for x in src[lo:hi]]
    eng = MT19937_64(mix_seed(rng_seed, mix_seed((hop << 32) | rel, dst)))
    idx = list(range(deg))
    out = []
    for i in range(fanout):
        j = uniform_u64(eng, i, deg - 1)
        idx[i], idx[j] = idx[j], idx[i]
        out.append(int(src[lo + idx[i]]))
    return out


# ---- graph view ----------------------------------------------------------------------------
class Graph:
    """Arrays of an exported HetGraph (hetgraph.hpp:58-74)."""

    def __init__(self, e: Dict[str, np.ndarray]):
        self.counts = [int(x) for x in e["node_counts"]]
        self.rel_src = [int(x) for x in e["rel_src"]]
        self.rel_dst = [int(x) for x in e["rel_dst"]]
        self.indptr = [np.asarray(e[f"rel{r}.indptr"], np.int64) for r in range(len(self.rel_src))]
        self.src = [np.asarray(e[f"rel{r}.src"], np.int64) for r in range(len(self.rel_src))]
        self.kinds = [int(x) for x in e["kinds"]]
        self.dims = [int(x) for x in e["dims"]]
        self.dense = {t: np.asarray(e[f"feat.t{t}"], np.float64) for t in range(len(self.counts)) if self.kinds[t] == 1}
        self.target = int(np.asarray(e["target"]).ravel()[0])
        self.num_classes = int(np.asarray(e["num_classes"]).ravel()[0])
        self.labels = np.asarray(e["labels"], np.int64)

    @property
    def ntypes(self):
        return len(self.counts)

    @property
    def nrels(self):
        return len(self.rel_src)


# ---- sampling.cpp:41-103 -------------------------------------------------------------------
def sample_khop(g: Graph, seeds: Sequence[int], fanouts: Sequence[int], rng_seed: int,
                hop_relations: Optional[Sequence[Sequence[int]]] = None) -> dict:
    if not fanouts:
        raise ValueError("fanouts must be non-empty")
    for s in seeds:
        if s >= g.counts[g.target]:
            raise ValueError(f"seed node id out of range: {s}")
    k = len(fanouts)
    frontier = [[[] for _ in range(g.ntypes)] for _ in range(k + 1)]
    frontier[0][g.target] = sorted(set(int(s) for s in seeds))
    hops = []
    for hop in range(1, k + 1):
        nxt = [[] for _ in range(g.ntypes)]
        blocks = []
        for r in range(g.nrels):
            if hop_relations is not None and r not in hop_relations[hop - 1]:
                continue
            front = frontier[hop - 1][g.rel_dst[r]]
            if not front:
                continue
            indptr, src_ids = [0], []
            for d in front:
                src_ids += sample_neighbors(g.indptr[r], g.src[r], d, fanouts[hop - 1], rng_seed, hop, r)
                indptr.append(len(src_ids))
            nxt[g.rel_src[r]] += src_ids
            blocks.append(dict(rel=r, dst_ids=list(front), indptr=indptr, src_ids=src_ids))
        for t in range(g.ntypes):
            frontier[hop][t] = sorted(set(nxt[t]))
        hops.append(blocks)
    return dict(k=k, hops=hops, frontier=frontier)


# ---- metapartition.cpp:32-53, hgnn.cpp:16-37 -----------------------------------------------
def bfs_metatree(g: Graph, k: int):
    """build_metatree BFS mode: positions (type, depth, parent, rel)."""
    pos = [(g.target, 0, -1, -1)]
    begin = 0
    for depth in range(1, k + 1):
        end = len(pos)
        for p in range(begin, end):
            for r in range(g.nrels):
                if g.rel_dst[r] == pos[p][0]:
                    pos.append((g.rel_src[r], depth, p, r))
        begin = end
    return pos


def hop_relation_sets(tree, k):
    out = [[] for _ in range(k)]
    for (_, depth, _, r) in tree:
        if r >= 0 and 1 <= depth <= k and r not in out[depth - 1]:
            out[depth - 1].append(r)
    return [sorted(v) for v in out]


def rels_by_dst_at_depth(tree, depth):
    out = {}
    for (_, d, parent, r) in tree:
        if d != depth or r < 0:
            continue
        v = out.setdefault(tree[parent][0], [])
        if r not in v:
            v.append(r)
    return {t: sorted(v) for t, v in out.items()}


# ---- hgnn.cpp:173-362: flat forward / loss / backward -----------------------------------------
def mean_aggregate(block, h_src: np.ndarray, src_front: Sequence[int]) -> np.ndarray:
    row = {v: i for i, v in enumerate(src_front)}
    out = np.zeros((len(block["dst_ids"]), h_src.shape[1]))
    ip = block["indptr"]
    for i in range(len(block["dst_ids"])):
        lo, hi = ip[i], ip[i + 1]
        if lo == hi:
            continue
        for e in range(lo, hi):
            out[i] += h_src[row[block["src_ids"][e]]]
        out[i] *= 1.0 / (hi - lo)
    return out


def forward_flat(g: Graph, tree, blocks: dict, weights: Dict[tuple, np.ndarray], learn: Dict[int, np.ndarray],
                 hidden: int):
    k = blocks["k"]
    H = [dict() for _ in range(k + 1)]
    for t in range(g.ntypes):
        front = blocks["frontier"][k][t]
        if not front:
            continue
        if g.kinds[t] == 1:
            H[k][t] = g.dense[t][front]
        elif g.kinds[t] == 2:
            H[k][t] = learn[t][front]
        else:
            raise RuntimeError(f"missing features for node type {t}")
    tape = []
    for l in range(1, k + 1):
        d = k - l + 1
        rels = rels_by_dst_at_depth(tree, d)
        dout = g.num_classes if l == k else hidden
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
                if s in H[d]:
                    mean = mean_aggregate(blk, H[d][s], blocks["frontier"][d][s])
                else:
                    mean = np.zeros((len(blk["dst_ids"]), g.dims[s] if l == 1 else hidden))
                out += mean @ weights[(r, l)]
                tape.append(dict(layer=l, rel=r, depth=d, dst=t, block=blk, mean=mean))
            if l < k:
                out = np.maximum(out, 0.0)
            H[d - 1][t] = out
    return H[0][g.target], H, tape


def cross_entropy(logits: np.ndarray, row_ids: Sequence[int], batch: Sequence[int], labels, num_classes: int):
    if len(batch) == 0:
        raise ValueError("empty batch")
    row = {v: i for i, v in enumerate(row_ids)}
    dz = np.zeros_like(logits)
    loss = 0.0
    invb = 1.0 / len(batch)
    for v in batch:
        y = int(labels[v])
        if y < 0 or y >= num_classes:
            raise ValueError(f"label out of range for node {v}")
        z = logits[row[v]]
        zmax = z.max()
        lse = zmax + np.log(np.exp(z - zmax).sum())
        loss += (lse - z[y]) * invb
        p = np.exp(z - lse)
        p[y] -= 1.0
        dz[row[v]] += p * invb
    return loss, dz


def backward_flat(g: Graph, tree, blocks, H, tape, weights, dlogits):
    k = blocks["k"]
    dH = [dict() for _ in range(k + 1)]
    dH[0][g.target] = dlogits
    wgrads, fgrads = {}, {}
    for l in range(k, 0, -1):
        d = k - l + 1
        for e in tape:
            if e["layer"] != l or e["dst"] not in dH[d - 1]:
                continue
            dpre = dH[d - 1][e["dst"]].copy()
            if l < k:
                dpre[H[d - 1][e["dst"]] <= 0.0] = 0.0
            w = weights[(e["rel"], l)]
            wgrads[(e["rel"], l)] = wgrads.get((e["rel"], l), np.zeros_like(w)) + e["mean"].T @ dpre
            dmean = dpre @ w.T
            s = g.rel_src[e["rel"]]
            front = blocks["frontier"][d][s]
            if s not in dH[d]:
                dH[d][s] = np.zeros((len(front), dmean.shape[1]))
            row = {v: i for i, v in enumerate(front)}
            blk = e["block"]
            ip = blk["indptr"]
            for i in range(len(blk["dst_ids"])):
                lo, hi = ip[i], ip[i + 1]
                if lo == hi:
                    continue
                for x in range(lo, hi):
                    dH[d][s][row[blk["src_ids"][x]]] += dmean[i] / (hi - lo)
    for t, m in dH[k].items():
        if g.kinds[t] == 2:
            fgrads[t] = (list(blocks["frontier"][k][t]), m)
    return wgrads, fgrads


# ---- hgnn.cpp:364-410 --------------------------------------------------------------------------
def adam_step(w, m, v, grad, t, lr=1e-2, b1=0.9, b2=0.999, eps=1e-8):
    if not np.all(np.isfinite(grad)):
        raise RuntimeError("non-finite gradient")
    m[:] = b1 * m + (1 - b1) * grad
    v[:] = b2 * v + (1 - b2) * grad * grad
    bc1, bc2 = 1 - b1 ** t, 1 - b2 ** t
    w -= lr * (m / bc1) / (np.sqrt(v / bc2) + eps)


# ---- cache.cpp:11-141 ----------------------------------------------------------------------------
def presample_hotness(g: Graph, tree, fanouts, epochs: int, seed: int, batch_size: int = 512):
    counts = [np.zeros(c, np.int64) for c in g.counts]
    hop_rels = hop_relation_sets(tree, len(fanouts))
    n = g.counts[g.target]
    for e in range(epochs):
        for lo in range(0, n, batch_size):
            batch = list(range(lo, min(lo + batch_size, n)))
            b = sample_khop(g, batch, fanouts, mix_seed(seed, e), hop_rels)
            for v in batch:
                counts[g.target][v] += 1
            for hop in b["hops"]:
                for blk in hop:
                    for s in blk["src_ids"]:
                        counts[g.rel_src[blk["rel"]]][s] += 1
    return counts


def profile_miss_penalty(g: Graph, read_ns=1.0, write_ns=1.0, overhead_ns=1000.0, elem_bytes=4):
    out = []
    for t in range(g.ntypes):
        if g.kinds[t] == 0:
            out.append(dict(learnable=False, record_bytes=0, transfer_ns=0.0, ratio=0.0))
            continue
        row = g.dims[t] * elem_bytes
        if row == 0:
            raise ValueError(f"zero record size for node type {t}")
        if g.kinds[t] == 2:
            rb, tns = 3 * row, 3.0 * (overhead_ns + read_ns * row) + 3.0 * (overhead_ns + write_ns * row)
        else:
            rb, tns = row, overhead_ns + read_ns * row
        out.append(dict(learnable=g.kinds[t] == 2, record_bytes=rb, transfer_ns=tns, ratio=tns / rb))
    return out


def allocate_cache(budget: int, counts, prof):
    denom = 0.0
    mass = []
    for t, p in enumerate(prof):
        m = float(int(np.sum(counts[t]))) * p["ratio"] if p["record_bytes"] > 0 else 0.0
        mass.append(m)
        denom += m
    if denom <= 0.0:
        raise ValueError("nothing to cache: all count*ratio products are zero")
    cap, nbytes = [], []
    for t, p in enumerate(prof):
        if p["record_bytes"] == 0:
            cap.append(0)
            nbytes.append(0)
            continue
        share = float(budget) * mass[t] / denom
        c = int(share) // p["record_bytes"]
        cap.append(c)
        nbytes.append(c * p["record_bytes"])
    return cap, nbytes


def fill_and_serve(capacity, counts):
    out = []
    for t, cap in enumerate(capacity):
        if cap == 0:
            out.append(np.zeros(0, np.int64))
            continue
        c = np.asarray(counts[t], np.int64)
        order = np.lexsort((np.arange(len(c)), -c))  # count desc, id asc
        out.append(np.sort(order[:cap]))
    return out


def cache_lookups(frontier_ids: Sequence[int], cached: np.ndarray, learnable: bool, transfer_ns: float,
                  state: Optional[dict] = None) -> dict:
    """CacheState::lookup / update (cache.cpp:87-113) over one frontier."""
    st = state or dict(hits=0, misses=0, penalty_ns=0.0)
    cached_set = set(int(x) for x in cached)
    for v in frontier_ids:
        for _ in range(2 if learnable else 1):
            if int(v) in cached_set:
                st["hits"] += 1
            else:
                st["misses"] += 1
                st["penalty_ns"] += transfer_ns
    return st
