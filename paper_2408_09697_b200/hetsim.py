"""Python mirror of the reference's interface for the mini-batch hot path.

Same names, argument meaning and error behaviour as the reference's C++ API
(/root/reference/proj/include/hetsim/*.hpp), so the parity tests read like the
reference's own tests. Everything runs through the C-ABI in include/hetgpu.h;
the heavy lifting is C++ (host) and sm_100a CUDA (device). ValueError mirrors
std::invalid_argument, HetGpuError mirrors std::runtime_error.
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import _native as N
from ._native import HetGpuError  # noqa: F401  (re-export)

# ---- bundled synthetic specs (harness.cpp:192-247) and the benchmark shapes --------------


def bundled_spec(name: str) -> dict:
    """bundled_spec (src/harness.cpp:192-247)."""
    if name == "mag-mini":
        return dict(name=name, target="paper", num_classes=8, label_noise=0.1,
                    node_types=[dict(name="paper", count=8000, dim=128, storage="dense"),
                                dict(name="author", count=6000, dim=64, storage="learnable"),
                                dict(name="institution", count=500, dim=64, storage="learnable"),
                                dict(name="field", count=1000, dim=64, storage="learnable")],
                    relations=[dict(src="author", edge="writes", dst="paper", edges=30000, degree="powerlaw", alpha=1.6),
                               dict(src="author", edge="affiliated", dst="institution", edges=6000),
                               dict(src="paper", edge="cites", dst="paper", edges=40000, degree="powerlaw", alpha=1.8),
                               dict(src="paper", edge="has_topic", dst="field", edges=24000)],
                    self_paired=["cites"])
    if name == "freebase-mini":
        return dict(name=name, target="book", num_classes=8, label_noise=0.05,
                    node_types=[dict(name="book", count=5000, dim=32, storage="learnable"),
                                dict(name="film", count=4000, dim=32, storage="learnable"),
                                dict(name="music", count=8000, dim=32, storage="learnable"),
                                dict(name="people", count=6000, dim=32, storage="learnable")],
                    relations=[dict(src="people", edge="authored", dst="book", edges=20000, degree="powerlaw", alpha=1.7),
                               dict(src="film", edge="adapted", dst="book", edges=8000),
                               dict(src="music", edge="scored", dst="film", edges=10000),
                               dict(src="people", edge="liked", dst="music", edges=15000, degree="powerlaw", alpha=2.0)])
    if name == "donor-mini":
        return dict(name=name, target="project", num_classes=2, label_noise=0.05,
                    node_types=[dict(name="project", count=2000, dim=789, storage="dense"),
                                dict(name="donation", count=3000, dim=17, storage="dense"),
                                dict(name="donor", count=3000, dim=7, storage="dense")],
                    relations=[dict(src="donor", edge="gave", dst="project", edges=8000, degree="powerlaw", alpha=2.0),
                               dict(src="donor", edge="made", dst="donation", edges=6000),
                               dict(src="donation", edge="to_project", dst="project", edges=6000)])
    if name == "igb-mini":
        return dict(name=name, target="paper", num_classes=16, label_noise=0.1,
                    node_types=[dict(name="paper", count=10000, dim=128, storage="dense"),
                                dict(name="author", count=8000, dim=128, storage="dense"),
                                dict(name="institute", count=400, dim=128, storage="dense"),
                                dict(name="fos", count=700, dim=128, storage="dense")],
                    relations=[dict(src="author", edge="written", dst="paper", edges=30000, degree="powerlaw", alpha=1.6),
                               dict(src="author", edge="affiliated", dst="institute", edges=8000),
                               dict(src="paper", edge="cites", dst="paper", edges=30000, degree="powerlaw", alpha=1.8),
                               dict(src="paper", edge="topic", dst="fos", edges=20000)],
                    self_paired=["cites"])
    raise ValueError("unknown bundled spec: " + name)


def bundled_spec_names() -> List[str]:
    return ["mag-mini", "freebase-mini", "donor-mini", "igb-mini"]


def toy_spec() -> dict:
    """BASELINE.json configs[0] / SURVEY §8(d) C1: 4 types x 128-d, 5 uniform relations."""
    return dict(name="toy", target="paper", num_classes=8, label_noise=0.0, add_reverse=False,
                node_types=[dict(name="paper", count=40000, dim=128, storage="dense"),
                            dict(name="author", count=35000, dim=128, storage="dense"),
                            dict(name="institution", count=5000, dim=128, storage="dense"),
                            dict(name="field", count=20000, dim=128, storage="dense")],
                relations=[dict(src="author", edge="writes", dst="paper", edges=400000),
                           dict(src="paper", edge="rev_writes", dst="author", edges=400000),
                           dict(src="institution", edge="affiliated", dst="author", edges=35000),
                           dict(src="paper", edge="cites", dst="paper", edges=400000),
                           dict(src="field", edge="topic", dst="paper", edges=300000)])


def ogbn_mag_spec() -> dict:
    """BASELINE.json configs[1] / SURVEY §8(d) C2: ogbn-mag shape, uniform degrees."""
    return dict(name="ogbn-mag-shape", target="paper", num_classes=349, label_noise=0.1,
                node_types=[dict(name="paper", count=736389, dim=128, storage="dense"),
                            dict(name="author", count=1134649, dim=64, storage="learnable"),
                            dict(name="institution", count=8740, dim=64, storage="learnable"),
                            dict(name="field", count=59965, dim=64, storage="learnable")],
                relations=[dict(src="author", edge="writes", dst="paper", edges=7145660),
                           dict(src="author", edge="affiliated", dst="institution", edges=1043998),
                           dict(src="paper", edge="cites", dst="paper", edges=5416271),
                           dict(src="paper", edge="has_topic", dst="field", edges=7505078)],
                self_paired=["cites"])


def mag240m_spec(scale: float = 1.0) -> dict:
    """BASELINE.json configs[3] / SURVEY §8(d) C4: MAG240M shape (paper 121,751,666 with
    768-d features, author 122,383,112 and institution 25,721 learnable 64-d; writes 386.0M,
    affiliated 44.6M, cites 1,297.7M edges; 153 classes), uniform degrees, every count
    multiplied by `scale` (the full size exceeds one B200 and this host's memory)."""
    def n(x):
        return max(1, int(round(x * scale)))
    return dict(name=f"mag240m-shape-x{scale:g}", target="paper", num_classes=153, label_noise=0.1,
                node_types=[dict(name="paper", count=n(121751666), dim=768, storage="dense"),
                            dict(name="author", count=n(122383112), dim=64, storage="learnable"),
                            dict(name="institution", count=n(25721), dim=64, storage="learnable")],
                relations=[dict(src="author", edge="writes", dst="paper", edges=n(386000000)),
                           dict(src="author", edge="affiliated", dst="institution", edges=n(44600000)),
                           dict(src="paper", edge="cites", dst="paper", edges=n(1297700000))],
                self_paired=["cites"])


def igb_het_spec(scale: float = 1.0) -> dict:
    """BASELINE.json configs[4] / SURVEY §8 C5: IGB-HET shape (4 types,
    2.6e7 nodes, 4.9e8 edges with reverses, 7 edge types, 1024-d features on every type),
    split as IGB-HET medium's public statistics (paper 10.0M, author 15.5M, institute 23K,
    fos 415K; cites 120M, written 40M, affiliated 7.5M, topic 128M forward edges), uniform
    degrees, 19 classes, every count multiplied by `scale`."""
    def n(x):
        return max(1, int(round(x * scale)))
    return dict(name=f"igb-het-shape-x{scale:g}", target="paper", num_classes=19, label_noise=0.1,
                node_types=[dict(name="paper", count=n(10000000), dim=1024, storage="dense"),
                            dict(name="author", count=n(15544654), dim=1024, storage="dense"),
                            dict(name="institute", count=n(23256), dim=1024, storage="dense"),
                            dict(name="fos", count=n(415054), dim=1024, storage="dense")],
                relations=[dict(src="paper", edge="cites", dst="paper", edges=n(120077694)),
                           dict(src="author", edge="written", dst="paper", edges=n(39854592)),
                           dict(src="author", edge="affiliated", dst="institute", edges=n(7501203)),
                           dict(src="fos", edge="topic", dst="paper", edges=n(127565080))],
                self_paired=["cites"])


def mix_seed(a: int, b: int) -> int:
    """mix_seed (src/sampling.cpp:9-15)."""
    return int(N.lib().hg_mix_seed(a, b))


def mt64_outputs(seed: int, start: int, n: int) -> np.ndarray:
    """n raw std::mt19937_64(seed) outputs from index start on, by jump-ahead (the chunked
    feature streams of gen_synthetic, harness.cpp:153-162)."""
    out = np.empty(n, np.uint64)
    N.check(N.lib().hg_mt64_outputs(seed, start, n, out.ctypes.data))
    return out


# ---- graphs --------------------------------------------------------------------------------


class HetGraph:
    """Host graph owned by the native layer (hetgraph.hpp:58-74)."""

    def __init__(self, handle):
        self._h = handle if handle else N.raise_last()

    def __del__(self):
        if getattr(self, "_h", None) and N._lib is not None:
            N._lib.hg_graph_free(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def export(self) -> Dict[str, np.ndarray]:
        return N.take(N.lib().hg_graph_export(self._h))


def gen_synthetic(spec: dict, seed: int) -> HetGraph:
    """gen_synthetic (src/harness.cpp:74-186): bit-exact graph, features and labels."""
    keep = []

    def cs(s):
        b = s.encode()
        keep.append(b)
        return b

    for t in spec["node_types"]:
        if t.get("storage", "dense") not in ("dense", "learnable"):
            raise ValueError("unknown storage kind: " + t["storage"])
    for r in spec["relations"]:
        if r.get("degree", "uniform") not in ("uniform", "powerlaw"):
            raise ValueError("unknown degree distribution: " + r["degree"])
    types = (N.SpecNodeType * max(1, len(spec["node_types"])))()
    for i, t in enumerate(spec["node_types"]):
        types[i] = N.SpecNodeType(cs(t["name"]), int(t["count"]), int(t["dim"]),
                                  1 if t.get("storage", "dense") == "dense" else 2)
    rels = (N.SpecRelation * max(1, len(spec["relations"])))()
    for i, r in enumerate(spec["relations"]):
        rels[i] = N.SpecRelation(cs(r["src"]), cs(r["edge"]), cs(r["dst"]), int(r["edges"]),
                                 1 if r.get("degree", "uniform") == "powerlaw" else 0, float(r.get("alpha", 2.0)))
    sp = spec.get("self_paired", [])
    sp_arr = (C.c_char_p * max(1, len(sp)))(*[cs(x) for x in sp])
    s = N.Spec(cs(spec["target"]), int(spec["num_classes"]), float(spec.get("label_noise", 0.0)),
               len(spec["node_types"]), types, len(spec["relations"]), rels, int(spec.get("add_reverse", True)),
               len(sp), sp_arr)
    return HetGraph(N.lib().hg_graph_generate(C.byref(s), seed))


def load_container(path: str) -> HetGraph:
    """load_container (src/container.cpp:92-154): an HGC1 file."""
    return HetGraph(N.lib().hg_graph_load(str(path).encode()))


def save_container(g: HetGraph, path: str) -> None:
    """save_container (src/container.cpp:47-90): byte-identical to the reference's writer."""
    N.check(N.lib().hg_graph_save(g.handle, str(path).encode()))


def graph_from_export(e: Dict[str, np.ndarray]) -> HetGraph:
    """A HetGraph from exported arrays (the oracle's or ours): CSR per relation."""
    counts = np.asarray(e["node_counts"], np.uint64)
    nt = len(counts)
    rs = np.asarray(e["rel_src"], np.int32)
    rd = np.asarray(e["rel_dst"], np.int32)
    rr = np.asarray(e.get("rel_reverse", np.zeros(len(rs))), np.int32)
    ip = np.concatenate([np.asarray(e[f"rel{r}.indptr"], np.uint64) for r in range(len(rs))] or [np.zeros(1, np.uint64)])
    sr = np.concatenate([np.asarray(e[f"rel{r}.src"], np.uint32) for r in range(len(rs))] or [np.zeros(1, np.uint32)])
    if sr.size == 0:
        sr = np.zeros(1, np.uint32)
    kinds = np.asarray(e["kinds"], np.int32)
    dims = np.asarray(e["dims"], np.int32)
    dense = [np.asarray(e[f"feat.t{t}"], np.float32).ravel() for t in range(nt) if kinds[t] == 1]
    dense = np.concatenate(dense) if dense else np.zeros(1, np.float32)
    labels = np.asarray(e["labels"], np.int32)
    return HetGraph(N.lib().hg_graph_from_csr(nt, N.ptr(counts), len(rs), N.ptr(rs), N.ptr(rd), N.ptr(rr),
                                              N.ptr(ip), N.ptr(sr), N.ptr(kinds), N.ptr(dims), N.ptr(dense),
                                              int(np.asarray(e["target"]).ravel()[0]),
                                              int(np.asarray(e["num_classes"]).ravel()[0]), N.ptr(labels)))


def build_hetgraph(counts: Sequence[int], relations: Sequence[tuple], edges: Sequence[Sequence[tuple]],
                   target: int, num_classes: int) -> HetGraph:
    """build_hetgraph (src/hetgraph.cpp:126-156); relations = [(src_type, dst_type)]."""
    cnt = np.asarray(counts, np.uint64)
    rs = np.asarray([r[0] for r in relations], np.int32)
    rd = np.asarray([r[1] for r in relations], np.int32)
    pc = np.asarray([len(e) for e in edges], np.uint64)
    ps = np.asarray([p[0] for e in edges for p in e] or [0], np.uint32)
    pd = np.asarray([p[1] for e in edges for p in e] or [0], np.uint32)
    return HetGraph(N.lib().hg_graph_from_pairs(len(cnt), N.ptr(cnt), len(rs), N.ptr(rs), N.ptr(rd), N.ptr(pc),
                                                N.ptr(ps), N.ptr(pd), target, num_classes))


def meta_partition(g: HetGraph, k: int, p: int) -> Dict[str, np.ndarray]:
    """meta_partition + cacheable_types + hop_relation_sets (metapartition.cpp:283, cache.cpp:143)."""
    return N.take(N.lib().hg_meta_partition(g.handle, k, p))


def init_model(g: HetGraph, k: int, hidden: int, seed: int) -> Dict[str, np.ndarray]:
    """init_model (src/hgnn.cpp:39-62) on the BFS metatree of depth k: w.r{r}.l{l} f64."""
    return N.take(N.lib().hg_init_model(g.handle, k, hidden, seed))


def init_learnable(g: HetGraph, seed: int) -> Dict[str, np.ndarray]:
    """init_learnable (src/hgnn.cpp:64-81): learn.t{t} f64 [count x dim]."""
    return N.take(N.lib().hg_init_learnable(g.handle, seed))


def meta_partition_work_aware(g: HetGraph, k: int, p: int, work: Sequence[float]) -> Dict[str, np.ndarray]:
    """Work-aware plan (not the reference's policy): worker groups replicate sets of
    sub-metatrees so the busiest worker's share of `work` is smallest."""
    w = np.ascontiguousarray(work, dtype=np.float64)
    return N.take(N.lib().hg_meta_partition_work_aware(g.handle, k, p, N.ptr(w), len(w)))


def sub_work(g: HetGraph, fanouts: Sequence[int], n_batches: int = 4, batch_size: int = 1024, seed: int = 1,
             device: int = 0) -> Dict[str, np.ndarray]:
    """Per sub-metatree: sampled edges ("work") and learnable layer-0 rows ("learn_rows") per
    batch, from device samplers restricted to the sub's relations."""
    fo = np.asarray(fanouts, np.int32)
    return N.take(N.lib().hg_sub_work(g.handle, N.ptr(fo), len(fo), n_batches, batch_size, seed, device))


def make_batches(g: HetGraph, batch_size: int, max_batches: int, seed: int) -> List[np.ndarray]:
    """make_batches (src/harness.cpp:327-340)."""
    b = N.take(N.lib().hg_make_batches(g.handle, batch_size, max_batches, seed))
    return [b[f"batch{i}"] for i in range(len(b))]


def cache_plan(g: HetGraph, hot: Dict[str, np.ndarray], n_types: int, budget: int, read_ns=1.0, write_ns=1.0,
               overhead_ns=1000.0, elem_bytes=4) -> Dict[str, np.ndarray]:
    """profile_miss_penalty + allocate_cache + fill_and_serve (src/cache.cpp:11-141)."""
    counts = np.concatenate([np.asarray(hot[f"hot.t{t}"], np.uint64) for t in range(n_types)])
    return N.take(N.lib().hg_cache_plan(g.handle, N.ptr(counts), budget, read_ns, write_ns, overhead_ns, elem_bytes))


# ---- device engine ---------------------------------------------------------------------------


class Engine:
    """One meta-partition of the RAF engine on one GPU (run_raf_batch, raf.cpp:344-530)."""

    FEAT_DTYPES = {"f32": 0, "f16": 1, "bf16": 2}
    MODELS = {"rgcn": 0, "rgat": 1}  # RGAT: relational attention (no reference counterpart)

    def __init__(self, g: HetGraph, fanouts: Sequence[int], hidden: int = 64, batch_cap: int = 1024, p: int = 1,
                 rank: int = 0, model_seed: int = 0, learn_seed: int = 0, device: int = 0, feat_dtype: str = "f32",
                 feat_host: bool = False, sub_work: Optional[Sequence[float]] = None, model: str = "rgcn",
                 heads: int = 4):
        fo = (C.c_int * len(fanouts))(*[int(f) for f in fanouts])
        self._fo = fo
        if feat_dtype not in self.FEAT_DTYPES:
            raise ValueError("feature dtype must be one of f32, f16, bf16")
        if model not in self.MODELS:
            raise ValueError("model must be one of rgcn, rgat")
        opts = N.EngineOpts(len(fanouts), fo, hidden, batch_cap, p, rank, model_seed, learn_seed, device,
                            self.FEAT_DTYPES[feat_dtype], int(bool(feat_host)), self.MODELS[model], heads)
        self.model = model
        self.heads = heads
        self.k = len(fanouts)
        self.graph = g  # keep alive
        if sub_work is None:
            self._h = N.lib().hg_engine_create(g.handle, C.byref(opts))
        else:  # the work-aware plan (not the reference's meta_partition)
            w = np.ascontiguousarray(sub_work, dtype=np.float64)
            self._h = N.lib().hg_engine_create_work_aware(g.handle, C.byref(opts), N.ptr(w), len(w))
        if not self._h:
            N.raise_last()

    @classmethod
    def from_container(cls, path: str, fanouts: Sequence[int], hidden: int = 64, batch_cap: int = 1024, p: int = 1,
                       rank: int = 0, model_seed: int = 0, learn_seed: int = 0, device: int = 0,
                       feat_dtype: str = "f32", feat_host: bool = False, model: str = "rgcn",
                       heads: int = 4) -> "Engine":
        """Streaming loader: the graph goes from an HGC1 container (container.cpp:92-154)
        straight into HBM, relation pairs and feature rows through pinned buffers."""
        self = cls.__new__(cls)
        fo = (C.c_int * len(fanouts))(*[int(f) for f in fanouts])
        self._fo = fo
        if feat_dtype not in cls.FEAT_DTYPES or model not in cls.MODELS:
            raise ValueError("feature dtype must be one of f32, f16, bf16 and model one of rgcn, rgat")
        opts = N.EngineOpts(len(fanouts), fo, hidden, batch_cap, p, rank, model_seed, learn_seed, device,
                            cls.FEAT_DTYPES[feat_dtype], int(bool(feat_host)), cls.MODELS[model], heads)
        self.k, self.model, self.heads, self.graph = len(fanouts), model, heads, None
        self._h = N.lib().hg_engine_create_from_container(str(path).encode(), C.byref(opts))
        if not self._h:
            N.raise_last()
        return self

    @classmethod
    def for_experiment(cls, g: HetGraph, fanouts, hidden, seed, **kw) -> "Engine":
        """Seeds as run_experiment derives them (harness.cpp:365-366)."""
        return cls(g, fanouts, hidden, model_seed=mix_seed(seed, 0xD0DE1), learn_seed=mix_seed(seed, 0x1EA4A), **kw)

    def __del__(self):
        if getattr(self, "_h", None) and N._lib is not None:
            N._lib.hg_engine_free(self._h)
            self._h = None

    def step(self, batch, rng_seed: int, designated: int = 0, train: bool = True) -> dict:
        b = np.ascontiguousarray(batch, dtype=np.uint32)
        rep = N.StepReport()
        N.check(N.lib().hg_engine_step(self._h, N.ptr(b), len(b), rng_seed, designated, int(train), C.byref(rep)))
        # ExecutionReport fields (raf.hpp:66-77); sync_bytes is this rank's replica
        # group's share: sum it over the ranks whose sync_leader is set
        return dict(loss=rep.loss, sampled_edges=int(rep.sampled_edges),
                    active_rows=[rep.active_rows[i] for i in range(rep.n_active)],
                    sync_bytes=int(rep.sync_bytes), sync_leader=bool(rep.sync_leader),
                    message_bound_ok=bool(rep.message_bound_ok), target_only_ok=bool(rep.target_only_ok),
                    cross_ids_target_only=bool(rep.target_only_ok),
                    boundary_counts=[int(rep.boundary_counts[i]) for i in range(rep.n_boundary)],
                    boundary_cut_edges=int(rep.boundary_cut_edges))

    def prefetch(self, batch, rng_seed: int) -> None:
        """Sample a future batch now (sampling stream, second sample slot); the
        step() with the same (batch, rng_seed) then trains on it while the
        next prefetch samples. Keeps the numbers identical to an unprefetched step."""
        b = np.ascontiguousarray(batch, dtype=np.uint32)
        N.check(N.lib().hg_engine_prefetch(self._h, N.ptr(b), len(b), rng_seed))

    def sample(self, seeds, rng_seed: int) -> None:
        b = np.ascontiguousarray(seeds, dtype=np.uint32)
        if b.size == 0:
            raise ValueError("empty batch")
        N.check(N.lib().hg_engine_sample(self._h, N.ptr(b), len(b), rng_seed))

    def read(self, *names: str) -> Dict[str, np.ndarray]:
        return N.take(N.lib().hg_engine_read(self._h, ",".join(names).encode() if names else None))

    def bench(self, batches: Sequence[np.ndarray], seeds: Sequence[int], train: bool = True):
        flat = np.ascontiguousarray(np.concatenate(batches), dtype=np.uint32)
        lens = np.asarray([len(b) for b in batches], np.int32)
        sd = np.asarray(seeds, np.uint64)
        ms, edges, loss = C.c_double(), C.c_uint64(), C.c_double()
        N.check(N.lib().hg_engine_bench(self._h, N.ptr(flat), N.ptr(lens), N.ptr(sd), len(batches), int(train),
                                        C.byref(ms), C.byref(edges), C.byref(loss)))
        return ms.value, int(edges.value), loss.value

    def profile(self, on: bool = True):
        N.lib().hg_engine_profile(self._h, int(on))

    def profile_read(self) -> Dict[str, np.ndarray]:
        return N.take(N.lib().hg_engine_profile_read(self._h))

    def info(self) -> dict:
        pc, db, ms = C.c_uint64(), C.c_uint64(), C.c_int()
        N.check(N.lib().hg_engine_info(self._h, C.byref(pc), C.byref(db), C.byref(ms)))
        return dict(param_count=pc.value, device_bytes=db.value, model_step=ms.value)

    def set_option(self, name: str, value) -> None:
        N.check(N.lib().hg_engine_set_option(self._h, name.encode(), int(value)))

    def count_launches(self, n: int, train: bool = True) -> int:
        return N.check(N.lib().hg_engine_count_launches(self._h, n, int(train)))

    def presample_hotness(self, epochs: int, seed: int, batch_size: int = 512) -> Dict[str, np.ndarray]:
        return N.take(N.lib().hg_engine_presample_hotness(self._h, epochs, seed, batch_size))

    def set_cache(self, cached: Sequence[np.ndarray]):
        ids = np.concatenate([np.asarray(c, np.uint32) for c in cached] or [np.zeros(0, np.uint32)])
        if ids.size == 0:
            ids = np.zeros(1, np.uint32)
        lens = np.asarray([len(c) for c in cached], np.uint64)
        N.check(N.lib().hg_engine_set_cache(self._h, N.ptr(ids), N.ptr(lens), len(cached)))

    def cache_counters(self) -> Dict[str, np.ndarray]:
        return N.take(N.lib().hg_engine_cache_counters(self._h))

    def attach_nccl(self, unique_id: bytes, nranks: int, rank: int):
        buf = C.create_string_buffer(unique_id, len(unique_id))
        N.check(N.lib().hg_engine_attach_nccl(self._h, buf, len(unique_id), nranks, rank))

    def replica_handle(self) -> bytes:
        """CUDA IPC handle of this partition's gradient-exchange arena (b"" without replicas)."""
        buf = C.create_string_buffer(4096)
        n = N.check(N.lib().hg_engine_replica_handle(self._h, buf, 4096))
        return buf.raw[:n]

    def attach_replicas(self, handles: Sequence[bytes]):
        """Map the replica peers' exchange arenas (handles of every rank, rank order)."""
        size = max([len(h) for h in handles] + [1])
        flat = b"".join(h.ljust(size, b"\0") for h in handles)
        buf = C.create_string_buffer(flat, len(flat))
        N.check(N.lib().hg_engine_attach_replicas(self._h, buf, size, len(handles)))

    # ---- reference-named views --------------------------------------------------------
    def sample_khop_restricted(self, seeds, rng_seed: int) -> Dict[str, np.ndarray]:
        """sample_khop_restricted (sampling.cpp:99-103) with this engine's hop relation sets."""
        self.sample(seeds, rng_seed)
        names = [n for n in self.tensor_names() if n.startswith(("frontier", "hop"))]
        return self.read(*names)

    def tensor_names(self) -> List[str]:
        raw = N.take(N.lib().hg_engine_read(self._h, b"?"))["names"]
        return [x for x in bytes(raw.astype(np.uint8)).decode().split(",") if x]


class Sampler:
    """Device sampler for sample_khop / sample_khop_restricted (sampling.cpp:94-103):
    explicit per-hop relation sets (None = every relation at every hop)."""

    def __init__(self, g: HetGraph, fanouts: Sequence[int], hop_relations: Optional[Sequence[Sequence[int]]] = None,
                 batch_cap: int = 1024, device: int = 0):
        if len(fanouts) == 0:
            raise ValueError("fanouts must be non-empty")
        fo = np.asarray(fanouts, np.int32)
        self.k = len(fanouts)
        self.graph = g
        if hop_relations is None:
            flat = cnt = None
        else:
            if len(hop_relations) != len(fanouts):
                raise ValueError("hop_relations must have one entry per hop")
            flat = np.asarray([r for h in hop_relations for r in h] or [-1], np.int32)
            cnt = np.asarray([len(h) for h in hop_relations], np.int32)
        self._h = N.lib().hg_sampler_create(g.handle, N.ptr(fo), len(fo), N.ptr(flat), N.ptr(cnt), batch_cap, device)
        if not self._h:
            N.raise_last()

    def __del__(self):
        if getattr(self, "_h", None) and N._lib is not None:
            N._lib.hg_engine_free(self._h)
            self._h = None

    def sample(self, seeds, rng_seed: int) -> Dict[str, np.ndarray]:
        """frontier{h}.t{t} and hop{h}.rel{r}.{dst_ids,indptr,src_ids} of one call."""
        b = np.ascontiguousarray(seeds, dtype=np.uint32)
        if b.size == 0:
            raise ValueError("empty batch")
        N.check(N.lib().hg_engine_sample(self._h, N.ptr(b), len(b), rng_seed))
        names = [x for x in bytes(N.take(N.lib().hg_engine_read(self._h, b"?"))["names"].astype(np.uint8)).decode()
                 .split(",") if x.startswith(("frontier", "hop")) and not x.endswith(".col")]
        return N.take(N.lib().hg_engine_read(self._h, ",".join(names).encode()))


def cache_stats(counters: Dict[str, np.ndarray], kinds: Sequence[int], transfer_ns: Sequence[float]) -> List[dict]:
    """CacheState accounting (cache.cpp:87-113, hook harness.cpp:425-437) from the
    engine's per-type lookup counters: every layer-0 frontier id is looked up,
    and learnable types (kind 2) are also updated, which counts a second
    hit/miss; each miss adds the type's transfer penalty."""
    out = []
    for t, kind in enumerate(kinds):
        key = f"cache.t{t}"
        if key not in counters:
            continue
        hits, misses = (int(x) for x in counters[key])
        mult = 2 if int(kind) == 2 else 1
        h, m = hits * mult, misses * mult
        out.append(dict(type=t, hits=h, misses=m, hit_rate=h / (h + m) if h + m else 0.0,
                        penalty_ns=m * float(transfer_ns[t])))
    return out


def agg_all_comm_bytes(active_rows: Sequence[int], designated: int, num_classes: int, elem_bytes: int = 4,
                       header_bytes: int = 32) -> Dict[str, int]:
    """CommStats of one batch's AGG_all exchange (raf.cpp:427-466, payload_bytes
    raf.cpp:113-115): every partition q != designated with at least one active
    row sends a PartialAgg of rows x C elements and receives the mirrored
    PartialGrad. `active_rows` is the per-partition list a step reports."""
    sent = [header_bytes + int(a) * num_classes * elem_bytes
            for q, a in enumerate(active_rows) if q != designated and int(a) > 0]
    return {"messages": 2 * len(sent), "partial_agg_bytes": sum(sent), "partial_grad_bytes": sum(sent),
            "total_bytes": 2 * sum(sent)}


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(256)
    n = N.check(N.lib().hg_nccl_unique_id(buf, 256))
    return buf.raw[:n]
