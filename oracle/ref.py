"""TEST INFRASTRUCTURE ONLY — the checker, never the thing measured or shipped.

ctypes binding of oracle/_ref/libhetsim_ref.so: the *unmodified* reference
library (hetsim, /root/reference/proj/src/*.cpp) compiled by oracle/Makefile,
plus the C-ABI shim in oracle/ref_shim.cpp. Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs may import this module.

Every shim call returns a "bundle" (name -> numpy array) that `_take` converts.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from typing import Dict, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libhetsim_ref.so")
_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"reference oracle not built: {LIB_PATH} (run `make -C oracle`)")
        L = C.CDLL(LIB_PATH)
        vp, u64, i32 = C.c_void_p, C.c_ulonglong, C.c_int
        L.ref_last_error.restype = C.c_char_p
        L.ref_bundle_size.argtypes = [vp]
        L.ref_bundle_name.argtypes = [vp, i32]
        L.ref_bundle_name.restype = C.c_char_p
        L.ref_bundle_dtype.argtypes = [vp, i32]
        L.ref_bundle_dtype.restype = C.c_char_p
        L.ref_bundle_ndim.argtypes = [vp, i32]
        L.ref_bundle_dim.argtypes = [vp, i32, i32]
        L.ref_bundle_dim.restype = C.c_longlong
        L.ref_bundle_nbytes.argtypes = [vp, i32]
        L.ref_bundle_nbytes.restype = C.c_longlong
        L.ref_bundle_data.argtypes = [vp, i32]
        L.ref_bundle_data.restype = vp
        L.ref_bundle_free.argtypes = [vp]
        for name, args in {
            "ref_graph_random": [u64, i32, i32, i32],
            "ref_graph_bundled": [C.c_char_p, u64],
            "ref_graph_spec": [C.c_char_p, u64],
            "ref_graph_load": [C.c_char_p],
            "ref_graph_save": [vp, C.c_char_p],
            "ref_graph_build": [i32, vp, i32, vp, vp, vp, vp, vp, i32, i32, vp, vp, vp, vp],
            "ref_graph_export": [vp],
            "ref_graph_round_features": [vp, i32],
            "ref_meta_partition": [vp, i32, i32],
            "ref_sample_neighbors": [vp, i32, vp, C.c_uint, i32, u64, i32, i32],
            "ref_sample_khop": [vp, vp, i32, vp, i32, u64, vp, vp],
            "ref_flat_step": [vp, i32, i32, u64, u64, vp, i32, vp, u64, i32],
            "ref_raf_train": [vp, i32, i32, i32, u64, vp, vp, i32, vp, i32, i32],
            "ref_check_equivalence": [vp, i32, i32, i32, u64, u64, vp, i32, vp, u64, i32],
            "ref_cache_sim": [vp, i32, vp, i32, u64, i32, u64, C.c_double, C.c_double, C.c_double, i32],
            "ref_run_experiment": [C.c_char_p],
            "ref_bench_raf": [vp, i32, i32, i32, u64, i32, vp, i32, i32, i32],
        }.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = vp
        L.ref_graph_free.argtypes = [vp]
        L.ref_mix_seed.argtypes = [u64, u64]
        L.ref_mix_seed.restype = u64
        _lib = L
    return _lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _check(h):
    if not h:
        raise RuntimeError(lib().ref_last_error().decode())
    return h


def _take(h) -> Dict[str, np.ndarray]:
    L = lib()
    _check(h)
    out = {}
    try:
        for i in range(L.ref_bundle_size(h)):
            name = L.ref_bundle_name(h, i).decode()
            dt = np.dtype(L.ref_bundle_dtype(h, i).decode())
            shape = tuple(L.ref_bundle_dim(h, i, d) for d in range(L.ref_bundle_ndim(h, i)))
            nb = L.ref_bundle_nbytes(h, i)
            buf = (C.c_char * nb).from_address(L.ref_bundle_data(h, i)) if nb else b""
            arr = np.frombuffer(bytes(buf), dtype=dt).reshape(shape).copy()
            out[name] = arr
    finally:
        L.ref_bundle_free(h)
    return out


def as_text(a: np.ndarray) -> str:
    return bytes(a.astype(np.uint8)).decode()


class RefGraph:
    """Owns a reference HetGraph (the oracle's own copy)."""

    def __init__(self, handle):
        self.h = _check(handle)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_graph_free(self.h)
            self.h = None

    @classmethod
    def random(cls, seed: int, max_types=5, max_rels=8, max_nodes=200) -> "RefGraph":
        return cls(lib().ref_graph_random(seed, max_types, max_rels, max_nodes))

    @classmethod
    def bundled(cls, name: str, seed: int) -> "RefGraph":
        return cls(lib().ref_graph_bundled(name.encode(), seed))

    @classmethod
    def from_spec(cls, spec: dict, seed: int) -> "RefGraph":
        return cls(lib().ref_graph_spec(json.dumps(spec).encode(), seed))

    @classmethod
    def build(cls, counts, rels, edges, target, num_classes, labels, kinds, dims, dense=None):
        """rels: [(src_type, dst_type)], edges: per relation list of (src, dst)."""
        counts = np.asarray(counts, np.uint64)
        rs = np.asarray([r[0] for r in rels], np.int32)
        rd = np.asarray([r[1] for r in rels], np.int32)
        ec = np.asarray([len(e) for e in edges], np.uint64)
        es = np.asarray([p[0] for e in edges for p in e] or [0], np.uint32)
        ed = np.asarray([p[1] for e in edges for p in e] or [0], np.uint32)
        lab = np.asarray(labels, np.int32)
        kd = np.asarray(kinds, np.int32)
        dm = np.asarray(dims, np.int32)
        dv = np.concatenate([np.asarray(d, np.float64).ravel() for d in (dense or [])] or [np.zeros(1)])
        return cls(lib().ref_graph_build(len(counts), _ptr(counts), len(rels), _ptr(rs), _ptr(rd),
                                         _ptr(ec), _ptr(es), _ptr(ed), target, num_classes,
                                         _ptr(lab), _ptr(kd), _ptr(dm), _ptr(dv)))

    @classmethod
    def load(cls, path: str) -> "RefGraph":
        return cls(lib().ref_graph_load(str(path).encode()))

    def save(self, path: str) -> None:
        _take(lib().ref_graph_save(self.h, str(path).encode()))

    def export(self) -> Dict[str, np.ndarray]:
        return _take(lib().ref_graph_export(self.h))

    def round_features(self, dtype: str) -> None:
        """Dense features rounded in place to fp16 ("f16") or bf16 ("bf16") values."""
        _take(lib().ref_graph_round_features(self.h, {"f16": 1, "bf16": 2}[dtype]))

    def meta_partition(self, k: int, p: int) -> Dict[str, np.ndarray]:
        return _take(lib().ref_meta_partition(self.h, k, p))

    def sample_khop(self, seeds: Sequence[int], fanouts: Sequence[int], rng_seed: int,
                    hop_relations: Optional[Sequence[Sequence[int]]] = None):
        sd = np.asarray(seeds, np.uint32)
        fo = np.asarray(fanouts, np.int32)
        if hop_relations is None:
            flat, cnt = None, None
        else:
            flat = np.asarray([r for h in hop_relations for r in h] or [0], np.int32)
            cnt = np.asarray([len(h) for h in hop_relations], np.int32)
        return _take(lib().ref_sample_khop(self.h, _ptr(sd), len(sd), _ptr(fo), len(fo), rng_seed,
                                           _ptr(flat), _ptr(cnt)))

    def flat_step(self, k, hidden, model_seed, learn_seed, batch, fanouts, rng_seed, want_init=True):
        """want_init: True = initial state with full learnable tables; "rows" = the
        learnable tables only at the rows the batch touches (init/post .learn_rows)."""
        want_init = 2 if want_init == "rows" else int(bool(want_init))
        bt = np.asarray(batch, np.uint32)
        fo = np.asarray(fanouts, np.int32)
        return _take(lib().ref_flat_step(self.h, k, hidden, model_seed, learn_seed, _ptr(bt), len(bt),
                                         _ptr(fo), rng_seed, want_init))

    def raf_train(self, k, hidden, p, seed, batches, fanouts, elem_bytes=4, full_tables=True):
        flat = np.asarray([v for b in batches for v in b], np.uint32)
        cnt = np.asarray([len(b) for b in batches], np.int32)
        fo = np.asarray(fanouts, np.int32)
        return _take(lib().ref_raf_train(self.h, k, hidden, p, seed, _ptr(flat), _ptr(cnt),
                                         len(batches), _ptr(fo), elem_bytes, int(full_tables)))

    def check_equivalence(self, k, hidden, p, model_seed, learn_seed, batch, fanouts, rng_seed,
                          designated):
        bt = np.asarray(batch, np.uint32)
        fo = np.asarray(fanouts, np.int32)
        return _take(lib().ref_check_equivalence(self.h, k, hidden, p, model_seed, learn_seed, _ptr(bt),
                                                 len(bt), _ptr(fo), rng_seed, designated))

    def cache_sim(self, k, fanouts, epochs, seed, batch_size, budget=0, read_ns=1.0, write_ns=1.0,
                  overhead_ns=1000.0, elem_bytes=4):
        fo = np.asarray(fanouts, np.int32)
        return _take(lib().ref_cache_sim(self.h, k, _ptr(fo), epochs, seed, batch_size, budget,
                                         read_ns, write_ns, overhead_ns, elem_bytes))

    def bench_raf(self, k, hidden, p, seed, batch_size, fanouts, first_batch, n_batches, n_threads):
        fo = np.asarray(fanouts, np.int32)
        return _take(lib().ref_bench_raf(self.h, k, hidden, p, seed, batch_size, _ptr(fo),
                                         first_batch, n_batches, n_threads))


def sample_neighbors(indptr, src, dst, fanout, rng_seed, hop, rel) -> np.ndarray:
    ip = np.asarray(indptr, np.uint64)
    sr = np.asarray(src, np.uint32)
    if sr.size == 0:
        sr = np.zeros(1, np.uint32)
    return _take(lib().ref_sample_neighbors(_ptr(ip), len(ip) - 1, _ptr(sr), dst, fanout, rng_seed,
                                            hop, rel))["out"]


def run_experiment(config: dict):
    r = _take(lib().ref_run_experiment(json.dumps(config).encode()))
    return json.loads(as_text(r["stats"])), as_text(r["hash"]), bool(r["checks_ok"][0])


def mix_seed(a: int, b: int) -> int:
    return int(lib().ref_mix_seed(a, b))
