"""ctypes binding of the C-ABI in include/hetgpu.h (libhetgpu.so, built in-tree).

There is no fallback: if the shared library is missing, importing the product
API raises. The library is the product; this module only marshals arguments.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# HETGPU_LIB: an alternative build of the same library (A/B measurements)
LIB_PATH = os.environ.get("HETGPU_LIB") or os.path.join(HERE, "libhetgpu.so")

_lib = None


class HetGpuError(RuntimeError):
    pass


class SpecNodeType(C.Structure):
    _fields_ = [("name", C.c_char_p), ("count", C.c_uint64), ("dim", C.c_int), ("storage", C.c_int)]


class SpecRelation(C.Structure):
    _fields_ = [("src", C.c_char_p), ("edge", C.c_char_p), ("dst", C.c_char_p), ("edges", C.c_uint64),
                ("powerlaw", C.c_int), ("alpha", C.c_double)]


class Spec(C.Structure):
    _fields_ = [("target", C.c_char_p), ("num_classes", C.c_int), ("label_noise", C.c_double),
                ("n_types", C.c_int), ("types", C.POINTER(SpecNodeType)), ("n_rels", C.c_int),
                ("rels", C.POINTER(SpecRelation)), ("add_reverse", C.c_int), ("n_self_paired", C.c_int),
                ("self_paired", C.POINTER(C.c_char_p))]


class EngineOpts(C.Structure):
    _fields_ = [("k", C.c_int), ("fanouts", C.POINTER(C.c_int)), ("hidden", C.c_int), ("batch_cap", C.c_int),
                ("p", C.c_int), ("rank", C.c_int), ("model_seed", C.c_uint64), ("learn_seed", C.c_uint64),
                ("device", C.c_int), ("feat_dtype", C.c_int), ("feat_host", C.c_int),
                ("model", C.c_int), ("heads", C.c_int)]


class StepReport(C.Structure):
    _fields_ = [("loss", C.c_double), ("sampled_edges", C.c_uint64), ("n_active", C.c_int),
                ("active_rows", C.c_int * 64), ("sync_bytes", C.c_uint64), ("sync_leader", C.c_int),
                ("message_bound_ok", C.c_int), ("target_only_ok", C.c_int), ("n_boundary", C.c_int),
                ("boundary_cut_edges", C.c_uint64), ("boundary_counts", C.c_uint64 * 64)]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise HetGpuError(f"native library missing: {LIB_PATH} (run __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        vp, i32, u64 = C.c_void_p, C.c_int, C.c_uint64
        sig = {
            "hg_last_error": ([], C.c_char_p),
            "hg_last_error_kind": ([], i32),
            "hg_version": ([], C.c_char_p),
            "hg_bundle_size": ([vp], i32),
            "hg_bundle_name": ([vp, i32], C.c_char_p),
            "hg_bundle_dtype": ([vp, i32], C.c_char_p),
            "hg_bundle_ndim": ([vp, i32], i32),
            "hg_bundle_dim": ([vp, i32, i32], C.c_longlong),
            "hg_bundle_nbytes": ([vp, i32], C.c_longlong),
            "hg_bundle_data": ([vp, i32], vp),
            "hg_bundle_free": ([vp], None),
            "hg_mix_seed": ([u64, u64], u64),
            "hg_mt64_outputs": ([u64, u64, u64, vp], i32),
            "hg_engine_create_from_container": ([C.c_char_p, C.POINTER(EngineOpts)], vp),
            "hg_graph_generate": ([C.POINTER(Spec), u64], vp),
            "hg_graph_from_csr": ([i32, vp, i32, vp, vp, vp, vp, vp, vp, vp, vp, i32, i32, vp], vp),
            "hg_graph_from_pairs": ([i32, vp, i32, vp, vp, vp, vp, vp, i32, i32], vp),
            "hg_graph_free": ([vp], None),
            "hg_graph_load": ([C.c_char_p], vp),
            "hg_graph_save": ([vp, C.c_char_p], i32),
            "hg_graph_export": ([vp], vp),
            "hg_graph_schema": ([vp], vp),
            "hg_sampler_create": ([vp, vp, i32, vp, vp, i32, i32], vp),
            "hg_meta_partition": ([vp, i32, i32], vp),
            "hg_make_batches": ([vp, i32, i32, u64], vp),
            "hg_engine_create": ([vp, C.POINTER(EngineOpts)], vp),
            "hg_engine_free": ([vp], None),
            "hg_engine_step": ([vp, vp, i32, u64, i32, i32, C.POINTER(StepReport)], i32),
            "hg_engine_sample": ([vp, vp, i32, u64], i32),
            "hg_engine_prefetch": ([vp, vp, i32, u64], i32),
            "hg_engine_read": ([vp, C.c_char_p], vp),
            "hg_engine_bench": ([vp, vp, vp, vp, i32, i32, C.POINTER(C.c_double), C.POINTER(C.c_uint64),
                                 C.POINTER(C.c_double)], i32),
            "hg_engine_profile": ([vp, i32], None),
            "hg_engine_profile_read": ([vp], vp),
            "hg_engine_info": ([vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_int)], i32),
            "hg_engine_count_launches": ([vp, i32, i32], i32),
            "hg_selftest_contractions": ([vp, i32, i32], vp),
            "hg_engine_set_option": ([vp, C.c_char_p, i32], i32),
            "hg_engine_presample_hotness": ([vp, i32, u64, i32], vp),
            "hg_cache_plan": ([vp, vp, u64, C.c_double, C.c_double, C.c_double, i32], vp),
            "hg_engine_set_cache": ([vp, vp, vp, i32], i32),
            "hg_engine_cache_counters": ([vp], vp),
            "hg_nccl_unique_id": ([vp, i32], i32),
            "hg_engine_attach_nccl": ([vp, vp, i32, i32, i32], i32),
            "hg_engine_replica_handle": ([vp, vp, i32], i32),
            "hg_engine_attach_replicas": ([vp, vp, i32, i32], i32),
            "hg_init_model": ([vp, i32, i32, u64], vp),
            "hg_meta_partition_work_aware": ([vp, i32, i32, vp, i32], vp),
            "hg_sub_work": ([vp, vp, i32, i32, i32, u64, i32], vp),
            "hg_engine_create_work_aware": ([vp, C.POINTER(EngineOpts), vp, i32], vp),
            "hg_init_learnable": ([vp, u64], vp),
            "hg_engine_load_weights": ([vp, i32, i32, vp, i32, i32], i32),
            "hg_engine_load_table_rows": ([vp, i32, vp, C.c_int64, vp, i32], i32),
            "hg_sample_neighbors": ([vp, u64, vp, C.c_uint32, i32, u64, i32, i32, vp, vp, i32], i32),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def raise_last():
    L = lib()
    msg = L.hg_last_error().decode()
    kind = L.hg_last_error_kind()
    if kind == 1:
        raise ValueError(msg)  # std::invalid_argument
    raise HetGpuError(msg)     # std::runtime_error and CUDA errors


def check(rc):
    if rc is None or (isinstance(rc, int) and rc < 0):
        raise_last()
    return rc


def ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def take(h) -> Dict[str, np.ndarray]:
    if not h:
        raise_last()
    L = lib()
    out = {}
    try:
        for i in range(L.hg_bundle_size(h)):
            name = L.hg_bundle_name(h, i).decode()
            dt = np.dtype(L.hg_bundle_dtype(h, i).decode())
            shape = tuple(L.hg_bundle_dim(h, i, d) for d in range(L.hg_bundle_ndim(h, i)))
            nb = L.hg_bundle_nbytes(h, i)
            raw = C.string_at(L.hg_bundle_data(h, i), nb) if nb else b""
            out[name] = np.frombuffer(raw, dtype=dt).reshape(shape).copy()
    finally:
        L.hg_bundle_free(h)
    return out
