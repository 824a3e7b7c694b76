"""B200-native community detection: PLP / PLM / PLMR / EPP on sm_100a.

Python mirror of the reference's detector interface
(/root/reference/proj/include/commdet, "H/" below) over the C ABI of
``libcommdet_cuda.so`` (include/commdet_cuda.h).  Names, argument meaning and
error behaviour follow the reference:

    Graph.from_edges            H/graph.hpp:48       -> cd_graph_from_edges
    generate_planted            H/generator.hpp:52   -> cd_graph_generate_planted
    run_plp                     H/plp.hpp:67         -> cd_plp_run
    run_plm / run_plmr          H/louvain.hpp:290/297 -> cd_louvain_run
    run_epp                     H/ensemble.hpp:111   -> cd_epp_run
    modularity / coverage       H/quality.hpp:35/21  -> cd_modularity
    coarsen / prolong           H/louvain.hpp:154/223 -> cd_coarsen / cd_prolong
    compacted / community_count H/partition.hpp:39/55 -> cd_compact / cd_community_count
    combine_hashed              H/ensemble.hpp:86    -> cd_combine_hashed
    move_phase / dominant_label H/louvain.hpp:65, H/plp.hpp:32

Exceptions: ``InputError`` (commdet::input_error), ``InvalidArgument``
(std::invalid_argument, a ValueError), ``DomainError`` (std::domain_error),
``OutOfRange`` (std::out_of_range, an IndexError).

There is no CPU path: importing works anywhere, but every call needs the
built library and a CUDA device, and fails loudly otherwise.
"""
from __future__ import annotations

import ctypes as C
import os
import time
import weakref
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "Context", "Graph", "PlpConfig", "LouvainConfig", "EnsembleConfig", "RunReport",
    "InputError", "InvalidArgument", "DomainError", "OutOfRange", "CudaError",
    "generate_planted", "generate_rmat", "generate_lfr", "run_plp", "run_plm", "run_plmr", "run_epp",
    "run_louvain", "modularity", "coverage", "community_volumes", "coarsen", "prolong", "compacted",
    "community_count", "combine_hashed", "plp_sweep_sync", "move_eval", "move_phase", "move_phase_sequential",
    "dominant_label",
    "is_stable", "library_path", "load_library", "default_context", "ALGO_PLP", "ALGO_PLM", "ALGO_PLMR",
    "LoopbackGroup", "nccl_unique_id", "shard_bounds", "read_metis", "read_edge_list", "graph_rand_index",
]

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_NAME = "libcommdet_cuda.so"
ALGO_PLP, ALGO_PLM, ALGO_PLMR = 0, 1, 2


class CommdetError(RuntimeError):
    pass


class InputError(CommdetError):
    """commdet::input_error (H/graph.hpp:21-24)."""


class InvalidArgument(ValueError):
    """std::invalid_argument."""


class DomainError(ValueError):
    """std::domain_error."""


class OutOfRange(IndexError):
    """std::out_of_range."""


class CudaError(CommdetError):
    pass


# ---------------------------------------------------------------------------
# C ABI structs (mirror include/commdet_cuda.h)
# ---------------------------------------------------------------------------
class _PlpConfig(C.Structure):
    _fields_ = [("theta", C.c_int64), ("max_iterations", C.c_int64), ("randomize_order", C.c_int32),
                ("workers", C.c_int32), ("seed", C.c_uint64), ("buckets", C.c_int32), ("reserved", C.c_int32)]


class _LouvainConfig(C.Structure):
    _fields_ = [("gamma", C.c_double), ("max_move_iterations", C.c_int64), ("max_levels", C.c_int64),
                ("seed", C.c_uint64), ("workers", C.c_int32), ("refine", C.c_int32), ("buckets", C.c_int32),
                ("singleton_guard", C.c_int32), ("move_theta", C.c_int64), ("move_tol", C.c_double),
                ("move_stall", C.c_double), ("prune", C.c_int32), ("reserved", C.c_int32),
                ("move_qtol", C.c_double)]


class _EnsembleConfig(C.Structure):
    _fields_ = [("ensemble_size", C.c_int64), ("base", C.c_int32), ("final_algo", C.c_int32),
                ("seed", C.c_uint64), ("workers", C.c_int32), ("reserved", C.c_int32),
                ("base_plp", _PlpConfig), ("final_louvain", _LouvainConfig)]


class _IterRec(C.Structure):
    _fields_ = [("updated", C.c_int64), ("ms", C.c_double)]


class _LevelRec(C.Structure):
    _fields_ = [("move_ms", C.c_double), ("coarsen_ms", C.c_double), ("refine_ms", C.c_double),
                ("nodes", C.c_int64), ("entries", C.c_int64), ("passes", C.c_int64), ("moves", C.c_int64)]


class _Report(C.Structure):
    _fields_ = [("algorithm", C.c_char * 16), ("workers", C.c_int32), ("reserved", C.c_int32),
                ("seed", C.c_uint64), ("total_ms", C.c_double), ("modularity", C.c_double),
                ("coverage", C.c_double), ("community_count", C.c_int64), ("n_iterations", C.c_int64),
                ("iterations", _IterRec * 1024), ("n_levels", C.c_int64), ("levels", _LevelRec * 64),
                ("base_ms", C.c_double), ("combine_ms", C.c_double), ("coarsen_ms", C.c_double),
                ("final_ms", C.c_double), ("kernel_launches", C.c_int64)]


class _GraphInfo(C.Structure):
    _fields_ = [("n", C.c_int64), ("D", C.c_int64), ("m", C.c_int64), ("total_weight", C.c_double),
                ("weighted", C.c_int32), ("reserved", C.c_int32), ("max_degree", C.c_int64),
                ("isolated", C.c_int64), ("shard_rank", C.c_int32), ("shard_size", C.c_int32),
                ("own_lo", C.c_int64), ("own_hi", C.c_int64), ("D_global", C.c_int64)]


class _LfrSpec(C.Structure):
    _fields_ = [("n", C.c_int64), ("tau1", C.c_double), ("avg_degree", C.c_double), ("max_degree", C.c_int32),
                ("tau2", C.c_double), ("min_community", C.c_int32), ("max_community", C.c_int32),
                ("mu", C.c_double)]


class _KStat(C.Structure):
    _fields_ = [("name", C.c_char * 48), ("launches", C.c_int64), ("total_ms", C.c_double),
                ("bytes", C.c_double), ("items", C.c_double)]


_lib = None

# every symbol include/commdet_cuda.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "cd_last_error", "cd_version", "cd_plp_config_default", "cd_louvain_config_default", "cd_louvain_config_reference",
    "cd_ensemble_config_default", "cd_ctx_create", "cd_ctx_destroy", "cd_ctx_synchronize", "cd_ctx_stream",
    "cd_ctx_set_profiling", "cd_ctx_reset_stats", "cd_ctx_kernel_stats", "cd_ctx_launch_count",
    "cd_graph_from_edges", "cd_graph_from_csr", "cd_graph_generate_planted", "cd_graph_generate_rmat",
    "cd_graph_generate_rmat_shard",
    "cd_graph_generate_lfr", "cd_graph_get_info", "cd_graph_download", "cd_graph_destroy", "cd_modularity",
    "cd_community_volumes", "cd_compact", "cd_community_count", "cd_coarsen", "cd_prolong", "cd_combine_hashed",
    "cd_plp_sweep_sync", "cd_move_eval", "cd_move_phase", "cd_move_phase_sequential", "cd_plp_run", "cd_louvain_run",
    "cd_epp_run", "cd_epp_run_bases",
    "cd_nccl_unique_id", "cd_ctx_attach_nccl", "cd_loopback_create", "cd_loopback_destroy",
    "cd_ctx_attach_loopback", "cd_ctx_detach", "cd_ctx_world", "cd_shard_bounds", "cd_graph_shard", "cd_graph_from_csr_rows",
    "cd_graph_read_metis", "cd_graph_read_edge_list", "cd_graph_load_metis", "cd_graph_load_edge_list",
    "cd_graph_original_ids", "cd_rand_index",
]


# MoveObserver (H/louvain.hpp:60) as the C ABI's cd_move_observer
_MoveObserver = C.CFUNCTYPE(None, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_double)


def library_path() -> str:
    return os.path.join(HERE, _LIB_NAME)


def load_library():
    """Load libcommdet_cuda.so (in-tree).  Raises if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    # COMMDET_CUDA_LIB: an alternative build of the same library (A/B timing)
    path = os.environ.get("COMMDET_CUDA_LIB") or library_path()
    if not os.path.exists(path):
        raise CommdetError(f"{path} is missing: build it with `make lib` (or __graft_entry__.build())")
    L = C.CDLL(path)
    vp, vpp = C.c_void_p, C.POINTER(C.c_void_p)
    i64, i32, f64 = C.c_int64, C.c_int32, C.c_double
    L.cd_last_error.restype = C.c_char_p
    L.cd_version.restype = C.c_char_p
    sig = {
        "cd_ctx_create": [C.c_int, vpp], "cd_ctx_destroy": [vp], "cd_ctx_synchronize": [vp],
        "cd_ctx_stream": [vp, vpp], "cd_ctx_set_profiling": [vp, C.c_int], "cd_ctx_reset_stats": [vp],
        "cd_ctx_kernel_stats": [vp, vp, i32, C.POINTER(i32)], "cd_ctx_launch_count": [vp, C.POINTER(i64)],
        "cd_graph_from_edges": [vp, i64, i64, vp, vp, vp, i32, vpp],
        "cd_graph_from_csr": [vp, i64, vp, vp, vp, vpp],
        "cd_graph_generate_planted": [vp, i64, i64, f64, f64, C.c_uint64, vpp, vp],
        "cd_graph_generate_rmat": [vp, i32, i32, f64, f64, f64, i32, C.c_uint64, vpp],
        "cd_graph_generate_rmat_shard": [vp, i32, i32, f64, f64, f64, i32, C.c_uint64, vpp],
        "cd_graph_generate_lfr": [vp, C.POINTER(_LfrSpec), C.c_uint64, vpp, vp],
        "cd_graph_get_info": [vp, C.POINTER(_GraphInfo)], "cd_graph_download": [vp, vp, vp, vp, vp, vp],
        "cd_graph_destroy": [vp],
        "cd_modularity": [vp, vp, vp, i64, f64, C.POINTER(f64), C.POINTER(f64)],
        "cd_community_volumes": [vp, vp, vp, i64, vp],
        "cd_compact": [vp, i64, vp, vp, C.POINTER(i64)], "cd_community_count": [vp, i64, vp, C.POINTER(i64)],
        "cd_coarsen": [vp, vp, vp, vpp, vp], "cd_prolong": [vp, i64, vp, i64, vp, vp],
        "cd_combine_hashed": [vp, i64, i64, vp, vp, C.POINTER(i64)],
        "cd_plp_sweep_sync": [vp, vp, vp, vp, C.POINTER(i64)],
        "cd_move_eval": [vp, vp, vp, vp, i64, f64, vp, vp],
        "cd_move_phase": [vp, vp, vp, C.POINTER(_LouvainConfig), C.POINTER(i32)],
        "cd_plp_run": [vp, vp, C.POINTER(_PlpConfig), vp, vp, C.POINTER(_Report)],
        "cd_louvain_run": [vp, vp, C.POINTER(_LouvainConfig), vp, C.POINTER(_Report)],
        "cd_epp_run": [vp, vp, C.POINTER(_EnsembleConfig), vp, C.POINTER(_Report)],
        "cd_epp_run_bases": [vp, vp, C.POINTER(_EnsembleConfig), vp, vp, C.POINTER(_Report)],
        "cd_move_phase_sequential": [vp, vp, vp, i64, C.POINTER(_LouvainConfig), _MoveObserver, vp,
                                     C.POINTER(i32)],
        "cd_nccl_unique_id": [vp], "cd_ctx_attach_nccl": [vp, i32, i32, vp],
        "cd_loopback_create": [i32, vpp], "cd_loopback_destroy": [vp], "cd_ctx_attach_loopback": [vp, vp, i32],
        "cd_ctx_detach": [vp], "cd_ctx_world": [vp, C.POINTER(i32), C.POINTER(i32)],
        "cd_shard_bounds": [i64, vp, i32, vp], "cd_graph_shard": [vp, vp, vpp],
        "cd_graph_from_csr_rows": [vp, i64, vp, i64, i64, vp, vp, vpp],
        "cd_graph_read_metis": [vp, vp, i64, vpp], "cd_graph_read_edge_list": [vp, vp, i64, i32, vpp],
        "cd_graph_load_metis": [vp, C.c_char_p, vpp], "cd_graph_load_edge_list": [vp, C.c_char_p, i32, vpp],
        "cd_graph_original_ids": [vp, vp], "cd_rand_index": [vp, vp, vp, vp, C.POINTER(f64)],
    }
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = C.c_int
    L.cd_plp_config_default.argtypes = [C.POINTER(_PlpConfig)]
    L.cd_plp_config_default.restype = None
    L.cd_louvain_config_default.argtypes = [C.POINTER(_LouvainConfig)]
    L.cd_louvain_config_default.restype = None
    L.cd_louvain_config_reference.argtypes = [C.POINTER(_LouvainConfig)]
    L.cd_louvain_config_reference.restype = None
    L.cd_ensemble_config_default.argtypes = [C.POINTER(_EnsembleConfig)]
    L.cd_ensemble_config_default.restype = None
    _lib = L
    return L


_ERR = {1: InvalidArgument, 2: DomainError, 3: OutOfRange, 4: InputError, 5: MemoryError, 6: CudaError,
        7: CudaError, 8: CommdetError}


def _check(rc):
    if rc != 0:
        msg = load_library().cd_last_error().decode(errors="replace")
        raise _ERR.get(rc, CommdetError)(msg)


# ---------------------------------------------------------------------------
# context
# ---------------------------------------------------------------------------
class Context:
    """One CUDA device + stream + memory pool (cd_ctx).  Not thread-safe."""

    def __init__(self, device: int = 0):
        L = load_library()
        h = C.c_void_p()
        _check(L.cd_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device
        self._graphs = weakref.WeakValueDictionary()  # id -> Graph living on this context's pool

    def close(self):
        if getattr(self, "h", None):
            for g in list(self._graphs.values()):  # a graph must not outlive its context
                g._release()
            load_library().cd_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self):
        _check(load_library().cd_ctx_synchronize(self.h))

    @property
    def stream(self) -> int:
        s = C.c_void_p()
        _check(load_library().cd_ctx_stream(self.h, C.byref(s)))
        return s.value or 0

    def set_profiling(self, on: bool):
        _check(load_library().cd_ctx_set_profiling(self.h, int(on)))

    def reset_stats(self):
        _check(load_library().cd_ctx_reset_stats(self.h))

    def kernel_stats(self) -> dict:
        L = load_library()
        cnt = C.c_int32()
        _check(L.cd_ctx_kernel_stats(self.h, None, 0, C.byref(cnt)))
        arr = (_KStat * max(cnt.value, 1))()
        _check(L.cd_ctx_kernel_stats(self.h, arr, cnt.value, C.byref(cnt)))
        return {arr[i].name.decode(): dict(launches=arr[i].launches, total_ms=arr[i].total_ms,
                                           bytes=arr[i].bytes, items=arr[i].items) for i in range(cnt.value)}

    def launch_count(self) -> int:
        c = C.c_int64()
        _check(load_library().cd_ctx_launch_count(self.h, C.byref(c)))
        return c.value

    # ---- sharded execution ----------------------------------
    def attach_nccl(self, nranks: int, rank: int, unique_id: bytes):
        """Join an NCCL communicator (one rank per GPU); collective over the ranks."""
        uid = (C.c_uint8 * 128).from_buffer_copy(bytes(unique_id))
        _check(load_library().cd_ctx_attach_nccl(self.h, nranks, rank, uid))

    def attach_loopback(self, group: "LoopbackGroup", rank: int):
        """Join an in-process loopback group (ranks = host threads on one device)."""
        _check(load_library().cd_ctx_attach_loopback(self.h, group.h, rank))
        self._group = group

    def detach(self):
        _check(load_library().cd_ctx_detach(self.h))
        self._group = None

    @property
    def world(self):
        r, n = C.c_int32(), C.c_int32()
        _check(load_library().cd_ctx_world(self.h, C.byref(r), C.byref(n)))
        return r.value, n.value


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(load_library().cd_nccl_unique_id(buf))
    return bytes(buf)


class LoopbackGroup:
    """In-process emulation of `nranks` ranks on one device (cd_loopback)."""

    def __init__(self, nranks: int):
        h = C.c_void_p()
        _check(load_library().cd_loopback_create(nranks, C.byref(h)))
        self.h = h
        self.nranks = nranks

    def __del__(self):
        try:
            if getattr(self, "h", None):
                load_library().cd_loopback_destroy(self.h)
                self.h = None
        except Exception:
            pass


def shard_bounds(off, nranks: int):
    """Ownership ranges of `nranks` ranks over CSR offsets `off` (host)."""
    off = np.ascontiguousarray(np.asarray(off), dtype=np.int64)
    n = off.shape[0] - 1
    out = np.zeros(nranks + 1, dtype=np.int64)
    _check(load_library().cd_shard_bounds(n, off.ctypes.data, nranks, out.ctypes.data))
    return out


_default_ctx = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


def _ctx(ctx):
    return ctx if ctx is not None else default_context()


# ---------------------------------------------------------------------------
# array helpers: numpy (host) or anything exposing a CUDA data_ptr (device)
# ---------------------------------------------------------------------------
def _is_dev(a) -> bool:
    return hasattr(a, "data_ptr") and getattr(a, "is_cuda", False)


def _ptr(a, dtype):
    """Returns (pointer, keepalive) for a host numpy-compatible array or a CUDA tensor."""
    if a is None:
        return None, None
    if _is_dev(a):
        return a.data_ptr(), a
    arr = np.ascontiguousarray(np.asarray(a), dtype=dtype)
    return arr.ctypes.data, arr


# ---------------------------------------------------------------------------
# graphs
# ---------------------------------------------------------------------------
class Graph:
    """Device-resident CSR graph (H/graph.hpp:41).  Immutable after build."""

    def __init__(self, handle, ctx: Context):
        self.h = handle
        self.ctx = ctx
        info = _GraphInfo()
        _check(load_library().cd_graph_get_info(self.h, C.byref(info)))
        self._info = info
        self._host = None
        ctx._graphs[id(self)] = self

    def _release(self):
        if getattr(self, "h", None):
            load_library().cd_graph_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self._release()
        except Exception:
            pass

    # --- construction -------------------------------------------------------
    @classmethod
    def from_edges(cls, n, edges, merge_duplicates=False, ctx=None):
        """Graph::from_edges (H/graph.hpp:48-81).  edges: iterable of (u, v[, w])
        or a tuple of arrays (u, v[, w]).  Weighted iff any weight is given."""
        ctx = _ctx(ctx)
        if isinstance(edges, tuple) and len(edges) in (2, 3) and hasattr(edges[0], "__len__") \
                and not np.isscalar(edges[0]):
            u = np.ascontiguousarray(edges[0], np.int64)
            v = np.ascontiguousarray(edges[1], np.int64)
            w = None if len(edges) == 2 or edges[2] is None else np.ascontiguousarray(edges[2], np.float32)
        else:
            edges = list(edges)
            u = np.array([e[0] for e in edges], np.int64)
            v = np.array([e[1] for e in edges], np.int64)
            ws = [e[2] for e in edges if len(e) > 2]
            w = np.array([float(e[2]) if len(e) > 2 else 1.0 for e in edges], np.float32) if ws else None
        if len(u) and (u.min() < 0 or v.min() < 0 or u.max() >= n or v.max() >= n):
            raise InputError("edge endpoint out of range")
        u32, v32 = u.astype(np.int32), v.astype(np.int32)
        h = C.c_void_p()
        _check(load_library().cd_graph_from_edges(ctx.h, n, len(u32), u32.ctypes.data if len(u32) else None,
                                                  v32.ctypes.data if len(v32) else None,
                                                  None if w is None or not len(w) else w.ctypes.data,
                                                  int(merge_duplicates), C.byref(h)))
        return cls(h, ctx)

    @classmethod
    def from_csr(cls, n, off, col, w=None, ctx=None):
        ctx = _ctx(ctx)
        po, ko = _ptr(off, np.int64)
        pc, kc = _ptr(col, np.int32)
        pw, kw = _ptr(w, np.float32)
        h = C.c_void_p()
        _check(load_library().cd_graph_from_csr(ctx.h, n, po, pc, pw, C.byref(h)))
        return cls(h, ctx)

    @classmethod
    def from_csr_rows(cls, n, off, lo, hi, col_rows, w_rows=None, ctx=None):
        """This rank's row shard from its own rows only (cd_graph_from_csr_rows):
        off = the whole graph's offsets, [lo, hi) = shard_bounds(off, world)[r:r+2],
        col_rows / w_rows = the entries of rows [lo, hi).  Collective."""
        ctx = _ctx(ctx)
        po, ko = _ptr(off, np.int64)
        pc, kc = _ptr(col_rows, np.int32)
        pw, kw = _ptr(w_rows, np.float32)
        h = C.c_void_p()
        _check(load_library().cd_graph_from_csr_rows(ctx.h, n, po, int(lo), int(hi), pc, pw, C.byref(h)))
        return cls(h, ctx)

    # --- reference accessors (H/graph.hpp:105-123) ---------------------------
    def node_count(self) -> int:
        return self._info.n

    def edge_count(self) -> int:
        return self._info.m

    def total_edge_weight(self) -> float:
        return self._info.total_weight

    @property
    def entries(self) -> int:
        return self._info.D

    @property
    def weighted(self) -> bool:
        return bool(self._info.weighted)

    @property
    def max_degree(self) -> int:
        return self._info.max_degree

    @property
    def isolated(self) -> int:
        return self._info.isolated

    # --- sharding --------------------------------------------
    def shard(self, ctx: Context = None) -> "Graph":
        """This rank's row shard (owned rows only) under ctx's communicator."""
        ctx = ctx or self.ctx
        h = C.c_void_p()
        _check(load_library().cd_graph_shard(ctx.h, self.h, C.byref(h)))
        return Graph(h, ctx)

    def original_ids(self):
        """Dense id -> original id of a graph read by read_edge_list."""
        out = np.zeros(max(self.node_count(), 1), np.uint64)
        _check(load_library().cd_graph_original_ids(self.h, out.ctypes.data))
        return out[: self.node_count()]

    @property
    def owned_range(self):
        return self._info.own_lo, self._info.own_hi

    @property
    def is_shard(self) -> bool:
        return self._info.shard_size > 1 or self._info.own_hi - self._info.own_lo < self._info.n

    def csr(self):
        """Host copy: dict(off, col, w (None if unweighted), vol, loop)."""
        if self._host is None:
            n, D = self._info.n, self._info.D
            off = np.zeros(n + 1, np.int64)
            col = np.zeros(max(D, 1), np.int32)
            w = np.zeros(max(D, 1), np.float32) if self.weighted else None
            vol = np.zeros(max(n, 1), np.float64)
            loop = np.zeros(max(n, 1), np.float64)
            _check(load_library().cd_graph_download(self.h, off.ctypes.data, col.ctypes.data,
                                                    None if w is None else w.ctypes.data, vol.ctypes.data,
                                                    loop.ctypes.data))
            self._host = dict(off=off, col=col[:D], w=None if w is None else w[:D], vol=vol[:n], loop=loop[:n])
        return self._host

    def _check_node(self, u):
        if not 0 <= u < self.node_count():
            raise OutOfRange(f"node id {u} out of range")

    def degree(self, u) -> int:
        self._check_node(u)
        off = self.csr()["off"]
        return int(off[u + 1] - off[u])

    def volume(self, u) -> float:
        self._check_node(u)
        return float(self.csr()["vol"][u])

    def loop_weight(self, u) -> float:
        self._check_node(u)
        return float(self.csr()["loop"][u])

    def for_neighbors(self, u):
        c = self.csr()
        s, e = c["off"][u], c["off"][u + 1]
        ws = c["w"][s:e] if c["w"] is not None else np.ones(e - s, np.float32)
        return list(zip(c["col"][s:e].tolist(), ws.tolist()))

    def __eq__(self, other):
        a, b = self.csr(), other.csr()
        wa = a["w"] if a["w"] is not None else np.ones(len(a["col"]), np.float32)
        wb = b["w"] if b["w"] is not None else np.ones(len(b["col"]), np.float32)
        return (np.array_equal(a["off"], b["off"]) and np.array_equal(a["col"], b["col"])
                and np.array_equal(wa, wb))

    __hash__ = None


def generate_planted(n, k, p_in, p_out, seed=1, ctx=None):
    """generate_planted (H/generator.hpp:52-104): bit-exact edge set; returns (Graph, truth)."""
    ctx = _ctx(ctx)
    truth = np.zeros(max(n, 1), np.int32)
    h = C.c_void_p()
    _check(load_library().cd_graph_generate_planted(ctx.h, n, k, p_in, p_out, seed, C.byref(h),
                                                    truth.ctypes.data))
    return Graph(h, ctx), truth[:n]


def generate_rmat(scale, edge_factor=16, a=0.57, b=0.19, c=0.19, weighted=False, seed=1, ctx=None, shard=False):
    """Seeded R-MAT (DESIGN.md generators).  shard=True: collective over the
    context's ranks; this rank's row shard, built without the whole graph."""
    ctx = _ctx(ctx)
    h = C.c_void_p()
    fn = load_library().cd_graph_generate_rmat_shard if shard else load_library().cd_graph_generate_rmat
    _check(fn(ctx.h, scale, edge_factor, a, b, c, int(weighted), seed, C.byref(h)))
    return Graph(h, ctx)


LFR_C2 = dict(n=1_000_000, tau1=2.0, avg_degree=20.0, max_degree=200, tau2=1.0, min_community=20,
              max_community=1000, mu=0.3)


def generate_lfr(seed=1, ctx=None, **spec):
    ctx = _ctx(ctx)
    s = dict(LFR_C2)
    s.update(spec)
    cs = _LfrSpec(**s)
    truth = np.zeros(s["n"], np.int32)
    h = C.c_void_p()
    _check(load_library().cd_graph_generate_lfr(ctx.h, C.byref(cs), seed, C.byref(h), truth.ctypes.data))
    return Graph(h, ctx), truth


# ---------------------------------------------------------------------------
# text ingest (H/io.hpp) -- parsed on the device
# ---------------------------------------------------------------------------
def _text_arg(source):
    if isinstance(source, (bytes, bytearray, memoryview)):
        return bytes(source), None
    if _is_dev(source):
        return source, None
    return None, os.fspath(source)


def read_metis(source, ctx=None) -> Graph:
    """io::read_metis (H/io.hpp:83-165).  `source`: a path, or the file's bytes
    (host bytes or a uint8 CUDA tensor)."""
    ctx = _ctx(ctx)
    data, path = _text_arg(source)
    h = C.c_void_p()
    L = load_library()
    if path is not None:
        _check(L.cd_graph_load_metis(ctx.h, path.encode(), C.byref(h)))
    else:
        ptr = data.data_ptr() if _is_dev(data) else C.cast(C.c_char_p(data), C.c_void_p).value
        n = data.numel() if _is_dev(data) else len(data)
        _check(L.cd_graph_read_metis(ctx.h, ptr, n, C.byref(h)))
    return Graph(h, ctx)


def read_edge_list(source, merge_duplicates=False, ctx=None) -> Graph:
    """io::read_edge_list (H/io.hpp:190-237); `Graph.original_ids()` gives the
    dense -> original id map."""
    ctx = _ctx(ctx)
    data, path = _text_arg(source)
    h = C.c_void_p()
    L = load_library()
    if path is not None:
        _check(L.cd_graph_load_edge_list(ctx.h, path.encode(), int(merge_duplicates), C.byref(h)))
    else:
        ptr = data.data_ptr() if _is_dev(data) else C.cast(C.c_char_p(data), C.c_void_p).value
        n = data.numel() if _is_dev(data) else len(data)
        _check(L.cd_graph_read_edge_list(ctx.h, ptr, n, int(merge_duplicates), C.byref(h)))
    return Graph(h, ctx)


# ---------------------------------------------------------------------------
# configs / reports (H/plp.hpp:16-22, H/louvain.hpp:15-22, H/ensemble.hpp:19-31)
# ---------------------------------------------------------------------------
def _sat64(v):
    """The reference's caps are uint64 counts; the C ABI takes int64: saturate."""
    return min(int(v), (1 << 63) - 1)


@dataclass
class PlpConfig:
    theta: int = -1
    max_iterations: int = 100
    randomize_order: bool = False
    seed: int = 1
    workers: int = 1
    buckets: int = 4

    def _c(self):
        return _PlpConfig(self.theta, _sat64(self.max_iterations), int(self.randomize_order), self.workers, self.seed,
                          self.buckets, 0)


@dataclass
class LouvainConfig:
    gamma: float = 1.0
    max_move_iterations: int = 32
    max_levels: int = 64
    seed: int = 1
    workers: int = 1
    refine: bool = False
    buckets: int = 0           # by graph: 8 if its max degree > 4096, else 4
    singleton_guard: bool = True
    move_theta: int = -1
    move_tol: float = 1e-3
    move_stall: float = 0.95
    prune: int = 1
    move_qtol: float = -1.0    # by graph: 5e-3 if its max degree > 4096, else 2e-3

    @classmethod
    def reference(cls, **kw):
        """The reference's stopping rule alone (cd_louvain_config_reference):
        no early stops, no pruning; buckets and the singleton guard kept."""
        d = dict(move_theta=0, move_tol=0.0, move_stall=0.0, prune=0, move_qtol=0.0)
        d.update(kw)
        return cls(**d)

    def _c(self):
        return _LouvainConfig(self.gamma, _sat64(self.max_move_iterations), _sat64(self.max_levels), self.seed, self.workers,
                              int(self.refine), self.buckets, int(self.singleton_guard), self.move_theta,
                              self.move_tol, self.move_stall, int(self.prune), 0, self.move_qtol)


@dataclass
class EnsembleConfig:
    ensemble_size: int = 4
    base: int = ALGO_PLP
    final_algo: int = ALGO_PLMR
    seed: int = 1
    workers: int = 1
    base_plp: PlpConfig = field(default_factory=lambda: PlpConfig(randomize_order=True))
    final_louvain: LouvainConfig = field(default_factory=LouvainConfig)
    # test hook (H/ensemble.hpp:30): f(g, seed) -> labels, replaces the base detector
    base_override: object = None

    def _c(self):
        return _EnsembleConfig(self.ensemble_size, self.base, self.final_algo, self.seed, self.workers, 0,
                               self.base_plp._c(), self.final_louvain._c())


@dataclass
class RunReport:
    """RunReport (H/report.hpp:26-41)."""
    algorithm: str
    workers: int
    seed: int
    total_ms: float
    modularity: float
    coverage: float
    community_count: int
    iterations: list
    levels: list
    base_ms: float = 0.0
    combine_ms: float = 0.0
    coarsen_ms: float = 0.0
    final_ms: float = 0.0
    kernel_launches: int = 0

    @classmethod
    def _from(cls, r: _Report):
        its = [dict(updated=r.iterations[i].updated, ms=r.iterations[i].ms)
               for i in range(min(r.n_iterations, 1024))]
        lvs = [dict(move_ms=r.levels[i].move_ms, coarsen_ms=r.levels[i].coarsen_ms,
                    refine_ms=r.levels[i].refine_ms, nodes=r.levels[i].nodes, entries=r.levels[i].entries,
                    passes=r.levels[i].passes, moves=r.levels[i].moves)
               for i in range(min(r.n_levels, 64))]
        return cls(r.algorithm.decode(), r.workers, r.seed, r.total_ms, r.modularity, r.coverage,
                   r.community_count, its, lvs, r.base_ms, r.combine_ms, r.coarsen_ms, r.final_ms,
                   r.kernel_launches)

    def to_json(self) -> dict:
        """RunReport::to_json field names (H/report.hpp:42-70)."""
        j = dict(algorithm=self.algorithm, input="", workers=self.workers, seed=self.seed, total_ms=self.total_ms,
                 modularity=self.modularity, coverage=self.coverage, communities=self.community_count)
        if self.levels:
            j["levels"] = [dict(move_ms=l["move_ms"], coarsen_ms=l["coarsen_ms"], refine_ms=l["refine_ms"])
                           for l in self.levels]
        if self.iterations:
            j["iterations"] = self.iterations
        if self.algorithm == "epp":
            j["phases"] = dict(base_ms=self.base_ms, combine_ms=self.combine_ms, coarsen_ms=self.coarsen_ms,
                               final_ms=self.final_ms)
        return j


def _labels_out(g: Graph, out):
    if out is not None:
        return out, (out.data_ptr() if _is_dev(out) else np.asarray(out).ctypes.data)
    arr = np.zeros(max(g.node_count(), 1), np.int32)
    return arr, arr.ctypes.data


def _trim(g, arr):
    return arr[: g.node_count()] if isinstance(arr, np.ndarray) else arr


# ---------------------------------------------------------------------------
# detectors
# ---------------------------------------------------------------------------
def run_plp(g: Graph, cfg: PlpConfig = None, initial=None, out=None, report=True):
    """run_plp (H/plp.hpp:67-149).  Returns (labels, RunReport); labels are raw
    (not compacted).  ``out`` may be a preallocated int32 CUDA tensor."""
    cfg = cfg or PlpConfig()
    if initial is not None and len(initial) != g.node_count():
        raise InvalidArgument("initial partition does not cover the graph")
    pi, ki = _ptr(initial, np.int32)
    labels, lp = _labels_out(g, out)
    rep = _Report()
    c = cfg._c()
    _check(load_library().cd_plp_run(g.ctx.h, g.h, C.byref(c), pi, lp, C.byref(rep) if report else None))
    return _trim(g, labels), (RunReport._from(rep) if report else None)


def run_louvain(g: Graph, cfg: LouvainConfig = None, out=None, report=True):
    """run_plm / run_plmr by cfg.refine.  report=False skips the quality
    evaluation (the reference's total_ms excludes it too) and returns None."""
    cfg = cfg or LouvainConfig()
    z, zp = _labels_out(g, out)
    rep = _Report()
    c = cfg._c()
    _check(load_library().cd_louvain_run(g.ctx.h, g.h, C.byref(c), zp, C.byref(rep) if report else None))
    return _trim(g, z), (RunReport._from(rep) if report else None)


def run_plm(g: Graph, cfg: LouvainConfig = None, out=None):
    """run_plm (H/louvain.hpp:290-295): compacted partition + report."""
    cfg = LouvainConfig(**{**(cfg or LouvainConfig()).__dict__, "refine": False})
    return run_louvain(g, cfg, out)


def run_plmr(g: Graph, cfg: LouvainConfig = None, out=None):
    """run_plmr (H/louvain.hpp:297-301)."""
    cfg = LouvainConfig(**{**(cfg or LouvainConfig()).__dict__, "refine": True})
    return run_louvain(g, cfg, out)


def run_epp(g: Graph, cfg: EnsembleConfig = None, out=None):
    """run_epp (H/ensemble.hpp:111-199).  cfg.base_override, when set, is
    called as f(g, seed + i) for each base (H/ensemble.hpp:30, :127-128) and
    its partitions replace the base detector's runs."""
    cfg = cfg or EnsembleConfig()
    z, zp = _labels_out(g, out)
    rep = _Report()
    c = cfg._c()
    if cfg.base_override is None:
        _check(load_library().cd_epp_run(g.ctx.h, g.h, C.byref(c), zp, C.byref(rep)))
        return _trim(g, z), RunReport._from(rep)
    if cfg.ensemble_size < 1:
        raise InvalidArgument("ensemble size must be >= 1")
    t0 = time.perf_counter()
    bases = [cfg.base_override(g, cfg.seed + i) for i in range(cfg.ensemble_size)]
    base_ms = 1e3 * (time.perf_counter() - t0)
    keep = []
    for b in bases:
        if len(b) != len(bases[0]):
            raise InvalidArgument("ensemble partitions cover different node sets")  # H/ensemble.hpp:33-39
        _check_cover(g, b)
        keep.append(b if _is_dev(b) else np.ascontiguousarray(b, np.int32))
    ptrs = (C.c_void_p * len(keep))(*[b.data_ptr() if _is_dev(b) else b.ctypes.data for b in keep])
    _check(load_library().cd_epp_run_bases(g.ctx.h, g.h, C.byref(c), ptrs, zp, C.byref(rep)))
    r = RunReport._from(rep)
    r.base_ms = base_ms
    r.total_ms += base_ms
    return _trim(g, z), r


# ---------------------------------------------------------------------------
# quality / partitions / sub-kernels
# ---------------------------------------------------------------------------
def _check_cover(g: Graph, z):
    if len(z) != g.node_count():
        raise InvalidArgument(f"partition length {len(z)} does not match node count {g.node_count()}")


def _ub(z, ub):
    if ub is not None:
        return int(ub)
    if _is_dev(z):
        return int(z.max().item()) + 1 if len(z) else 1
    z = np.asarray(z)
    return int(z.max()) + 1 if len(z) else 1


def modularity(g: Graph, z, gamma=1.0, ub=None) -> float:
    """modularity (H/quality.hpp:35-51)."""
    _check_cover(g, z)
    pz, kz = _ptr(z, np.int32)
    q, cov = C.c_double(), C.c_double()
    _check(load_library().cd_modularity(g.ctx.h, g.h, pz, _ub(z, ub), gamma, C.byref(q), C.byref(cov)))
    return q.value


def graph_rand_index(g: Graph, a, b) -> float:
    """graph_rand_index (H/quality.hpp:56-69): fraction of edges on which the
    partitions agree; DomainError for an edgeless graph."""
    _check_cover(g, a)
    _check_cover(g, b)
    pa, ka = _ptr(a, np.int32)
    pb, kb = _ptr(b, np.int32)
    out = C.c_double()
    _check(load_library().cd_rand_index(g.ctx.h, g.h, pa, pb, C.byref(out)))
    return out.value


def coverage(g: Graph, z) -> float:
    """coverage (H/quality.hpp:21-31); 0 for edgeless graphs."""
    _check_cover(g, z)
    if g.total_edge_weight() == 0.0:
        return 0.0
    pz, kz = _ptr(z, np.int32)
    q, cov = C.c_double(), C.c_double()
    _check(load_library().cd_modularity(g.ctx.h, g.h, pz, _ub(z, None), 1.0, C.byref(q), C.byref(cov)))
    return cov.value


def community_volumes(g: Graph, z, ub=None):
    _check_cover(g, z)
    ub = _ub(z, ub)
    pz, kz = _ptr(z, np.int32)
    out = np.zeros(ub, np.float64)
    _check(load_library().cd_community_volumes(g.ctx.h, g.h, pz, ub, out.ctypes.data))
    return out


def compacted(z, ctx=None):
    """Partition::compacted (H/partition.hpp:39-53): returns (labels, k)."""
    ctx = _ctx(ctx)
    z = np.ascontiguousarray(z, np.int32)
    out = np.zeros(max(len(z), 1), np.int32)
    k = C.c_int64()
    _check(load_library().cd_compact(ctx.h, len(z), z.ctypes.data, out.ctypes.data, C.byref(k)))
    return out[: len(z)], k.value


def community_count(z, ctx=None) -> int:
    ctx = _ctx(ctx)
    z = np.ascontiguousarray(z, np.int32)
    k = C.c_int64()
    _check(load_library().cd_community_count(ctx.h, len(z), z.ctypes.data, C.byref(k)))
    return k.value


def coarsen(g: Graph, z):
    """coarsen (H/louvain.hpp:154-220): returns (coarse Graph, pi)."""
    _check_cover(g, z)
    pz, kz = _ptr(z, np.int32)
    pi = np.zeros(max(g.node_count(), 1), np.int32)
    h = C.c_void_p()
    _check(load_library().cd_coarsen(g.ctx.h, g.h, pz, C.byref(h), pi.ctypes.data))
    return Graph(h, g.ctx), pi[: g.node_count()]


def prolong(z_coarse, pi, ctx=None):
    """prolong (H/louvain.hpp:223-233)."""
    ctx = _ctx(ctx)
    zc = np.ascontiguousarray(z_coarse, np.int32)
    pi = np.ascontiguousarray(pi, np.int32)
    out = np.zeros(max(len(pi), 1), np.int32)
    _check(load_library().cd_prolong(ctx.h, len(zc), zc.ctypes.data if len(zc) else None, len(pi),
                                     pi.ctypes.data if len(pi) else None, out.ctypes.data))
    return out[: len(pi)]


def combine_hashed(solutions, ctx=None):
    """combine_hashed (H/ensemble.hpp:86-107): returns (core labels, k)."""
    ctx = _ctx(ctx)
    if len(solutions) == 0:
        raise InvalidArgument("empty ensemble")
    sols = [np.ascontiguousarray(s, np.int32) for s in solutions]
    if any(len(s) != len(sols[0]) for s in sols):
        raise InvalidArgument("ensemble partitions cover different node sets")
    n = len(sols[0])
    ptrs = (C.c_void_p * len(sols))(*[s.ctypes.data for s in sols])
    out = np.zeros(max(n, 1), np.int32)
    k = C.c_int64()
    _check(load_library().cd_combine_hashed(ctx.h, len(sols), n, ptrs, out.ctypes.data, C.byref(k)))
    return out[:n], k.value


def plp_sweep_sync(g: Graph, z_in, out=None):
    """One synchronous PLP sweep (dominant_label of every non-isolated node)."""
    _check_cover(g, z_in)
    pz, kz = _ptr(z_in, np.int32)
    z, zp = _labels_out(g, out)
    upd = C.c_int64()
    _check(load_library().cd_plp_sweep_sync(g.ctx.h, g.h, pz, zp, C.byref(upd)))
    return _trim(g, z), upd.value


def move_eval(g: Graph, z, vols, gamma=1.0):
    """Synchronous move evaluation (H/louvain.hpp:91-120 rule): (best, gain)."""
    _check_cover(g, z)
    pz, kz = _ptr(z, np.int32)
    vols = np.ascontiguousarray(vols, np.float64)
    best = np.zeros(max(g.node_count(), 1), np.int32)
    gain = np.zeros(max(g.node_count(), 1), np.float64)
    _check(load_library().cd_move_eval(g.ctx.h, g.h, pz, vols.ctypes.data, len(vols), gamma, best.ctypes.data,
                                       gain.ctypes.data))
    return best[: g.node_count()], gain[: g.node_count()]


def move_phase(g: Graph, z, cfg: LouvainConfig = None):
    """move_phase (H/louvain.hpp:65-141) with the bucketed device order: (z, changed)."""
    cfg = cfg or LouvainConfig()
    _check_cover(g, z)
    z = np.array(z, np.int32, copy=True)
    ch = C.c_int32()
    c = cfg._c()
    _check(load_library().cd_move_phase(g.ctx.h, g.h, z.ctypes.data if len(z) else None, C.byref(c),
                                        C.byref(ch)))
    return z, bool(ch.value)


def move_phase_sequential(g: Graph, z, cfg: LouvainConfig = None, observer=None, ub=None):
    """move_phase (H/louvain.hpp:65-141) in the reference's one-worker order
    (u = 0..n-1, each move applied before the next node): returns (z, changed).
    Like the reference's ``Partition &z``, a contiguous int32 numpy ``z`` is
    updated in place.  observer(u, source, target, gain) is the MoveObserver
    (:60, :127-128): each call comes after ``z[u] = target``, so an observer
    holding ``z`` sees the partition right after that move.  Only cfg.gamma
    and cfg.max_move_iterations are read."""
    cfg = cfg or LouvainConfig()
    _check_cover(g, z)
    if not (isinstance(z, np.ndarray) and z.dtype == np.int32 and z.flags.c_contiguous and z.flags.writeable):
        z = np.array(z, np.int32, copy=True)
    ub = int(ub) if ub is not None else max(int(z.max()) + 1 if len(z) else 1, 1)
    dz = z.copy()  # the device's in/out copy; z itself follows the replayed moves
    err = []

    def trampoline(_user, u, c, d, gain):
        if err:
            return
        try:
            z[u] = d
            observer(u, c, d, gain)
        except BaseException as e:  # noqa: BLE001 -- re-raised after the call
            err.append(e)

    cb = _MoveObserver(trampoline) if observer is not None else _MoveObserver()
    ch = C.c_int32()
    c = cfg._c()
    _check(load_library().cd_move_phase_sequential(g.ctx.h, g.h, dz.ctypes.data if len(dz) else None, ub,
                                                   C.byref(c), cb, None, C.byref(ch)))
    if err:
        raise err[0]
    z[:] = dz
    return z, bool(ch.value)


def dominant_label(g: Graph, z, u) -> int:
    """dominant_label (H/plp.hpp:32-53); isolated -> InvalidArgument."""
    if g.degree(u) == 0:
        raise InvalidArgument(f"dominant_label: node {u} is isolated")
    out, _ = plp_sweep_sync(g, z)
    return int(out[u])


def is_stable(g: Graph, z) -> bool:
    """is_stable (H/plp.hpp:57-62)."""
    out, upd = plp_sweep_sync(g, z)
    return upd == 0
