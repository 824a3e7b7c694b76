"""ctypes front end of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference legs) may import this module, and only as the checker.
The product package (paper_1304_4453_b200) never imports it.

Two libraries:
  * ``libcommdet_oracle.so`` (oracle/commdet_oracle.c): plain-C restatement
    of the reference path plus ports of the device's bucketed update order
    and synthetic generators.
  * ``_ref/libcommdet_ref.so`` (oracle/ref_capi.cpp): the unmodified
    reference headers (/root/reference/proj/include/commdet) behind a C ABI.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_REF = None

i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


class _CGraph(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("D", C.c_int64), ("m", C.c_int64), ("total", C.c_double),
        ("off", C.POINTER(C.c_int64)), ("col", C.POINTER(C.c_int32)), ("w", C.POINTER(C.c_double)),
        ("vol", C.POINTER(C.c_double)), ("loop", C.POINTER(C.c_double)),
    ]


class _LfrSpec(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("tau1", C.c_double), ("avg_degree", C.c_double), ("max_degree", C.c_int32),
        ("tau2", C.c_double), ("min_community", C.c_int32), ("max_community", C.c_int32), ("mu", C.c_double),
    ]


class _PlpCfg(C.Structure):
    _fields_ = [("theta", C.c_int64), ("max_iterations", C.c_int64), ("seed", C.c_uint64), ("buckets", C.c_int32)]


class _LouvainCfg(C.Structure):
    _fields_ = [
        ("gamma", C.c_double), ("max_move_iterations", C.c_int64), ("max_levels", C.c_int64),
        ("seed", C.c_uint64), ("buckets", C.c_int32), ("refine", C.c_int32), ("singleton_guard", C.c_int32),
        ("move_theta", C.c_int64), ("move_tol", C.c_double), ("move_stall", C.c_double), ("prune", C.c_int32),
        ("move_qtol", C.c_double),
    ]


class _RefReport(C.Structure):
    _fields_ = [
        ("total_ms", C.c_double), ("modularity", C.c_double), ("coverage", C.c_double),
        ("community_count", C.c_int64), ("iterations", C.c_int64), ("levels", C.c_int64),
        ("base_ms", C.c_double), ("combine_ms", C.c_double), ("coarsen_ms", C.c_double), ("final_ms", C.c_double),
    ]


class OracleError(RuntimeError):
    pass


class OracleInputError(OracleError):
    """commdet::input_error"""


class OracleInvalidArgument(OracleError, ValueError):
    """std::invalid_argument"""


class OracleDomainError(OracleError, ValueError):
    """std::domain_error"""


class OracleOutOfRange(OracleError, IndexError):
    """std::out_of_range"""


_CODES = {-1: "input_error", -2: "invalid_argument", -3: "domain_error", -4: "out_of_range", -5: "ENOMEM"}
_EXC = {-1: OracleInputError, -2: OracleInvalidArgument, -3: OracleDomainError, -4: OracleOutOfRange}


def _check(rc):
    if rc < 0:
        raise _EXC.get(rc, OracleError)(_CODES.get(rc, f"error {rc}"))
    return rc


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "libcommdet_oracle.so")
        if not os.path.exists(path):
            raise OracleError("oracle not built: run `make -C oracle`")
        L = C.CDLL(path)
        gp = C.POINTER(_CGraph)
        L.cdo_graph_free.argtypes = [gp]
        L.cdo_graph_from_edges.argtypes = [C.c_int64, C.c_int64, i32p, i32p, C.c_void_p, C.c_int, gp]
        L.cdo_graph_from_csr.argtypes = [C.c_int64, i64p, i32p, C.c_void_p, gp]
        L.cdo_generate_planted.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_uint64, gp, C.c_void_p]
        L.cdo_generate_rmat.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_int, C.c_uint64, gp]
        L.cdo_generate_lfr.argtypes = [C.POINTER(_LfrSpec), C.c_uint64, gp, C.c_void_p]
        L.cdo_splitmix64.argtypes = [C.c_uint64]
        L.cdo_splitmix64.restype = C.c_uint64
        L.cdo_modularity.argtypes = [gp, i32p, C.c_int64, C.c_double, C.POINTER(C.c_double)]
        L.cdo_coverage.argtypes = [gp, i32p]
        L.cdo_coverage.restype = C.c_double
        L.cdo_community_volumes.argtypes = [gp, i32p, C.c_int64, f64p]
        L.cdo_compact.argtypes = [C.c_int64, i32p, i32p]
        L.cdo_compact.restype = C.c_int64
        L.cdo_community_count.argtypes = [C.c_int64, i32p]
        L.cdo_community_count.restype = C.c_int64
        L.cdo_dominant_label.argtypes = [gp, i32p, C.c_int32, C.POINTER(C.c_int32)]
        L.cdo_plp_sweep_sync.argtypes = [gp, i32p, i32p]
        L.cdo_plp_sweep_sync.restype = C.c_int64
        L.cdo_is_stable.argtypes = [gp, i32p]
        L.cdo_delta_mod.argtypes = [gp, i32p, f64p, C.c_int32, C.c_int32, C.c_double]
        L.cdo_delta_mod.restype = C.c_double
        L.cdo_move_eval.argtypes = [gp, i32p, f64p, C.c_int64, C.c_double, i32p, f64p]
        L.cdo_move_eval.restype = None
        L.cdo_coarsen.argtypes = [gp, i32p, gp]
        L.cdo_move_phase_sequential.argtypes = [gp, i32p, C.c_int64, C.c_double, C.c_int64, C.c_void_p,
                                                C.POINTER(C.c_int32)]
        L.cdo_prolong.argtypes = [C.c_int64, i32p, C.c_int64, i32p, i32p]
        L.cdo_djb2.argtypes = [C.c_char_p, C.c_uint64]
        L.cdo_djb2.restype = C.c_uint64
        L.cdo_combine_hashed.argtypes = [C.c_int64, C.c_int64, C.POINTER(C.c_void_p), i32p]
        L.cdo_combine_hashed.restype = C.c_int64
        L.cdo_bucket_key.argtypes = [C.c_uint64, C.c_uint64]
        L.cdo_bucket_key.restype = C.c_uint64
        L.cdo_bucket_of.argtypes = [C.c_uint64, C.c_int32, C.c_int32]
        L.cdo_plp_bucketed.argtypes = [gp, C.POINTER(_PlpCfg), C.c_void_p, i32p, C.POINTER(C.c_int64), i64p,
                                       C.c_int64]
        L.cdo_move_phase_bucketed.argtypes = [gp, i32p, C.POINTER(_LouvainCfg), C.c_uint64, C.POINTER(C.c_int32)]
        L.cdo_louvain_bucketed.argtypes = [gp, C.POINTER(_LouvainCfg), i32p, C.POINTER(C.c_int64),
                                           C.POINTER(C.c_int64)]
        L.cdo_epp_bucketed.argtypes = [gp, C.c_int64, C.c_uint64, C.POINTER(_PlpCfg), C.POINTER(_LouvainCfg), i32p,
                                       C.POINTER(C.c_int64)]
        L.cdo_plp_subsweep.argtypes = [gp, i32p, C.c_void_p, C.c_uint64, C.c_int32, C.c_int32, C.c_int64,
                                       C.c_int64, i32p, i32p]
        L.cdo_plp_subsweep.restype = C.c_int64
        L.cdo_move_subsweep.argtypes = [gp, i32p, f64p, i32p, C.c_void_p, C.POINTER(_LouvainCfg), C.c_uint64,
                                        C.c_int32, C.c_int64, C.c_int64, i32p, i32p, C.POINTER(C.c_longlong)]
        L.cdo_activate.argtypes = [gp, C.c_int64, i32p, C.c_void_p]
        L.cdo_activate.restype = None
        L.cdo_move_subsweep.restype = C.c_int64
        _LIB = L
    return _LIB


def ref_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libcommdet_ref.so"))


def ref():
    global _REF
    if _REF is None:
        path = os.path.join(HERE, "_ref", "libcommdet_ref.so")
        if not os.path.exists(path):
            raise OracleError("reference oracle not built (oracle/_ref/libcommdet_ref.so)")
        R = C.CDLL(path)
        vpp = C.POINTER(C.c_void_p)
        R.ref_last_error.restype = C.c_char_p
        R.ref_graph_free.argtypes = [C.c_void_p]
        R.ref_graph_from_edges.argtypes = [C.c_int64, C.c_int64, i32p, i32p, C.c_void_p, C.c_int, vpp]
        R.ref_graph_from_csr.argtypes = [C.c_int64, i64p, i32p, C.c_void_p, vpp]
        R.ref_graph_info.argtypes = [C.c_void_p] + [C.POINTER(C.c_int64)] * 3 + [C.POINTER(C.c_double)]
        R.ref_graph_csr.argtypes = [C.c_void_p, i64p, i32p, f64p, f64p, f64p]
        R.ref_generate_planted.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_uint64, C.c_int, vpp,
                                           C.c_void_p]
        R.ref_modularity.argtypes = [C.c_void_p, i32p, C.c_int64, C.c_double, C.POINTER(C.c_double),
                                     C.POINTER(C.c_double)]
        R.ref_dominant_label.argtypes = [C.c_void_p, i32p, C.c_int64, C.POINTER(C.c_int32)]
        R.ref_is_stable.argtypes = [C.c_void_p, i32p]
        R.ref_run_plp.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_uint64, C.c_int, C.c_void_p, i32p,
                                  C.POINTER(_RefReport), C.c_void_p, C.c_int64]
        R.ref_run_louvain.argtypes = [C.c_void_p, C.c_double, C.c_int64, C.c_int64, C.c_uint64, C.c_int, C.c_int,
                                      i32p, C.POINTER(_RefReport)]
        R.ref_move_phase.argtypes = [C.c_void_p, i32p, C.c_int64, C.c_double, C.c_int64, C.c_int,
                                     C.POINTER(C.c_int)]
        R.ref_move_phase_log.argtypes = [C.c_void_p, i32p, C.c_int64, C.c_double, C.c_int64, C.c_int, i32p, i32p,
                                         i32p, f64p, C.c_void_p, C.c_int64, C.POINTER(C.c_int64),
                                         C.POINTER(C.c_int)]
        R.ref_delta_mod.argtypes = [C.c_void_p, i32p, C.c_int64, C.c_int64, C.c_int64, C.c_double,
                                    C.POINTER(C.c_double)]
        R.ref_coarsen.argtypes = [C.c_void_p, i32p, C.c_int, vpp, i32p]
        R.ref_compacted.argtypes = [C.c_int64, i32p, i32p]
        R.ref_compacted.restype = C.c_int64
        R.ref_combine_hashed.argtypes = [C.c_int64, C.c_int64, C.POINTER(C.c_void_p), C.c_int, i32p]
        R.ref_combine_exact.argtypes = [C.c_int64, C.c_int64, C.POINTER(C.c_void_p), i32p]
        R.ref_djb2.argtypes = [C.c_char_p, C.c_uint64]
        R.ref_djb2.restype = C.c_uint64
        R.ref_read_metis.argtypes = [C.c_char_p, vpp]
        R.ref_write_metis.argtypes = [C.c_void_p, C.c_char_p]
        R.ref_write_partition.argtypes = [C.c_int64, i32p, C.c_char_p]
        R.ref_write_community_graph.argtypes = [C.c_void_p, i32p, C.c_char_p]
        R.ref_graph_rand_index.argtypes = [C.c_void_p, i32p, i32p, C.POINTER(C.c_double)]
        R.ref_read_edge_list.argtypes = [C.c_char_p, C.c_int, vpp, C.c_void_p, C.c_int64]
        R.ref_run_epp.argtypes = [C.c_void_p, C.c_int64, C.c_uint64, C.c_int, i32p, C.POINTER(_RefReport)]
        R.ref_max_threads.restype = C.c_int
        _REF = R
    return _REF


def _rcheck(rc):
    if rc != 0:
        msg = ref().ref_last_error().decode(errors="replace")
        raise _EXC.get(rc, OracleError)(f"{_CODES.get(rc, 'error')}: {msg}")


# --------------------------------------------------------------------------- #
# Graph containers                                                             #
# --------------------------------------------------------------------------- #

@dataclass
class CSR:
    """Host CSR in the reference's conventions (H/graph.hpp:38-40)."""
    n: int
    off: np.ndarray   # int64[n+1]
    col: np.ndarray   # int32[D]
    w: np.ndarray     # float64[D]
    vol: np.ndarray   # float64[n]
    loop: np.ndarray  # float64[n]
    m: int
    total: float

    @property
    def D(self) -> int:
        return int(self.off[-1])


def _take(g: _CGraph) -> CSR:
    n, D = g.n, g.D
    out = CSR(
        n=n,
        off=np.ctypeslib.as_array(g.off, (n + 1,)).copy(),
        col=np.ctypeslib.as_array(g.col, (max(D, 1),))[:D].copy(),
        w=np.ctypeslib.as_array(g.w, (max(D, 1),))[:D].copy(),
        vol=np.ctypeslib.as_array(g.vol, (max(n, 1),))[:n].copy(),
        loop=np.ctypeslib.as_array(g.loop, (max(n, 1),))[:n].copy(),
        m=g.m, total=g.total,
    )
    lib().cdo_graph_free(C.byref(g))
    return out


class _Borrow:
    """Temporary _CGraph view over a CSR (no ownership)."""

    def __init__(self, g: CSR):
        self.keep = [np.ascontiguousarray(g.off, np.int64), np.ascontiguousarray(g.col, np.int32),
                     np.ascontiguousarray(g.w, np.float64), np.ascontiguousarray(g.vol, np.float64),
                     np.ascontiguousarray(g.loop, np.float64)]
        off, col, w, vol, loop = self.keep
        self.c = _CGraph(g.n, g.D, g.m, g.total,
                         off.ctypes.data_as(C.POINTER(C.c_int64)), col.ctypes.data_as(C.POINTER(C.c_int32)),
                         w.ctypes.data_as(C.POINTER(C.c_double)), vol.ctypes.data_as(C.POINTER(C.c_double)),
                         loop.ctypes.data_as(C.POINTER(C.c_double)))

    @property
    def ref(self):
        return C.byref(self.c)


def _i32(a):
    return np.ascontiguousarray(np.asarray(a), dtype=np.int32)


def from_edges(n, edges, merge_duplicates=False) -> CSR:
    """Graph::from_edges (H/graph.hpp:48-81). edges: iterable of (u, v[, w])."""
    edges = list(edges)
    eu = _i32([e[0] for e in edges]) if edges else np.zeros(0, np.int32)
    ev = _i32([e[1] for e in edges]) if edges else np.zeros(0, np.int32)
    ew = np.ascontiguousarray([float(e[2]) if len(e) > 2 else 1.0 for e in edges], np.float64)
    g = _CGraph()
    _check(lib().cdo_graph_from_edges(n, len(edges), eu, ev, ew.ctypes.data if len(edges) else None,
                                      int(merge_duplicates), C.byref(g)))
    return _take(g)


def from_arrays(n, eu, ev, ew=None, merge_duplicates=False) -> CSR:
    eu, ev = _i32(eu), _i32(ev)
    w = None if ew is None else np.ascontiguousarray(ew, np.float64)
    g = _CGraph()
    _check(lib().cdo_graph_from_edges(n, len(eu), eu, ev, None if w is None else w.ctypes.data,
                                      int(merge_duplicates), C.byref(g)))
    return _take(g)


def from_csr(n, off, col, w=None) -> CSR:
    off = np.ascontiguousarray(off, np.int64)
    col = _i32(col)
    wa = None if w is None else np.ascontiguousarray(w, np.float64)
    g = _CGraph()
    _check(lib().cdo_graph_from_csr(n, off, col, None if wa is None else wa.ctypes.data, C.byref(g)))
    return _take(g)


def generate_planted(n, k, p_in, p_out, seed):
    g = _CGraph()
    truth = np.zeros(max(n, 1), np.int32)
    _check(lib().cdo_generate_planted(n, k, p_in, p_out, seed, C.byref(g), truth.ctypes.data))
    return _take(g), truth[:n]


def generate_rmat(scale, edge_factor=16, a=0.57, b=0.19, c=0.19, weighted=False, seed=1) -> CSR:
    g = _CGraph()
    _check(lib().cdo_generate_rmat(scale, edge_factor, a, b, c, int(weighted), seed, C.byref(g)))
    return _take(g)


LFR_C2 = dict(n=1_000_000, tau1=2.0, avg_degree=20.0, max_degree=200, tau2=1.0, min_community=20,
              max_community=1000, mu=0.3)


def generate_lfr(seed=1, **spec):
    s = dict(LFR_C2)
    s.update(spec)
    cs = _LfrSpec(**s)
    g = _CGraph()
    truth = np.zeros(s["n"], np.int32)
    _check(lib().cdo_generate_lfr(C.byref(cs), seed, C.byref(g), truth.ctypes.data))
    return _take(g), truth


def splitmix64(x):
    return lib().cdo_splitmix64(x)


# --------------------------------------------------------------------------- #
# quality / partition                                                          #
# --------------------------------------------------------------------------- #

def modularity(g: CSR, z, gamma=1.0, ub=None) -> float:
    z = _i32(z)
    ub = int(z.max()) + 1 if ub is None else ub
    q = C.c_double()
    b = _Borrow(g)
    _check(lib().cdo_modularity(b.ref, z, max(ub, 1), gamma, C.byref(q)))
    return q.value


def coverage(g: CSR, z) -> float:
    return lib().cdo_coverage(_Borrow(g).ref, _i32(z))


def community_volumes(g: CSR, z, ub=None):
    z = _i32(z)
    ub = int(z.max()) + 1 if ub is None else ub
    out = np.zeros(ub, np.float64)
    lib().cdo_community_volumes(_Borrow(g).ref, z, ub, out)
    return out


def compact(z):
    z = _i32(z)
    out = np.zeros_like(z)
    k = lib().cdo_compact(len(z), z, out)
    return out, k


def community_count(z):
    z = _i32(z)
    return lib().cdo_community_count(len(z), z)


def dominant_label(g: CSR, z, u) -> int:
    out = C.c_int32()
    _check(lib().cdo_dominant_label(_Borrow(g).ref, _i32(z), u, C.byref(out)))
    return out.value


def plp_sweep_sync(g: CSR, z):
    z = _i32(z)
    out = np.zeros_like(z)
    upd = lib().cdo_plp_sweep_sync(_Borrow(g).ref, z, out)
    _check(upd)
    return out, upd


def is_stable(g: CSR, z) -> bool:
    return bool(lib().cdo_is_stable(_Borrow(g).ref, _i32(z)))


def delta_mod(g: CSR, z, vols, u, target, gamma=1.0):
    return lib().cdo_delta_mod(_Borrow(g).ref, _i32(z), np.ascontiguousarray(vols, np.float64), u, target, gamma)


def move_eval(g: CSR, z, vols, gamma=1.0):
    z = _i32(z)
    vols = np.ascontiguousarray(vols, np.float64)
    best = np.zeros_like(z)
    gain = np.zeros(len(z), np.float64)
    lib().cdo_move_eval(_Borrow(g).ref, z, vols, len(vols), gamma, best, gain)
    return best, gain


class _MoveLog(C.Structure):
    _fields_ = [("node", C.c_void_p), ("source", C.c_void_p), ("target", C.c_void_p), ("gain", C.c_void_p),
                ("capacity", C.c_int64), ("count", C.c_int64)]


def move_phase_sequential(g: CSR, z, gamma=1.0, max_move_iterations=32, ub=None):
    """move_phase with one worker (H/louvain.hpp:65-141): (z, changed, moves[(u, c, d, gain)])."""
    z = _i32(z).copy()
    ub = int(ub) if ub is not None else max(int(z.max()) + 1 if len(z) else 1, 1)
    cap = max(len(z), 1) * max(int(max_move_iterations), 1)
    lu, lc, ld = (np.zeros(cap, np.int32) for _ in range(3))
    lg = np.zeros(cap, np.float64)
    log = _MoveLog(lu.ctypes.data, lc.ctypes.data, ld.ctypes.data, lg.ctypes.data, cap, 0)
    ch = C.c_int32()
    _check(lib().cdo_move_phase_sequential(_Borrow(g).ref, z, ub, gamma, max_move_iterations, C.byref(log),
                                           C.byref(ch)))
    k = min(log.count, cap)
    return z, bool(ch.value), list(zip(lu[:k].tolist(), lc[:k].tolist(), ld[:k].tolist(), lg[:k].tolist()))


def coarsen(g: CSR, z) -> CSR:
    out = _CGraph()
    _check(lib().cdo_coarsen(_Borrow(g).ref, _i32(z), C.byref(out)))
    return _take(out)


def prolong(zc, pi):
    zc, pi = _i32(zc), _i32(pi)
    out = np.zeros_like(pi)
    _check(lib().cdo_prolong(len(zc), zc, len(pi), pi, out))
    return out


def djb2(data: bytes) -> int:
    return lib().cdo_djb2(data, len(data))


def combine_hashed(solutions):
    """H/ensemble.hpp:86-107 incl. check_ensemble_lengths (:33-39)."""
    sols = [_i32(s) for s in solutions]
    if not sols or any(len(s) != len(sols[0]) for s in sols):
        raise OracleInvalidArgument("empty ensemble or partitions of different lengths")
    n = len(sols[0])
    ptrs = (C.c_void_p * len(sols))(*[s.ctypes.data for s in sols])
    out = np.zeros(n, np.int32)
    k = lib().cdo_combine_hashed(len(sols), n, ptrs, out)
    _check(k)
    return out, k


# --------------------------------------------------------------------------- #
# ports of the device drivers                                                  #
# --------------------------------------------------------------------------- #

def bucket_key(seed, salt):
    return lib().cdo_bucket_key(seed, salt)


def bucket_of(key, u, buckets):
    return lib().cdo_bucket_of(key, u, buckets)


def plp_bucketed(g: CSR, theta=-1, max_iterations=100, seed=1, buckets=4, initial=None):
    cfg = _PlpCfg(theta, max_iterations, seed, buckets)
    labels = np.zeros(g.n, np.int32)
    iters = C.c_int64()
    trace = np.zeros(max(max_iterations, 1), np.int64)
    init = None if initial is None else _i32(initial)
    _check(lib().cdo_plp_bucketed(_Borrow(g).ref, C.byref(cfg), None if init is None else init.ctypes.data,
                                  labels, C.byref(iters), trace, len(trace)))
    return labels, trace[: iters.value].copy()


def louvain_cfg(gamma=1.0, max_move_iterations=32, max_levels=64, seed=1, buckets=0, refine=False,
                singleton_guard=True, move_theta=-1, move_tol=1e-3, move_stall=0.95, prune=True, move_qtol=-1.0):
    """buckets 0 / move_qtol < 0: by graph (8 / 5e-3 when max degree > 4096, else 4 / 2e-3)."""
    return _LouvainCfg(gamma, max_move_iterations, max_levels, seed, buckets, int(refine), int(singleton_guard),
                       move_theta, move_tol, move_stall, int(prune), move_qtol)


def move_phase_bucketed(g: CSR, z, salt=0, **kw):
    z = _i32(z).copy()
    cfg = louvain_cfg(**kw)
    ch = C.c_int32()
    _check(lib().cdo_move_phase_bucketed(_Borrow(g).ref, z, C.byref(cfg), salt, C.byref(ch)))
    return z, bool(ch.value)


def louvain_bucketed(g: CSR, **kw):
    cfg = louvain_cfg(**kw)
    z = np.zeros(g.n, np.int32)
    k, lv = C.c_int64(), C.c_int64()
    _check(lib().cdo_louvain_bucketed(_Borrow(g).ref, C.byref(cfg), z, C.byref(k), C.byref(lv)))
    return z, k.value, lv.value


def epp_bucketed(g: CSR, ensemble_size=4, seed=1, theta=-1, max_iterations=100, buckets=4, **kw):
    base = _PlpCfg(theta, max_iterations, seed, buckets)
    fc = louvain_cfg(**kw)  # the final solver's own schedule (by the core graph)
    z = np.zeros(g.n, np.int32)
    k = C.c_int64()
    _check(lib().cdo_epp_bucketed(_Borrow(g).ref, ensemble_size, seed, C.byref(base), C.byref(fc), z, C.byref(k)))
    return z, k.value


def activate(g: CSR, moved_nodes, active):
    """Activation after a sub-sweep's moves (cdo_activate)."""
    mu = _i32(moved_nodes)
    lib().cdo_activate(_Borrow(g).ref, len(mu), mu, active.ctypes.data)


def plp_subsweep(g: CSR, labels, active, key, bucket, buckets, lo, hi):
    """One sharded-protocol PLP sub-sweep over [lo, hi): returns the moves
    (node, label) and deactivates non-movers in `active` (uint8, in place)."""
    mu = np.zeros(max(hi - lo, 1), np.int32)
    ml = np.zeros(max(hi - lo, 1), np.int32)
    assert active.dtype == np.uint8 and active.flags.c_contiguous
    nm = lib().cdo_plp_subsweep(_Borrow(g).ref, _i32(labels), active.ctypes.data, key, bucket, buckets, lo, hi,
                                mu, ml)
    if nm < 0:
        _check(int(nm))
    return mu[:nm].copy(), ml[:nm].copy()


def move_subsweep(g: CSR, z, vols, csize, active, key, bucket, lo, hi, **kw):
    """`active` (uint8, in place) is used when pruning (kw prune, default on)."""
    cfg = louvain_cfg(**kw)
    mu = np.zeros(max(hi - lo, 1), np.int32)
    ml = np.zeros(max(hi - lo, 1), np.int32)
    assert active.dtype == np.uint8 and active.flags.c_contiguous
    gfx = C.c_longlong()
    nm = lib().cdo_move_subsweep(_Borrow(g).ref, _i32(z), np.ascontiguousarray(vols, np.float64), _i32(csize),
                                 active.ctypes.data, C.byref(cfg), key, bucket, lo, hi, mu, ml, C.byref(gfx))
    if nm < 0:
        _check(int(nm))
    return mu[:nm].copy(), ml[:nm].copy(), gfx.value


# --------------------------------------------------------------------------- #
# the unmodified reference (oracle/_ref)                                       #
# --------------------------------------------------------------------------- #

class RefGraph:
    """A reference commdet::Graph built through Graph::from_edges."""

    def __init__(self, handle):
        self.h = C.c_void_p(handle)

    @classmethod
    def from_csr(cls, g: CSR):
        h = C.c_void_p()
        _rcheck(ref().ref_graph_from_csr(g.n, np.ascontiguousarray(g.off, np.int64), _i32(g.col),
                                         np.ascontiguousarray(g.w, np.float64).ctypes.data, C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_edges(cls, n, edges, merge_duplicates=False):
        edges = list(edges)
        eu = _i32([e[0] for e in edges]) if edges else np.zeros(0, np.int32)
        ev = _i32([e[1] for e in edges]) if edges else np.zeros(0, np.int32)
        ew = np.ascontiguousarray([float(e[2]) if len(e) > 2 else 1.0 for e in edges], np.float64)
        h = C.c_void_p()
        _rcheck(ref().ref_graph_from_edges(n, len(edges), eu, ev, ew.ctypes.data if edges else None,
                                           int(merge_duplicates), C.byref(h)))
        return cls(h.value)

    @classmethod
    def planted(cls, n, k, p_in, p_out, seed, workers=0):
        h = C.c_void_p()
        truth = np.zeros(max(n, 1), np.int32)
        _rcheck(ref().ref_generate_planted(n, k, p_in, p_out, seed, workers, C.byref(h), truth.ctypes.data))
        return cls(h.value), truth[:n]

    @classmethod
    def read_metis(cls, path):
        """io::read_metis (H/io.hpp:83) on a file."""
        h = C.c_void_p()
        _rcheck(ref().ref_read_metis(str(path).encode(), C.byref(h)))
        return cls(h.value)

    @classmethod
    def read_edge_list(cls, path, merge_duplicates=False, max_ids=1 << 20):
        """io::read_edge_list (H/io.hpp:190) on a file: (RefGraph, original ids)."""
        h = C.c_void_p()
        ids = np.zeros(max_ids, np.uint64)
        _rcheck(ref().ref_read_edge_list(str(path).encode(), int(merge_duplicates), C.byref(h), ids.ctypes.data,
                                         max_ids))
        g = cls(h.value)
        return g, ids[: g.info()[0]].copy()

    def write_metis(self, path):
        _rcheck(ref().ref_write_metis(self.h, str(path).encode()))

    def write_community_graph(self, z, path):
        _rcheck(ref().ref_write_community_graph(self.h, _i32(z), str(path).encode()))

    def rand_index(self, a, b):
        out = C.c_double()
        _rcheck(ref().ref_graph_rand_index(self.h, _i32(a), _i32(b), C.byref(out)))
        return out.value

    def __del__(self):
        if self.h and _REF is not None:
            _REF.ref_graph_free(self.h)
            self.h = None

    def info(self):
        n, D, m, t = C.c_int64(), C.c_int64(), C.c_int64(), C.c_double()
        ref().ref_graph_info(self.h, C.byref(n), C.byref(D), C.byref(m), C.byref(t))
        return n.value, D.value, m.value, t.value

    def csr(self) -> CSR:
        n, D, m, t = self.info()
        off = np.zeros(n + 1, np.int64)
        col = np.zeros(max(D, 1), np.int32)
        w = np.zeros(max(D, 1), np.float64)
        vol = np.zeros(max(n, 1), np.float64)
        loop = np.zeros(max(n, 1), np.float64)
        ref().ref_graph_csr(self.h, off, col, w, vol, loop)
        return CSR(n, off, col[:D], w[:D], vol[:n], loop[:n], m, t)

    def modularity(self, z, gamma=1.0, ub=0):
        q, cov = C.c_double(), C.c_double()
        _rcheck(ref().ref_modularity(self.h, _i32(z), ub, gamma, C.byref(q), C.byref(cov)))
        return q.value, cov.value

    def dominant_label(self, z, u):
        out = C.c_int32()
        _rcheck(ref().ref_dominant_label(self.h, _i32(z), u, C.byref(out)))
        return out.value

    def is_stable(self, z):
        return bool(ref().ref_is_stable(self.h, _i32(z)))

    def run_plp(self, theta=-1, max_iterations=100, randomize=False, seed=1, workers=1, initial=None):
        n = self.info()[0]
        labels = np.zeros(max(n, 1), np.int32)
        rep = _RefReport()
        trace = np.zeros(max(max_iterations, 1), np.int64)
        init = None if initial is None else _i32(initial)
        _rcheck(ref().ref_run_plp(self.h, theta, max_iterations, int(randomize), seed, workers,
                                  None if init is None else init.ctypes.data, labels, C.byref(rep),
                                  trace.ctypes.data, len(trace)))
        return labels[:n], _report(rep), trace[: rep.iterations].copy()

    def run_louvain(self, refine=False, gamma=1.0, max_move_iterations=32, max_levels=64, seed=1, workers=1):
        n = self.info()[0]
        z = np.zeros(max(n, 1), np.int32)
        rep = _RefReport()
        _rcheck(ref().ref_run_louvain(self.h, gamma, max_move_iterations, max_levels, seed, workers, int(refine), z,
                                      C.byref(rep)))
        return z[:n], _report(rep)

    def move_phase(self, z, gamma=1.0, max_move_iterations=32, workers=1, ub=0):
        z = _i32(z).copy()
        ch = C.c_int()
        _rcheck(ref().ref_move_phase(self.h, z, ub, gamma, max_move_iterations, workers, C.byref(ch)))
        return z, bool(ch.value)

    def move_phase_log(self, z, gamma=1.0, max_move_iterations=32, workers=1, ub=0, with_q=False):
        """move_phase with a MoveObserver: (z, changed, moves[(u, c, d, gain)], q after each move)."""
        z = _i32(z).copy()
        cap = max(len(z), 1) * max(int(max_move_iterations), 1)
        lu, lc, ld = (np.zeros(cap, np.int32) for _ in range(3))
        lg = np.zeros(cap, np.float64)
        lq = np.zeros(cap, np.float64) if with_q else None
        cnt, ch = C.c_int64(), C.c_int()
        _rcheck(ref().ref_move_phase_log(self.h, z, ub, gamma, max_move_iterations, workers, lu, lc, ld, lg,
                                         None if lq is None else lq.ctypes.data, cap, C.byref(cnt), C.byref(ch)))
        k = min(cnt.value, cap)
        moves = list(zip(lu[:k].tolist(), lc[:k].tolist(), ld[:k].tolist(), lg[:k].tolist()))
        return z, bool(ch.value), moves, (lq[:k].copy() if with_q else None)

    def delta_mod(self, z, u, target, gamma=1.0, ub=0):
        out = C.c_double()
        _rcheck(ref().ref_delta_mod(self.h, _i32(z), ub, u, target, gamma, C.byref(out)))
        return out.value

    def coarsen(self, z, workers=1):
        n = self.info()[0]
        h = C.c_void_p()
        pi = np.zeros(max(n, 1), np.int32)
        _rcheck(ref().ref_coarsen(self.h, _i32(z), workers, C.byref(h), pi))
        return RefGraph(h.value), pi[:n]

    def run_epp(self, ensemble_size=4, seed=1, workers=1):
        n = self.info()[0]
        z = np.zeros(max(n, 1), np.int32)
        rep = _RefReport()
        _rcheck(ref().ref_run_epp(self.h, ensemble_size, seed, workers, z, C.byref(rep)))
        return z[:n], _report(rep)


def _report(r: _RefReport) -> dict:
    return {k: getattr(r, k) for k, _ in _RefReport._fields_}


def ref_compacted(z):
    z = _i32(z)
    out = np.zeros_like(z)
    cnt = ref().ref_compacted(len(z), z, out)
    return out, cnt


def ref_combine_hashed(solutions, workers=1):
    sols = [_i32(s) for s in solutions]
    ptrs = (C.c_void_p * len(sols))(*[s.ctypes.data for s in sols])
    out = np.zeros(len(sols[0]) if sols else 0, np.int32)
    _rcheck(ref().ref_combine_hashed(len(sols), len(out), ptrs, workers, out))
    return out


def ref_combine_exact(solutions):
    sols = [_i32(s) for s in solutions]
    ptrs = (C.c_void_p * len(sols))(*[s.ctypes.data for s in sols])
    out = np.zeros(len(sols[0]) if sols else 0, np.int32)
    _rcheck(ref().ref_combine_exact(len(sols), len(out), ptrs, out))
    return out


def ref_djb2(data: bytes) -> int:
    return ref().ref_djb2(data, len(data))


def ref_max_threads() -> int:
    return ref().ref_max_threads()
