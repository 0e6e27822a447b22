"""levelrank-b200: level-scheduled PageRank (arXiv 1609.09068) on B200.

Python mirror of the reference levelrank API (proj/include/levelrank/*.hpp)
over the C-ABI in include/lr_cuda.h, loaded from the in-tree
``liblevelrank_b200.so``.  Host work (graph build, SCC/CAC partition, layout)
is C++; the solve is sm_100a CUDA.  There is no CPU fallback: without the
shared library or a CUDA device the solve raises.

Reference entry points and their mirrors here:
  Graph::from_edges (graph.cpp:14-36)           -> Graph.from_edges
  load_edge_list (graph.cpp:101-105)            -> Graph.load_edge_list
  find_components (partition.cpp:246-248)       -> find_components
  find_components_scc_only (partition.cpp:250)  -> find_components_scc_only
  build_schedule (schedule.cpp:32-137)          -> build_schedule
  compute_pagerank (engine.cpp:89-182)          -> compute_pagerank / Engine
  validate_params, iteration_cap (solvers.cpp:11-21), error_bound,
  propagate_weights (engine.cpp:74-87)          -> same names
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "Graph", "Partition", "Schedule", "SolverParams", "EngineResult", "Engine", "LoopPolicy",
    "ExecutionMode", "find_components", "find_components_scc_only", "build_schedule", "compute_pagerank",
    "validate_params", "iteration_cap", "error_bound", "propagate_weights", "rmat", "dangle", "planted",
    "deep_dag", "config_graph", "LevelrankError", "ConvergenceError", "CycleError", "DegenerateError",
    "CudaError", "library_path",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.environ.get("LR_LIB") or os.path.join(_HERE, "liblevelrank_b200.so")  # LR_LIB: A/B builds only

I32P = C.POINTER(C.c_int32)
I64P = C.POINTER(C.c_int64)
F64P = C.POINTER(C.c_double)
U8P = C.POINTER(C.c_uint8)
VP = C.c_void_p


class LevelrankError(RuntimeError):
    """Base of the errors raised by the C-ABI."""


class ConvergenceError(LevelrankError):
    """power series failed to converge (solvers.cpp:159)."""


class CycleError(LevelrankError):
    """cycle inside an acyclic component (solvers.cpp:84-85); std::logic_error."""


class DegenerateError(LevelrankError):
    """dense solve degenerated numerically (solvers.cpp:103-106)."""


class CudaError(LevelrankError):
    """CUDA / NCCL / device-memory failure."""


class LoopPolicy:
    Ignore = 0
    Keep = 1


class ExecutionMode:
    Sequential = "sequential"
    Parallel = "parallel"


class _Report(C.Structure):
    _fields_ = [
        ("vertices", C.c_int64), ("edges", C.c_int64), ("components", C.c_int64),
        ("scc_components", C.c_int64), ("cac_components", C.c_int64), ("singleton_cacs", C.c_int64),
        ("largest_component", C.c_int32), ("largest_is_scc", C.c_int32), ("max_level", C.c_int32),
        ("level_count", C.c_int32), ("large_scc_vertices", C.c_int64), ("eps_tot", C.c_double),
        ("eps_avg", C.c_double), ("total_iterations", C.c_int64), ("iterative_edge_work", C.c_int64),
        ("iterative_edges", C.c_int64), ("single_pass_edge_work", C.c_int64),
        ("cross_edge_count", C.c_int64), ("total_edge_work", C.c_int64),
        ("mean_iterations_per_edge", C.c_double), ("all_weights_zero", C.c_int32), ("threads", C.c_int32),
        ("wall_ms", C.c_double), ("n_units", C.c_int64), ("plan_ms", C.c_double), ("upload_ms", C.c_double),
        ("solve_ms", C.c_double), ("device_ms", C.c_double),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class _SolveInfo(C.Structure):
    _fields_ = [
        ("total_iterations", C.c_int64), ("iterative_edge_work", C.c_int64), ("all_weights_zero", C.c_int32),
        ("n_devices", C.c_int32), ("device_ms", C.c_double), ("spmv_ms", C.c_double),
        ("spmv_launches", C.c_int64), ("kernel_launches", C.c_int64), ("spmv_active_launches", C.c_int64),
        ("spmv_active_ms", C.c_double), ("spmv_bytes", C.c_int64), ("spmv_edges", C.c_int64),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class _Census(C.Structure):
    _fields_ = [
        ("components", C.c_int64), ("scc_components", C.c_int64), ("cac_components", C.c_int64),
        ("singleton_cacs", C.c_int64), ("largest_component", C.c_int32), ("largest_is_scc", C.c_int32),
        ("max_level", C.c_int32), ("level_count", C.c_int32),
    ]


class _Layout(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("n_levels", C.c_int32), ("keep_loops", C.c_int32), ("n_units", C.c_int64),
        ("nnz_cross", C.c_int64), ("nnz_intra", C.c_int64), ("depth_ptr_len", C.c_int64),
        ("level_row_begin", I32P), ("level_unit_begin", I32P), ("vertex_of", I32P), ("row_of", I32P),
        ("deg", I32P), ("loop", U8P), ("xptr", I64P), ("xsrc", I32P), ("iptr", I64P), ("isrc", I32P),
        ("unit_kind", U8P), ("unit_level", I32P), ("unit_row_begin", I32P), ("unit_edges", I64P),
        ("cac_depth_begin", I64P), ("depth_ptr", I32P),
    ]


class UnitRecord(C.Structure):
    """lr_unit_record (UnitRecord, engine.hpp:20-27)."""
    _fields_ = [("kind", C.c_int32), ("level", C.c_int32), ("size", C.c_int32), ("reserved", C.c_int32),
                ("edges", C.c_int64), ("iterations", C.c_int64), ("wall_ms", C.c_double)]


class _ReportMeta(C.Structure):
    _fields_ = [("method", C.c_char_p), ("mode", C.c_char_p), ("c", C.c_double), ("tol", C.c_double),
                ("keep_loops", C.c_int32), ("small_threshold", C.c_int32), ("threads", C.c_int32),
                ("reserved", C.c_int32)]


CP = C.POINTER(C.c_char)

# Every symbol declared in include/lr_cuda.h (tests check they are exported).
EXPORTS = {
    "lr_last_error": (C.c_char_p, []),
    "lr_version": (C.c_char_p, []),
    "lr_graph_from_edges": (C.c_int, [C.c_int32, I32P, I32P, C.c_int64, C.c_int, C.POINTER(VP)]),
    "lr_graph_from_csr": (C.c_int, [C.c_int32, I64P, I32P, C.c_int, C.POINTER(VP)]),
    "lr_graph_load_edge_list": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.POINTER(VP)]),
    "lr_graph_parse_edge_buffer": (C.c_int, [C.c_char_p, C.c_int64, C.c_int, C.c_int, C.POINTER(VP)]),
    "lr_graph_vertex_count": (C.c_int32, [VP]),
    "lr_graph_edge_count": (C.c_int64, [VP]),
    "lr_graph_csr": (C.c_int, [VP, I64P, I32P, U8P, I32P]),
    "lr_graph_free": (None, [VP]),
    "lr_find_components": (C.c_int, [VP, C.c_int, I32P, I32P, I32P, I32P, I32P, I32P, I64P]),
    "lr_plan_build": (C.c_int, [VP, C.c_int32, C.POINTER(VP)]),
    "lr_plan_build_baseline": (C.c_int, [VP, C.POINTER(VP)]),
    "lr_plan_free": (None, [VP]),
    "lr_plan_schedule_sizes": (C.c_int, [VP, I64P]),
    "lr_plan_schedule_get": (C.c_int, [VP, I32P, I32P, I64P, I32P, I32P, I32P, I64P, I64P, I32P, I32P, I32P,
                                       I32P, I32P, I32P, I32P]),
    "lr_plan_census": (C.c_int, [VP, C.POINTER(_Census)]),
    "lr_plan_layout": (C.c_int, [VP, C.POINTER(_Layout)]),
    "lr_ctx_create": (C.c_int, [C.c_int, C.POINTER(VP)]),
    "lr_ctx_upload": (C.c_int, [VP, C.POINTER(_Layout)]),
    "lr_solve": (C.c_int, [VP, F64P, C.c_double, C.c_double, F64P, F64P, C.POINTER(_SolveInfo), I64P]),
    "lr_solve_device": (C.c_int, [VP, VP, C.c_double, C.c_double, VP, VP, C.POINTER(_SolveInfo), I64P]),
    "lr_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "lr_ctx_set_comm": (C.c_int, [VP, C.c_int, C.c_int, C.c_char_p]),
    "lr_shard_rows": (C.c_int, [I64P, C.c_int32, C.c_int32, C.c_int32, I32P]),
    "lr_exchange_cuts": (C.c_int, [I64P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, I32P]),
    "lr_split_level_rows": (C.c_int, [I64P, I64P, I32P, U8P, C.c_int32, C.c_int32, C.c_int32, I32P]),
    "lr_ctx_stream": (VP, [VP]),
    "lr_ctx_device_bytes": (C.c_int64, [VP]),
    "lr_ctx_blk_units": (C.c_int32, [VP]),
    "lr_ctx_unit_times": (C.c_int, [VP, F64P, C.c_int64]),
    "lr_ctx_free": (None, [VP]),
    "lr_compute_pagerank": (C.c_int, [VP, F64P, C.c_int64, C.c_double, C.c_double, C.c_int32, C.c_int, F64P,
                                      F64P, C.POINTER(_Report), I64P, C.c_int64]),
    "lr_compute_baseline": (C.c_int, [VP, F64P, C.c_int64, C.c_double, C.c_double, C.c_int, F64P, F64P,
                                      C.POINTER(_Report)]),
    "lr_report_format": (C.c_int, [C.POINTER(_Report), C.POINTER(_ReportMeta), C.POINTER(UnitRecord), C.c_int64,
                                   C.c_int, C.POINTER(CP), C.POINTER(C.c_int64)]),
    "lr_ranks_format": (C.c_int, [F64P, C.c_int64, C.POINTER(CP), C.POINTER(C.c_int64)]),
    "lr_ranks_write": (C.c_int, [F64P, C.c_int64, C.c_char_p]),
    "lr_string_free": (None, [CP]),
    "lr_solve_unit": (C.c_int, [VP, C.c_int, I32P, C.c_int32, I32P, I32P, C.c_int64, F64P, C.c_double, C.c_double,
                                C.c_int, F64P, I64P, I64P]),
    "lr_series_stats_csr": (C.c_int, [C.c_int, C.c_int32, I64P, I32P, F64P, F64P, C.c_double, C.c_int64, F64P, I64P,
                                      F64P, C.c_int64, F64P]),
    "lr_solve_large_scc_stats": (C.c_int, [VP, I32P, C.c_int32, I32P, I32P, C.c_int64, F64P, C.c_double, C.c_double,
                                           C.c_int, F64P, I64P, F64P, C.c_int64, I64P, F64P]),
    "lr_validate_params": (C.c_int, [C.c_double, C.c_double]),
    "lr_iteration_cap": (C.c_int64, [C.c_double, C.c_double]),
    "lr_error_bound": (None, [C.c_int64, C.c_int64, C.c_double, C.c_double, F64P]),
    "lr_propagate_weights": (C.c_int, [C.c_int, I32P, I32P, I32P, C.c_int64, F64P, C.c_int64, C.c_double, F64P]),
    "lr_gen_rmat": (C.c_int, [C.c_int32, C.c_int64, C.c_double, C.c_double, C.c_double, C.c_uint64,
                              C.POINTER(VP)]),
    "lr_graph_dangle": (C.c_int, [VP, C.c_double, C.c_uint64, C.POINTER(VP)]),
    "lr_gen_planted": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_double, C.c_int64,
                                 C.c_double, C.c_uint64, C.POINTER(VP)]),
    "lr_gen_deep_dag": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_int32, C.c_int32,
                                  C.c_double, C.c_int32, C.c_uint64, C.POINTER(VP)]),
}

_lib = None


def library_path() -> str:
    return _SO


def lib():
    """The loaded liblevelrank_b200.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            raise ImportError(f"{_SO} is missing: build it with `make -C paper_1609_09068_b200` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(_SO)
        for name, (res, args) in EXPORTS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


_ERR = {1: ValueError, 2: ConvergenceError, 3: CycleError, 4: DegenerateError, 5: CudaError, 6: CudaError,
        7: MemoryError, 8: OSError}


def _check(st):
    if st != 0:
        raise _ERR.get(st, LevelrankError)(lib().lr_last_error().decode())


def _p(a, t):
    return a.ctypes.data_as(t)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# --------------------------------------------------------------- graph core
class Graph:
    """Compressed out-adjacency graph (graph.hpp:39-76), owned by the C++ side."""

    def __init__(self, handle):
        self._h = handle

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.lr_graph_free(h)
            self._h = None

    @classmethod
    def from_edges(cls, n, edges=None, src=None, dst=None, loop_policy=LoopPolicy.Ignore):
        if edges is not None:
            e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
            src, dst = e[:, 0], e[:, 1]
        src = _i32(src if src is not None else [])
        dst = _i32(dst if dst is not None else [])
        h = VP()
        _check(lib().lr_graph_from_edges(int(n), _p(src, I32P), _p(dst, I32P), len(src), int(loop_policy),
                                         C.byref(h)))
        return cls(h)

    @classmethod
    def from_csr(cls, n, offsets, targets, loop_policy=LoopPolicy.Ignore):
        off = np.ascontiguousarray(offsets, np.int64)
        tgt = _i32(targets)
        h = VP()
        _check(lib().lr_graph_from_csr(int(n), _p(off, I64P), _p(tgt, I32P), int(loop_policy), C.byref(h)))
        return cls(h)

    @classmethod
    def load_edge_list(cls, path, dense_ids=True, loop_policy=LoopPolicy.Ignore):
        h = VP()
        _check(lib().lr_graph_load_edge_list(os.fsencode(path), int(dense_ids), int(loop_policy), C.byref(h)))
        return cls(h)

    @classmethod
    def parse_edge_list(cls, text, dense_ids=True, loop_policy=LoopPolicy.Ignore):
        """parse_edge_list (graph.cpp:54-99) over a str/bytes buffer."""
        data = text.encode() if isinstance(text, str) else bytes(text)
        h = VP()
        _check(lib().lr_graph_parse_edge_buffer(data, len(data), int(dense_ids), int(loop_policy), C.byref(h)))
        return cls(h)

    @property
    def n(self) -> int:
        return int(lib().lr_graph_vertex_count(self._h))

    vertex_count = n

    @property
    def m(self) -> int:
        return int(lib().lr_graph_edge_count(self._h))

    edge_count = m

    def csr(self):
        """(offsets int64[n+1], targets int32[m], has_loop uint8[n], walk_out_degree int32[n])."""
        n, m = self.n, self.m
        off, tgt = np.zeros(n + 1, np.int64), np.zeros(m, np.int32)
        loop, deg = np.zeros(n, np.uint8), np.zeros(n, np.int32)
        _check(lib().lr_graph_csr(self._h, _p(off, I64P), _p(tgt, I32P), _p(loop, U8P), _p(deg, I32P)))
        return off, tgt, loop, deg


# ---------------------------------------------------------------- partition
@dataclass
class Partition:
    comp_of: np.ndarray
    kinds: np.ndarray  # 0 = Scc, 1 = Cac (partition.hpp:13)
    levels: np.ndarray
    sizes: np.ndarray
    max_level: int
    stats: tuple = (0, 0, 0)  # explore_edge_visits, merge_scan_edge_visits, finish_calls

    def component_count(self) -> int:
        return len(self.kinds)


def _partition(g: Graph, merge: bool) -> Partition:
    n = g.n
    comp = np.zeros(n, np.int32)
    kinds, levels, sizes = (np.zeros(max(n, 1), np.int32) for _ in range(3))
    k, ml = C.c_int32(), C.c_int32()
    st = np.zeros(3, np.int64)
    _check(lib().lr_find_components(g._h, int(merge), _p(comp, I32P), _p(kinds, I32P), _p(levels, I32P),
                                    _p(sizes, I32P), C.byref(k), C.byref(ml), _p(st, I64P)))
    k = k.value
    return Partition(comp, kinds[:k].copy(), levels[:k].copy(), sizes[:k].copy(), ml.value, tuple(int(x) for x in st))


def find_components(g: Graph) -> Partition:
    return _partition(g, True)


def find_components_scc_only(g: Graph) -> Partition:
    return _partition(g, False)


# ---------------------------------------------------------- plan / schedule
@dataclass
class Schedule:
    """Flattened reference Schedule (schedule.hpp:13-57); unit kinds 0 Singleton, 1 Cac, 2 SccSmall, 3 SccLarge."""
    level_values: np.ndarray
    level_unit_begin: np.ndarray
    level_cross_begin: np.ndarray
    unit_kind: np.ndarray
    unit_level: np.ndarray
    unit_size: np.ndarray
    unit_ids_begin: np.ndarray
    unit_edges_begin: np.ndarray
    ids: np.ndarray
    edge_src: np.ndarray
    edge_dst: np.ndarray
    cross_src: np.ndarray
    cross_dst: np.ndarray
    cross_deg: np.ndarray
    permutation: np.ndarray
    intra: int
    cross: int
    dropped: int


_SCHED_ORDER = ["level_values", "level_unit_begin", "level_cross_begin", "unit_kind", "unit_level", "unit_size",
                "unit_ids_begin", "unit_edges_begin", "ids", "edge_src", "edge_dst", "cross_src", "cross_dst",
                "cross_deg", "permutation"]


class Plan:
    """find_components + build_schedule + device Layout (lr_plan)."""

    def __init__(self, g: Graph, small_threshold: int = 100, baseline: bool = False):
        """baseline=True: the whole graph as one power-series unit (compute_baseline's
        layout, lr_plan_build_baseline) -- no partition, no schedule."""
        self.graph = g  # keeps the borrowed graph alive
        h = VP()
        if baseline:
            _check(lib().lr_plan_build_baseline(g._h, C.byref(h)))
        else:
            _check(lib().lr_plan_build(g._h, int(small_threshold), C.byref(h)))
        self._h = h
        self.small_threshold = small_threshold
        self.baseline = baseline

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.lr_plan_free(h)
            self._h = None

    def schedule(self) -> Schedule:
        sz = np.zeros(8, np.int64)
        _check(lib().lr_plan_schedule_sizes(self._h, _p(sz, I64P)))
        nl, nu, nid, ne, nx = (int(x) for x in sz[:5])
        arr = dict(level_values=np.zeros(nl, np.int32), level_unit_begin=np.zeros(nl + 1, np.int32),
                   level_cross_begin=np.zeros(nl + 1, np.int64), unit_kind=np.zeros(nu, np.int32),
                   unit_level=np.zeros(nu, np.int32), unit_size=np.zeros(nu, np.int32),
                   unit_ids_begin=np.zeros(nu + 1, np.int64), unit_edges_begin=np.zeros(nu + 1, np.int64),
                   ids=np.zeros(nid, np.int32), edge_src=np.zeros(ne, np.int32), edge_dst=np.zeros(ne, np.int32),
                   cross_src=np.zeros(nx, np.int32), cross_dst=np.zeros(nx, np.int32),
                   cross_deg=np.zeros(nx, np.int32), permutation=np.zeros(nid, np.int32))
        ptrs = [arr[k].ctypes.data_as(I64P if arr[k].dtype == np.int64 else I32P) for k in _SCHED_ORDER]
        _check(lib().lr_plan_schedule_get(self._h, *ptrs))
        return Schedule(**arr, intra=int(sz[5]), cross=int(sz[6]), dropped=int(sz[7]))

    def census(self) -> dict:
        c = _Census()
        _check(lib().lr_plan_census(self._h, C.byref(c)))
        return {k: getattr(c, k) for k, _ in c._fields_}

    def layout(self) -> dict:
        """Host copies of the device Layout arrays (schedule.hpp Layout)."""
        L = _Layout()
        _check(lib().lr_plan_layout(self._h, C.byref(L)))
        n, nl, nu = L.n, L.n_levels, L.n_units

        def arr(ptr, count, dt):
            if count == 0:
                return np.zeros(0, dt)
            return np.ctypeslib.as_array(ptr, shape=(count,)).astype(dt, copy=True)

        return dict(
            n=n, n_levels=nl, n_units=nu, keep_loops=L.keep_loops,
            level_row_begin=arr(L.level_row_begin, nl + 1, np.int32),
            level_unit_begin=arr(L.level_unit_begin, nl + 1, np.int32),
            vertex_of=arr(L.vertex_of, n, np.int32), row_of=arr(L.row_of, n, np.int32),
            deg=arr(L.deg, n, np.int32), loop=arr(L.loop, n, np.uint8),
            xptr=arr(L.xptr, n + 1, np.int64), xsrc=arr(L.xsrc, L.nnz_cross, np.int32),
            iptr=arr(L.iptr, n + 1, np.int64), isrc=arr(L.isrc, L.nnz_intra, np.int32),
            unit_kind=arr(L.unit_kind, nu, np.uint8), unit_level=arr(L.unit_level, nu, np.int32),
            unit_row_begin=arr(L.unit_row_begin, nu + 1, np.int32), unit_edges=arr(L.unit_edges, nu, np.int64),
            cac_depth_begin=arr(L.cac_depth_begin, nu, np.int64),
            depth_ptr=arr(L.depth_ptr, L.depth_ptr_len, np.int32))


def build_schedule(g: Graph, small_threshold: int = 100) -> Schedule:
    return Plan(g, small_threshold).schedule()


# ---------------------------------------------------------------- solving
@dataclass
class SolverParams:
    c: float = 0.85
    tol: float = 1e-9


def validate_params(params: SolverParams) -> None:
    _check(lib().lr_validate_params(params.c, params.tol))


def iteration_cap(params: SolverParams) -> int:
    return int(lib().lr_iteration_cap(params.c, params.tol))


def error_bound(large_scc_vertices: int, vertex_count: int, params: SolverParams):
    out = np.zeros(2)
    lib().lr_error_bound(int(large_scc_vertices), int(vertex_count), params.c, params.tol, _p(out, F64P))
    return float(out[0]), float(out[1])


def propagate_weights(src, dst, src_out_degree, ranks, c, weights, device=0):
    """weights[dst] += c * ranks[src] / src_out_degree, on the GPU (engine.cpp:83-87). Returns new weights."""
    src, dst, deg = _i32(src), _i32(dst), _i32(src_out_degree)
    r = _f64(ranks)
    w = _f64(weights).copy()
    _check(lib().lr_propagate_weights(int(device), _p(src, I32P), _p(dst, I32P), _p(deg, I32P), len(src),
                                      _p(r, F64P), len(r), float(c), _p(w, F64P)))
    return w


def _nccl_first():
    """The library dlopens "libnccl.so.2" on first NCCL use.  In a process that
    also uses torch, torch's bundled NCCL must be the one loaded under that
    soname (a system copy loaded first would leave torch's own symbols
    unresolved), so torch is imported before the library's first NCCL call."""
    try:
        import torch  # noqa: F401
    except ImportError:  # no torch: the library binds the system libnccl
        pass


def nccl_unique_id() -> bytes:
    """A fresh 128-byte NCCL id (rank 0 creates it and broadcasts it)."""
    _nccl_first()
    buf = C.create_string_buffer(128)
    _check(lib().lr_nccl_unique_id(buf))
    return buf.raw


def shard_rows(iptr, row_begin: int, row_end: int, world: int) -> np.ndarray:
    """The nnz-balanced row split the multi-GPU solve uses (lr_shard_rows)."""
    ip = np.ascontiguousarray(iptr, np.int64)
    out = np.zeros(world + 1, np.int32)
    _check(lib().lr_shard_rows(_p(ip, I64P), int(row_begin), int(row_end), int(world), _p(out, I32P)))
    return out


def split_level_rows(layout: dict, level: int, world: int) -> np.ndarray:
    """lr_split_level_rows on a Plan.layout(): world + 1 row bounds of one level."""
    ip = np.ascontiguousarray(layout["iptr"], np.int64)
    xp = np.ascontiguousarray(layout["xptr"], np.int64)
    urb = np.ascontiguousarray(layout["unit_row_begin"], np.int32)
    uk = np.ascontiguousarray(layout["unit_kind"], np.uint8)
    lub = layout["level_unit_begin"]
    out = np.zeros(world + 1, np.int32)
    _check(lib().lr_split_level_rows(_p(ip, I64P), _p(xp, I64P), _p(urb, I32P), _p(uk, U8P), int(lub[level]),
                                     int(lub[level + 1]), int(world), _p(out, I32P)))
    return out


def exchange_cuts(iptr, row_begin: int, row_end: int, world: int, chunks: int) -> np.ndarray:
    """lr_exchange_cuts: world * chunks + 1 row bounds of the chunked s' exchange."""
    ip = np.ascontiguousarray(iptr, np.int64)
    out = np.zeros(world * chunks + 1, np.int32)
    _check(lib().lr_exchange_cuts(_p(ip, I64P), int(row_begin), int(row_end), int(world), int(chunks), _p(out, I32P)))
    return out


@dataclass
class EngineResult:
    ranks: np.ndarray          # R3 (non-normalised PageRank), vertex order
    r1: np.ndarray             # R1 = R3 / ||R3||_1
    report: dict
    unit_iters: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    info: dict = field(default_factory=dict)


class Engine:
    """Plan once, upload once, then solve any number of weight vectors on one GPU."""

    def __init__(self, g: Graph, small_threshold: int = 100, device: int = 0, rank: int = 0, world: int = 1,
                 nccl_id: bytes | None = None, baseline: bool = False):
        """rank/world/nccl_id: row-shard the giant SCC units over `world` GPUs
        (one process per GPU, every rank passes the same graph and id).
        baseline=True: solve the whole graph as one power series (compute_baseline)."""
        import time
        t0 = time.perf_counter()
        self.plan = Plan(g, small_threshold, baseline=baseline)
        self.plan_ms = (time.perf_counter() - t0) * 1e3
        self.n = g.n
        self.m = g.m
        h = VP()
        _check(lib().lr_ctx_create(int(device), C.byref(h)))
        self._h = h
        if world > 1 or nccl_id is not None:
            _nccl_first()
            _check(lib().lr_ctx_set_comm(h, int(rank), int(world), nccl_id))
        self._layout = _Layout()
        _check(lib().lr_plan_layout(self.plan._h, C.byref(self._layout)))
        t1 = time.perf_counter()
        _check(lib().lr_ctx_upload(self._h, C.byref(self._layout)))
        self.upload_ms = (time.perf_counter() - t1) * 1e3
        self.n_units = int(self._layout.n_units)
        self.census = {} if baseline else self.plan.census()

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.lr_ctx_free(h)
            self._h = None

    @property
    def stream(self) -> int:
        return int(lib().lr_ctx_stream(self._h) or 0)

    def device_bytes(self) -> int:
        return int(lib().lr_ctx_device_bytes(self._h))

    def blk_units(self) -> int:
        """Levels whose grid SpMV runs as K5 (k_spmv_blk, dest-row blocks)."""
        return int(lib().lr_ctx_blk_units(self._h))

    def unit_times(self) -> np.ndarray:
        """UnitRecord::wall_ms of the last solve (device span of each unit's
        tasks); needs LR_UNIT_TIMES=1 in the environment when the Engine is built."""
        out = np.zeros(max(self.n_units, 1))
        _check(lib().lr_ctx_unit_times(self._h, _p(out, F64P), self.n_units))
        return out[:self.n_units]

    def solve(self, weights, params: SolverParams = SolverParams(), r3=None, r1=None, want_unit_iters=True):
        """Host buffers in, host buffers out (lr_solve).  Returns (r3, r1, info, unit_iters)."""
        w = _f64(weights)
        if len(w) != self.n:
            raise ValueError("weight vector does not match the vertex count")
        r3 = np.empty(self.n) if r3 is None else r3
        r1 = np.empty(self.n) if r1 is None else r1
        info = _SolveInfo()
        it = np.zeros(max(self.n_units, 1), np.int64) if want_unit_iters else None
        _check(lib().lr_solve(self._h, _p(w, F64P), params.c, params.tol, _p(r3, F64P), _p(r1, F64P),
                              C.byref(info), _p(it, I64P) if it is not None else None))
        return r3, r1, info.as_dict(), (it[:self.n_units] if it is not None else None)

    def solve_ptr(self, w_ptr: int, r3_ptr: int, r1_ptr: int, host: bool, params: SolverParams = SolverParams()):
        """Raw-pointer variant: host=True -> lr_solve on (pinned) host buffers, else lr_solve_device."""
        info = _SolveInfo()
        if host:
            _check(lib().lr_solve(self._h, C.cast(w_ptr, F64P), params.c, params.tol, C.cast(r3_ptr, F64P),
                                  C.cast(r1_ptr, F64P) if r1_ptr else None, C.byref(info), None))
        else:
            _check(lib().lr_solve_device(self._h, VP(w_ptr), params.c, params.tol, VP(r3_ptr),
                                         VP(r1_ptr) if r1_ptr else None, C.byref(info), None))
        return info.as_dict()


def compute_pagerank(g: Graph, weights, params: SolverParams = SolverParams(), mode=ExecutionMode.Sequential,
                     small_threshold: int = 100, threads: int = 0, device: int = 0) -> EngineResult:
    """compute_pagerank (engine.cpp:89-182): partition, layout, GPU level loop, R1."""
    w = _f64(weights)
    n = g.n
    ranks = np.zeros(n)
    r1 = np.zeros(n)
    rep = _Report()
    cap = max(n + 1, 1)
    it = np.zeros(cap, np.int64)
    _check(lib().lr_compute_pagerank(g._h, _p(w, F64P), len(w), float(params.c), float(params.tol),
                                     int(small_threshold), int(device), _p(ranks, F64P), _p(r1, F64P), C.byref(rep),
                                     _p(it, I64P), cap))
    d = rep.as_dict()
    d["method"] = "partitioned"
    d["mode"] = "parallel" if mode == ExecutionMode.Parallel else "sequential"
    d["threads"] = (threads or os.cpu_count() or 1) if mode == ExecutionMode.Parallel else 1
    d["c"], d["tol"], d["small_threshold"] = params.c, params.tol, small_threshold
    d["largest_component_kind"] = "scc" if d.pop("largest_is_scc") else "cac"
    d["all_weights_zero"] = bool(d["all_weights_zero"])
    return EngineResult(ranks, r1, d, it[: rep.n_units].copy())


UNIT_KINDS = {"singletons": 0, "cac": 1, "small_scc": 2, "large_scc": 3}


def solve_unit(g: Graph, kind, global_ids, edge_src, edge_dst, w_local, params: SolverParams = SolverParams(),
               device: int = 0):
    """The unit solvers solve_singletons / solve_cac / solve_small_scc /
    solve_large_scc (solvers.hpp:31-54) on the GPU.  kind: 0-3 or a UNIT_KINDS
    name; edges in local ids.  Returns (ranks, iterations, edge_visits)."""
    k = UNIT_KINDS.get(kind, kind)
    ids, es, ed = _i32(global_ids), _i32(edge_src), _i32(edge_dst)
    w = _f64(w_local)
    out = np.zeros(len(ids))
    it, vis = C.c_int64(), C.c_int64()
    _check(lib().lr_solve_unit(g._h, int(k), _p(ids, I32P), len(ids), _p(es, I32P), _p(ed, I32P), len(es), _p(w, F64P),
                               float(params.c), float(params.tol), int(device), _p(out, F64P), C.byref(it),
                               C.byref(vis)))
    return out, it.value, vis.value


def solve_large_scc_stats(g: Graph, global_ids, edge_src, edge_dst, w_local, params: SolverParams = SolverParams(),
                          device: int = 0, cap: int = 1 << 16):
    """solve_large_scc with PowerSeriesStats (solvers.hpp:23-27, :48-51):
    returns (ranks, iterations, increment L1 norms, smallest increment entry)."""
    ids, es, ed = _i32(global_ids), _i32(edge_src), _i32(edge_dst)
    w = _f64(w_local)
    out, l1 = np.zeros(len(ids)), np.zeros(cap)
    it, n1, mn = C.c_int64(), C.c_int64(), C.c_double()
    _check(lib().lr_solve_large_scc_stats(g._h, _p(ids, I32P), len(ids), _p(es, I32P), _p(ed, I32P), len(es),
                                          _p(w, F64P), float(params.c), float(params.tol), int(device), _p(out, F64P),
                                          C.byref(it), _p(l1, F64P), cap, C.byref(n1), C.byref(mn)))
    return out, it.value, l1[:min(n1.value, cap)].copy(), mn.value


def compute_baseline(g: Graph, weights, params: SolverParams = SolverParams(), device: int = 0) -> EngineResult:
    """compute_baseline (engine.cpp:184-218): the whole-graph power series
    (solve_baseline, solvers.cpp:164-198) on the GPU -- the partition-free
    "basic method" the level-scheduled solve is measured against."""
    w = _f64(weights)
    n = g.n
    ranks = np.zeros(n)
    r1 = np.zeros(n)
    rep = _Report()
    _check(lib().lr_compute_baseline(g._h, _p(w, F64P), len(w), float(params.c), float(params.tol), int(device),
                                     _p(ranks, F64P), _p(r1, F64P), C.byref(rep)))
    d = rep.as_dict()
    d["method"] = "baseline"
    d["c"], d["tol"] = params.c, params.tol
    d["all_weights_zero"] = bool(d["all_weights_zero"])
    for k in ("components", "scc_components", "cac_components", "singleton_cacs", "largest_component",
              "largest_is_scc", "level_count", "large_scc_vertices", "eps_tot", "eps_avg", "cross_edge_count",
              "single_pass_edge_work"):
        d.pop(k, None)
    d["max_level"] = -1
    return EngineResult(ranks, r1, d, np.array([rep.total_iterations], np.int64))


# ----------------------------------------------------------- output formats
def _take_string(fn, *args) -> str:
    out, n = CP(), C.c_int64()
    _check(fn(*args, C.byref(out), C.byref(n)))
    try:
        return C.string_at(out, n.value).decode()
    finally:
        lib().lr_string_free(out)


def _c_report(report: dict) -> _Report:
    r = _Report()
    for k, _ in _Report._fields_:
        if k == "largest_is_scc":
            r.largest_is_scc = int(report.get("largest_component_kind", "cac") == "scc")
        elif k in report and report[k] is not None:
            setattr(r, k, type(getattr(r, k))(report[k]))
    return r


def format_report(report: dict, units=(), fmt: str = "text") -> str:
    """SolveReport::write_text / write_json (proj/src/report.cpp:24-113) or a
    bench CSV row / header (proj/src/cli.cpp:262-281), byte-compatible with the
    reference.  `report` is an EngineResult.report dict; `units` a sequence of
    (kind, level, size, edges, iterations, wall_ms)."""
    code = {"text": 0, "json": 1, "csv_row": 2, "csv_header": 3}[fmt]
    meta = _ReportMeta(str(report.get("method", "partitioned")).encode(), str(report.get("mode", "sequential")).encode(),
                       float(report.get("c", 0.85)), float(report.get("tol", 1e-9)), int(report.get("keep_loops", 0)),
                       int(report.get("small_threshold", 100)), int(report.get("threads", 1)), 0)
    arr = (UnitRecord * max(len(units), 1))()
    for i, u in enumerate(units):
        arr[i] = UnitRecord(int(u[0]), int(u[1]), int(u[2]), 0, int(u[3]), int(u[4]), float(u[5]))
    return _take_string(lib().lr_report_format, C.byref(_c_report(report)), C.byref(meta), arr, len(units), code)


def format_ranks(ranks) -> str:
    """write_ranks (proj/src/cli.cpp:80-83): "v<TAB>rank" at 12 significant digits."""
    r = _f64(ranks)
    return _take_string(lib().lr_ranks_format, _p(r, F64P), len(r))


def write_ranks(ranks, path) -> None:
    r = _f64(ranks)
    _check(lib().lr_ranks_write(_p(r, F64P), len(r), os.fsencode(path)))


def report_units(plan_or_engine, unit_iters, wall_ms=None):
    """UnitRecords (kind, level, size, edges, iterations, wall_ms) in schedule order."""
    plan = getattr(plan_or_engine, "plan", plan_or_engine)
    L = plan.layout()
    size = np.diff(L["unit_row_begin"])
    wall = np.zeros(len(size)) if wall_ms is None else np.asarray(wall_ms, np.float64)
    return [(int(k), int(lv), int(sz), int(e), int(it), float(w)) for k, lv, sz, e, it, w in
            zip(L["unit_kind"], L["unit_level"], size, L["unit_edges"], unit_iters, wall)]


# --------------------------------------------------------- synthetic inputs
def _gen(fn, *args) -> Graph:
    h = VP()
    _check(fn(*args, C.byref(h)))
    return Graph(h)


def rmat(scale, edge_factor, a=0.57, b=0.19, c=0.19, seed=1) -> Graph:
    return _gen(lib().lr_gen_rmat, int(scale), int(edge_factor), float(a), float(b), float(c), int(seed))


def dangle(g: Graph, p, seed) -> Graph:
    h = VP()
    _check(lib().lr_graph_dangle(g._h, float(p), int(seed), C.byref(h)))
    return Graph(h)


def planted(n=100_000, n_scc=200, scc_min=16, scc_max=1024, scc_vertex_budget=50_000, scc_out_degree=4.0,
            inter_edges=50_000, dangling_fraction=0.10, seed=1) -> Graph:
    return _gen(lib().lr_gen_planted, int(n), int(n_scc), int(scc_min), int(scc_max), int(scc_vertex_budget),
                float(scc_out_degree), int(inter_edges), float(dangling_fraction), int(seed))


def deep_dag(levels=1000, width=16_000, scc_min=2, scc_max=64, scc_out_degree=6.0, branch_min=1, branch_max=4,
             inter_out_degree=4.5, reach=8, seed=1) -> Graph:
    return _gen(lib().lr_gen_deep_dag, int(levels), int(width), int(scc_min), int(scc_max), float(scc_out_degree),
                int(branch_min), int(branch_max), float(inter_out_degree), int(reach), int(seed))


# BASELINE.json configs.  `shrink` k > 0 makes
# a smaller graph of the same recipe for tests: R-MAT scale - k, planted and
# deep DAG divided by 2^k.
CONFIGS = {
    1: "planted 100k: 200 SCCs U[16,1024] rescaled to 50k vertices, out-trees, 50k inter edges, 10% dangling",
    2: "R-MAT scale 20, edge factor 16, (0.57,0.19,0.19,0.05), loops+dups removed",
    3: "R-MAT scale 23, edge factor 8, then 30% of vertices lose their out-edges",
    4: "deep DAG: 1000 levels x 16k vertices, SCCs U[2,64] (deg 6) + trees (branch U[1,4]), reach 1..8",
    5: "R-MAT scale 26, edge factor 16, (0.57,0.19,0.19,0.05), dedup",
}


def config_graph(cfg: int, shrink: int = 0) -> Graph:
    if cfg == 1:
        f = 2 ** shrink
        return planted(n=100_000 // f, n_scc=max(200 // f, 2), scc_vertex_budget=50_000 // f,
                       inter_edges=50_000 // f)
    if cfg == 2:
        return rmat(20 - shrink, 16, seed=1)
    if cfg == 3:
        return dangle(rmat(23 - shrink, 8, seed=1), 0.3, 2)
    if cfg == 4:
        f = 2 ** shrink
        return deep_dag(levels=max(1000 // f, 8), width=max(16_000 // f, 256))
    if cfg == 5:
        return rmat(26 - shrink, 16, seed=1)
    raise ValueError(f"unknown config {cfg}")
