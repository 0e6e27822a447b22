"""TEST INFRASTRUCTURE ONLY -- ctypes bindings for the CPU checkers.

* ``Oracle``  -> oracle/liblr_oracle.so, the plain-C restatement (lr_oracle.c)
* ``Ref``     -> oracle/_ref/liblevelrank_ref.so, the reference levelrank
  compiled from its own sources (oracle/Makefile ``ref`` target)

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liblr_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "liblevelrank_ref.so")

I32P = C.POINTER(C.c_int32)
I64P = C.POINTER(C.c_int64)
F64P = C.POINTER(C.c_double)
U8P = C.POINTER(C.c_uint8)

REPORT_FIELDS = [
    ("vertices", C.c_int64), ("edges", C.c_int64), ("components", C.c_int64),
    ("scc_components", C.c_int64), ("cac_components", C.c_int64), ("singleton_cacs", C.c_int64),
    ("largest_component", C.c_int32), ("largest_is_scc", C.c_int32), ("max_level", C.c_int32),
    ("level_count", C.c_int32), ("large_scc_vertices", C.c_int64), ("eps_tot", C.c_double),
    ("eps_avg", C.c_double), ("total_iterations", C.c_int64), ("iterative_edge_work", C.c_int64),
    ("iterative_edges", C.c_int64), ("single_pass_edge_work", C.c_int64),
    ("cross_edge_count", C.c_int64), ("total_edge_work", C.c_int64),
    ("mean_iterations_per_edge", C.c_double), ("all_weights_zero", C.c_int32),
    ("threads", C.c_int32), ("wall_ms", C.c_double), ("n_units", C.c_int64),
]


class Report(C.Structure):
    _fields_ = REPORT_FIELDS

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in REPORT_FIELDS}


STATUS_EXC = {1: ValueError, 2: RuntimeError, 3: ArithmeticError, 4: RuntimeError, 7: MemoryError, 9: RuntimeError}


def _p(a, t):
    return a.ctypes.data_as(t)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class PartitionOut:
    comp_of: np.ndarray
    kinds: np.ndarray  # 0 = Scc, 1 = Cac
    levels: np.ndarray
    sizes: np.ndarray
    max_level: int
    stats: tuple | None = None


@dataclass
class ScheduleOut:
    level_values: np.ndarray
    level_unit_begin: np.ndarray
    level_cross_begin: np.ndarray
    unit_kind: np.ndarray  # 0 Singleton, 1 Cac, 2 SccSmall, 3 SccLarge
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


@dataclass
class SolveOut:
    ranks: np.ndarray
    report: dict
    unit_iters: np.ndarray
    unit_kinds: np.ndarray


def _sched_arrays(sizes):
    nl, nu, nid, ne, nx = (int(x) for x in sizes[:5])
    return dict(
        level_values=np.zeros(nl, np.int32), level_unit_begin=np.zeros(nl + 1, np.int32),
        level_cross_begin=np.zeros(nl + 1, np.int64), unit_kind=np.zeros(nu, np.int32),
        unit_level=np.zeros(nu, np.int32), unit_size=np.zeros(nu, np.int32),
        unit_ids_begin=np.zeros(nu + 1, np.int64), unit_edges_begin=np.zeros(nu + 1, np.int64),
        ids=np.zeros(nid, np.int32), edge_src=np.zeros(ne, np.int32), edge_dst=np.zeros(ne, np.int32),
        cross_src=np.zeros(nx, np.int32), cross_dst=np.zeros(nx, np.int32),
        cross_deg=np.zeros(nx, np.int32), permutation=np.zeros(nid, np.int32))


_SCHED_ORDER = ["level_values", "level_unit_begin", "level_cross_begin", "unit_kind", "unit_level",
                "unit_size", "unit_ids_begin", "unit_edges_begin", "ids", "edge_src", "edge_dst",
                "cross_src", "cross_dst", "cross_deg", "permutation"]


def _ptr(a):
    return a.ctypes.data_as(I64P if a.dtype == np.int64 else I32P)


class _Lib:
    prefix = ""

    def _err(self):
        return getattr(self.lib, self.prefix + "last_error")().decode()

    def _check(self, rc):
        if rc != 0:
            raise STATUS_EXC.get(rc, RuntimeError)(self._err())


class Oracle(_Lib):
    """The plain-C restatement (oracle/lr_oracle.c)."""

    prefix = "lro_"

    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        lib = C.CDLL(path)
        self.lib = lib
        lib.lro_last_error.restype = C.c_char_p
        lib.lro_graph_from_edges.argtypes = [C.c_int32, I32P, I32P, C.c_int64, C.c_int, C.POINTER(C.c_void_p)]
        lib.lro_graph_from_csr.argtypes = [C.c_int32, I64P, I32P, C.c_int, C.POINTER(C.c_void_p)]
        lib.lro_graph_free.argtypes = [C.c_void_p]
        lib.lro_graph_edges.argtypes = [C.c_void_p]
        lib.lro_graph_edges.restype = C.c_int64
        lib.lro_graph_csr.argtypes = [C.c_void_p, I64P, I32P, U8P, I32P]
        lib.lro_find_components.argtypes = [C.c_void_p, C.c_int, I32P, I32P, I32P, I32P, I32P, I32P, I64P]
        lib.lro_schedule_new.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_void_p)]
        lib.lro_schedule_free.argtypes = [C.c_void_p]
        lib.lro_schedule_sizes.argtypes = [C.c_void_p, I64P]
        lib.lro_schedule_get.argtypes = [C.c_void_p] + [I32P, I32P, I64P, I32P, I32P, I32P, I64P, I64P] + [I32P] * 7
        lib.lro_iteration_cap.argtypes = [C.c_double, C.c_double]
        lib.lro_iteration_cap.restype = C.c_int64
        lib.lro_error_bound.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_double, F64P]
        lib.lro_compute_pagerank.argtypes = [C.c_void_p, F64P, C.c_int64, C.c_double, C.c_double, C.c_int32,
                                             F64P, C.POINTER(Report), I64P, I32P, C.c_int64]
        lib.lro_compute_baseline.argtypes = [C.c_void_p, F64P, C.c_int64, C.c_double, C.c_double, F64P,
                                             C.POINTER(Report)]
        lib.lro_normalize_r1.argtypes = [F64P, C.c_int64, F64P]
        lib.lro_sample_large_scc.argtypes = [C.c_void_p, C.c_void_p, F64P, C.c_double, C.c_int64, I64P, F64P]

        pp = C.POINTER(I32P)
        lib.lro_gen_rmat.argtypes = [C.c_int32, C.c_int64, C.c_double, C.c_double, C.c_double, C.c_uint64,
                                     C.c_double, C.c_uint64, C.c_int, pp, pp, I64P]
        lib.lro_gen_planted.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_double,
                                        C.c_int64, C.c_double, C.c_uint64, pp, pp, I64P]
        lib.lro_gen_deep_dag.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_int32,
                                         C.c_int32, C.c_double, C.c_int32, C.c_uint64, C.c_int, pp, pp, I64P]
        lib.lro_gen_free.argtypes = [I32P]

    def __getitem__(self, k):
        return getattr(self.lib, k)

    # -- synthetic inputs (oracle/lr_gen.c; same recipes as paper_1609_09068_b200.config_graph)
    def gen_config(self, cfg, shrink=0, threads=None):
        """Edge list (n, src, dst) of BASELINE.json config `cfg` (duplicates
        and, outside R-MAT, self-loops included; Graph::from_edges removes them)."""
        threads = int(threads or os.cpu_count() or 1)
        s, d, m = I32P(), I32P(), C.c_int64()
        f = 2 ** shrink
        if cfg in (2, 3, 5):
            scale, ef = {2: (20, 16), 3: (23, 8), 5: (26, 16)}[cfg]
            scale -= shrink
            n = 1 << scale
            self._check(self.lib.lro_gen_rmat(scale, ef, 0.57, 0.19, 0.19, 1, 0.3 if cfg == 3 else 0.0, 2, threads,
                                              C.byref(s), C.byref(d), C.byref(m)))
        elif cfg == 1:
            n = 100_000 // f
            self._check(self.lib.lro_gen_planted(n, max(200 // f, 2), 16, 1024, 50_000 // f, 4.0, 50_000 // f, 0.10,
                                                 1, C.byref(s), C.byref(d), C.byref(m)))
        elif cfg == 4:
            levels, width = max(1000 // f, 8), max(16_000 // f, 256)
            n = levels * width
            self._check(self.lib.lro_gen_deep_dag(levels, width, 2, 64, 6.0, 1, 4, 4.5, 8, 1, threads,
                                                  C.byref(s), C.byref(d), C.byref(m)))
        else:
            raise ValueError(f"unknown config {cfg}")
        try:
            src = np.ctypeslib.as_array(s, (m.value,)).copy() if m.value else np.zeros(0, np.int32)
            dst = np.ctypeslib.as_array(d, (m.value,)).copy() if m.value else np.zeros(0, np.int32)
        finally:
            self.lib.lro_gen_free(s)
            self.lib.lro_gen_free(d)
        return n, src, dst

    # -- graph
    def graph(self, n, src, dst, keep=False):
        src, dst = _i32(src), _i32(dst)
        h = C.c_void_p()
        self._check(self.lib.lro_graph_from_edges(n, _p(src, I32P), _p(dst, I32P), len(src), int(keep), C.byref(h)))
        return OracleGraph(self, h, n)

    def graph_from_csr(self, n, off, tgt, keep=False):
        off = np.ascontiguousarray(off, np.int64)
        tgt = _i32(tgt)
        h = C.c_void_p()
        self._check(self.lib.lro_graph_from_csr(n, _p(off, I64P), _p(tgt, I32P), int(keep), C.byref(h)))
        return OracleGraph(self, h, n)

    def iteration_cap(self, c, tol):
        return self.lib.lro_iteration_cap(c, tol)

    def error_bound(self, large, n, c, tol):
        out = np.zeros(2)
        self.lib.lro_error_bound(large, n, c, tol, _p(out, F64P))
        return float(out[0]), float(out[1])

    def normalize_r1(self, r3):
        r3 = _f64(r3)
        out = np.zeros_like(r3)
        self._check(self.lib.lro_normalize_r1(_p(r3, F64P), len(r3), _p(out, F64P)))
        return out


class OracleGraph:
    def __init__(self, o: Oracle, h, n):
        self.o, self.h, self.n = o, h, n
        self._sched = {}

    def __del__(self):
        try:
            for s in self._sched.values():
                self.o.lib.lro_schedule_free(s)
            self.o.lib.lro_graph_free(self.h)
        except Exception:
            pass

    @property
    def m(self):
        return int(self.o.lib.lro_graph_edges(self.h))

    def csr(self):
        off = np.zeros(self.n + 1, np.int64)
        tgt = np.zeros(self.m, np.int32)
        loop = np.zeros(self.n, np.uint8)
        deg = np.zeros(self.n, np.int32)
        self.o.lib.lro_graph_csr(self.h, _p(off, I64P), _p(tgt, I32P), _p(loop, U8P), _p(deg, I32P))
        return off, tgt, loop, deg

    def partition(self, merge=True) -> PartitionOut:
        n = self.n
        comp = np.zeros(n, np.int32)
        kinds, levels, sizes = (np.zeros(max(n, 1), np.int32) for _ in range(3))
        k, ml = C.c_int32(), C.c_int32()
        st = np.zeros(3, np.int64)
        self.o._check(self.o.lib.lro_find_components(self.h, int(merge), _p(comp, I32P), _p(kinds, I32P),
                                                     _p(levels, I32P), _p(sizes, I32P), C.byref(k),
                                                     C.byref(ml), _p(st, I64P)))
        k = k.value
        return PartitionOut(comp, kinds[:k].copy(), levels[:k].copy(), sizes[:k].copy(), ml.value, tuple(st))

    def _sched_handle(self, threshold):
        if threshold not in self._sched:
            h = C.c_void_p()
            self.o._check(self.o.lib.lro_schedule_new(self.h, threshold, C.byref(h)))
            self._sched[threshold] = h
        return self._sched[threshold]

    def schedule(self, threshold=100) -> ScheduleOut:
        h = self._sched_handle(threshold)
        sizes = np.zeros(8, np.int64)
        self.o.lib.lro_schedule_sizes(h, _p(sizes, I64P))
        arr = _sched_arrays(sizes)
        self.o.lib.lro_schedule_get(h, *[_ptr(arr[k]) for k in _SCHED_ORDER])
        return ScheduleOut(**arr, intra=int(sizes[5]), cross=int(sizes[6]), dropped=int(sizes[7]))

    def compute_pagerank(self, w, c=0.85, tol=1e-9, threshold=100) -> SolveOut:
        w = _f64(w)
        ranks = np.zeros(len(w))
        rep = Report()
        cap = self.n + 1
        it = np.zeros(cap, np.int64)
        kd = np.zeros(cap, np.int32)
        self.o._check(self.o.lib.lro_compute_pagerank(self.h, _p(w, F64P), len(w), c, tol, threshold,
                                                      _p(ranks, F64P), C.byref(rep), _p(it, I64P),
                                                      _p(kd, I32P), cap))
        nu = rep.n_units
        return SolveOut(ranks, rep.as_dict(), it[:nu].copy(), kd[:nu].copy())

    def compute_baseline(self, w, c=0.85, tol=1e-9):
        w = _f64(w)
        ranks = np.zeros(len(w))
        rep = Report()
        self.o._check(self.o.lib.lro_compute_baseline(self.h, _p(w, F64P), len(w), c, tol, _p(ranks, F64P),
                                                      C.byref(rep)))
        return ranks, rep.as_dict()

    def sample_large_scc(self, w, c, iters, threshold=100):
        h = self._sched_handle(threshold)
        w = _f64(w)
        eu = C.c_int64()
        ms = C.c_double()
        self.o._check(self.o.lib.lro_sample_large_scc(self.h, h, _p(w, F64P), c, iters, C.byref(eu), C.byref(ms)))
        return eu.value, ms.value


class Ref(_Lib):
    """The reference levelrank compiled from its own sources (oracle/_ref)."""

    prefix = "lrref_"

    @staticmethod
    def available(path=REF_SO):
        return os.path.exists(path)

    def __init__(self, path=REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        lib = C.CDLL(path)
        self.lib = lib
        lib.lrref_last_error.restype = C.c_char_p
        lib.lrref_graph_new.argtypes = [C.c_int32, I32P, I32P, C.c_int64, C.c_int]
        lib.lrref_graph_new.restype = C.c_void_p
        lib.lrref_graph_free.argtypes = [C.c_void_p]
        lib.lrref_graph_parse.argtypes = [C.c_char_p, C.c_int64, C.c_int]
        lib.lrref_graph_parse.restype = C.c_void_p
        lib.lrref_graph_vertex_count.argtypes = [C.c_void_p]
        lib.lrref_graph_vertex_count.restype = C.c_int32
        lib.lrref_graph_edge_count.argtypes = [C.c_void_p]
        lib.lrref_graph_edge_count.restype = C.c_int64
        lib.lrref_graph_csr.argtypes = [C.c_void_p, I64P, I32P, U8P, I32P]
        lib.lrref_partition_new.argtypes = [C.c_void_p, C.c_int]
        lib.lrref_partition_new.restype = C.c_void_p
        lib.lrref_partition_free.argtypes = [C.c_void_p]
        lib.lrref_partition_count.argtypes = [C.c_void_p]
        lib.lrref_partition_count.restype = C.c_int64
        lib.lrref_partition_get.argtypes = [C.c_void_p, I32P, I32P, I32P, I32P, I32P, I64P]
        lib.lrref_validate_partition.argtypes = [C.c_void_p, C.c_void_p]
        lib.lrref_schedule_new.argtypes = [C.c_void_p, C.c_void_p, C.c_int32]
        lib.lrref_schedule_new.restype = C.c_void_p
        lib.lrref_schedule_free.argtypes = [C.c_void_p]
        lib.lrref_schedule_sizes.argtypes = [C.c_void_p, I64P]
        lib.lrref_schedule_get.argtypes = [C.c_void_p] + [I32P, I32P, I64P, I32P, I32P, I32P, I64P, I64P] + [I32P] * 7
        lib.lrref_compute_pagerank.argtypes = [C.c_void_p, F64P, C.c_int64, C.c_double, C.c_double, C.c_int,
                                               C.c_int32, C.c_int, F64P, C.POINTER(Report), I64P, I32P,
                                               C.c_int64]
        lib.lrref_compute_baseline.argtypes = [C.c_void_p, F64P, C.c_int64, C.c_double, C.c_double, F64P,
                                               C.POINTER(Report)]
        lib.lrref_oracle_bridge.argtypes = [C.c_void_p, F64P, C.c_int64, C.c_double, F64P, F64P, F64P]
        lib.lrref_dense_whole.argtypes = [C.c_void_p, F64P, C.c_int64, C.c_double, F64P]
        lib.lrref_iteration_cap.argtypes = [C.c_double, C.c_double]
        lib.lrref_iteration_cap.restype = C.c_int64
        lib.lrref_error_bound.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_double, F64P]
        lib.lrref_propagate.argtypes = [I32P, I32P, I32P, C.c_int64, F64P, C.c_int64, C.c_double, F64P]
        CPP = C.POINTER(C.c_char)
        lib.lrref_report_format.argtypes = [C.POINTER(Report), C.c_char_p, C.c_char_p, C.c_double, C.c_double,
                                            C.c_int, C.c_int32, C.c_int, C.c_void_p, C.c_int64, C.c_int, I64P]
        lib.lrref_report_format.restype = CPP
        lib.lrref_ranks_format.argtypes = [F64P, C.c_int64, I64P]
        lib.lrref_ranks_format.restype = CPP
        lib.lrref_string_free.argtypes = [CPP]
        lib.lrref_solve_unit.argtypes = [C.c_void_p, C.c_int, I32P, C.c_int32, I32P, I32P, C.c_int64, F64P, C.c_double,
                                         C.c_double, F64P, I64P, I64P]
        lib.lrref_large_scc_stats.argtypes = [C.c_void_p, I32P, C.c_int32, I32P, I32P, C.c_int64, F64P, C.c_double,
                                              C.c_double, F64P, I64P, F64P, C.c_int64, I64P, F64P]
        lib.lrref_prep_new.argtypes = [C.c_void_p, C.c_int32]
        lib.lrref_prep_new.restype = C.c_void_p
        lib.lrref_prep_free.argtypes = [C.c_void_p]
        lib.lrref_prep_solve.argtypes = [C.c_void_p, C.c_void_p, F64P, C.c_int64, C.c_double, C.c_double,
                                         C.c_double, C.c_int, F64P, I64P, I64P, F64P]

    def graph(self, n, src, dst, keep=False):
        src, dst = _i32(src), _i32(dst)
        h = self.lib.lrref_graph_new(n, _p(src, I32P), _p(dst, I32P), len(src), int(keep))
        if not h:
            raise ValueError(self._err())
        return RefGraph(self, h, n)

    def parse(self, data: bytes, dense_ids=True):
        """parse_edge_list; returns RefGraph, or raises ValueError(message)."""
        h = self.lib.lrref_graph_parse(data, len(data), int(dense_ids))
        if not h:
            raise ValueError(self._err())
        return RefGraph(self, h, int(self.lib.lrref_graph_vertex_count(h)))

    def iteration_cap(self, c, tol):
        return self.lib.lrref_iteration_cap(c, tol)

    def error_bound(self, large, n, c, tol):
        out = np.zeros(2)
        self.lib.lrref_error_bound(large, n, c, tol, _p(out, F64P))
        return float(out[0]), float(out[1])

    def _string(self, p, n):
        if not p:
            raise RuntimeError("format unavailable")
        try:
            return C.string_at(p, n).decode()
        finally:
            self.lib.lrref_string_free(p)

    def format_report(self, report: dict, units=(), fmt="text"):
        """The reference's SolveReport::write_text / write_json (report.cpp) or the
        bench CSV row of cli.cpp:271-275, on the given field values."""
        r = Report()
        for k, _ in REPORT_FIELDS:
            if k == "largest_is_scc":
                r.largest_is_scc = int(report.get("largest_component_kind", "cac") == "scc")
            elif k in report and report[k] is not None:
                setattr(r, k, type(getattr(r, k))(report[k]))
        rec = np.zeros(max(len(units), 1), dtype=[("kind", "i4"), ("level", "i4"), ("size", "i4"), ("r", "i4"),
                                                  ("edges", "i8"), ("iterations", "i8"), ("wall_ms", "f8")])
        for i, u in enumerate(units):
            rec[i] = (u[0], u[1], u[2], 0, u[3], u[4], u[5])
        n = C.c_int64()
        code = {"text": 0, "json": 1, "csv_row": 2}[fmt]
        p = self.lib.lrref_report_format(C.byref(r), str(report.get("method", "partitioned")).encode(),
                                         str(report.get("mode", "sequential")).encode(), float(report.get("c", 0.85)),
                                         float(report.get("tol", 1e-9)), int(report.get("keep_loops", 0)),
                                         int(report.get("small_threshold", 100)), int(report.get("threads", 1)),
                                         rec.ctypes.data, len(units), code, C.byref(n))
        return self._string(p, n.value)

    def format_ranks(self, ranks):
        ranks = _f64(ranks)
        n = C.c_int64()
        return self._string(self.lib.lrref_ranks_format(_p(ranks, F64P), len(ranks), C.byref(n)), n.value)

    def propagate(self, src, dst, deg, ranks, c, weights):
        src, dst, deg = _i32(src), _i32(dst), _i32(deg)
        ranks = _f64(ranks)
        w = _f64(weights).copy()
        self.lib.lrref_propagate(_p(src, I32P), _p(dst, I32P), _p(deg, I32P), len(src), _p(ranks, F64P),
                                 len(ranks), c, _p(w, F64P))
        return w


class RefGraph:
    def __init__(self, r: Ref, h, n):
        self.r, self.h, self.n = r, h, n

    def __del__(self):
        try:
            self.r.lib.lrref_graph_free(self.h)
        except Exception:
            pass

    @property
    def m(self):
        return int(self.r.lib.lrref_graph_edge_count(self.h))

    def csr(self):
        off = np.zeros(self.n + 1, np.int64)
        tgt = np.zeros(self.m, np.int32)
        loop = np.zeros(self.n, np.uint8)
        deg = np.zeros(self.n, np.int32)
        self.r.lib.lrref_graph_csr(self.h, _p(off, I64P), _p(tgt, I32P), _p(loop, U8P), _p(deg, I32P))
        return off, tgt, loop, deg

    def _partition_handle(self, mode):
        h = self.r.lib.lrref_partition_new(self.h, mode)
        if not h:
            raise RuntimeError(self.r._err())
        return h

    def partition(self, mode=0) -> PartitionOut:
        """mode 0 find_components, 1 find_components_scc_only, 2 reference_partition."""
        h = self._partition_handle(mode)
        try:
            k = int(self.r.lib.lrref_partition_count(h))
            comp = np.zeros(self.n, np.int32)
            kinds, levels, sizes = (np.zeros(max(k, 1), np.int32) for _ in range(3))
            ml = C.c_int32()
            st = np.zeros(3, np.int64)
            self.r.lib.lrref_partition_get(h, _p(comp, I32P), _p(kinds, I32P), _p(levels, I32P),
                                           _p(sizes, I32P), C.byref(ml), _p(st, I64P))
            return PartitionOut(comp, kinds[:k].copy(), levels[:k].copy(), sizes[:k].copy(), ml.value,
                                tuple(st) if mode == 0 else None)
        finally:
            self.r.lib.lrref_partition_free(h)

    def solve_unit(self, kind, ids, es, ed, w, c, tol):
        """The reference's solve_singletons / solve_cac / solve_small_scc /
        solve_large_scc (kind 0-3) -> (ranks, iterations, edge_visits)."""
        ids, es, ed, w = _i32(ids), _i32(es), _i32(ed), _f64(w)
        out = np.zeros(len(ids))
        it, vis = C.c_int64(), C.c_int64()
        self.r._check(self.r.lib.lrref_solve_unit(self.h, int(kind), _p(ids, I32P), len(ids), _p(es, I32P),
                                                  _p(ed, I32P), len(es), _p(w, F64P), c, tol, _p(out, F64P),
                                                  C.byref(it), C.byref(vis)))
        return out, it.value, vis.value

    def large_scc_stats(self, ids, es, ed, w, c, tol, cap=4096):
        """solve_large_scc with PowerSeriesStats -> (ranks, iterations, l1 norms, min entry)."""
        ids, es, ed, w = _i32(ids), _i32(es), _i32(ed), _f64(w)
        out, l1 = np.zeros(len(ids)), np.zeros(cap)
        it, n1, mn = C.c_int64(), C.c_int64(), C.c_double()
        self.r._check(self.r.lib.lrref_large_scc_stats(self.h, _p(ids, I32P), len(ids), _p(es, I32P), _p(ed, I32P),
                                                       len(es), _p(w, F64P), c, tol, _p(out, F64P), C.byref(it),
                                                       _p(l1, F64P), cap, C.byref(n1), C.byref(mn)))
        return out, it.value, l1[:min(n1.value, cap)].copy(), mn.value

    def validate_partition(self):
        h = self._partition_handle(0)
        try:
            return int(self.r.lib.lrref_validate_partition(self.h, h))
        finally:
            self.r.lib.lrref_partition_free(h)

    def schedule(self, threshold=100) -> ScheduleOut:
        ph = self._partition_handle(0)
        try:
            sh = self.r.lib.lrref_schedule_new(self.h, ph, threshold)
            if not sh:
                raise ValueError(self.r._err())
            try:
                sizes = np.zeros(8, np.int64)
                self.r.lib.lrref_schedule_sizes(sh, _p(sizes, I64P))
                arr = _sched_arrays(sizes)
                self.r.lib.lrref_schedule_get(sh, *[_ptr(arr[k]) for k in _SCHED_ORDER])
                return ScheduleOut(**arr, intra=int(sizes[5]), cross=int(sizes[6]), dropped=int(sizes[7]))
            finally:
                self.r.lib.lrref_schedule_free(sh)
        finally:
            self.r.lib.lrref_partition_free(ph)

    def compute_pagerank(self, w, c=0.85, tol=1e-9, threshold=100, parallel=False, threads=0) -> SolveOut:
        w = _f64(w)
        ranks = np.zeros(len(w))
        rep = Report()
        cap = self.n + 1
        it = np.zeros(cap, np.int64)
        kd = np.zeros(cap, np.int32)
        self.r._check(self.r.lib.lrref_compute_pagerank(self.h, _p(w, F64P), len(w), c, tol, int(parallel),
                                                        threshold, threads, _p(ranks, F64P), C.byref(rep),
                                                        _p(it, I64P), _p(kd, I32P), cap))
        nu = rep.n_units
        return SolveOut(ranks, rep.as_dict(), it[:nu].copy(), kd[:nu].copy())

    def compute_baseline(self, w, c=0.85, tol=1e-9):
        w = _f64(w)
        ranks = np.zeros(len(w))
        rep = Report()
        self.r._check(self.r.lib.lrref_compute_baseline(self.h, _p(w, F64P), len(w), c, tol, _p(ranks, F64P),
                                                        C.byref(rep)))
        return ranks, rep.as_dict()

    def oracle_bridge(self, w, c=0.85):
        w = _f64(w)
        r1, r3 = np.zeros(len(w)), np.zeros(len(w))
        d = C.c_double()
        self.r._check(self.r.lib.lrref_oracle_bridge(self.h, _p(w, F64P), len(w), c, _p(r1, F64P),
                                                     _p(r3, F64P), C.byref(d)))
        return r1, r3, d.value

    def dense_whole(self, w, c=0.85):
        w = _f64(w)
        out = np.zeros(len(w))
        self.r._check(self.r.lib.lrref_dense_whole(self.h, _p(w, F64P), len(w), c, _p(out, F64P)))
        return out

    # -- bench reference arm
    def prepare(self, threshold=100):
        h = self.r.lib.lrref_prep_new(self.h, threshold)
        if not h:
            raise RuntimeError(self.r._err())
        return h

    def free_prep(self, h):
        self.r.lib.lrref_prep_free(h)

    def prep_solve(self, prep, w, c, tol, large_tol=0.0, threads=1):
        w = _f64(w)
        ranks = np.zeros(len(w))
        work, iters, ms = C.c_int64(), C.c_int64(), C.c_double()
        self.r._check(self.r.lib.lrref_prep_solve(self.h, prep, _p(w, F64P), len(w), c, tol, large_tol, threads,
                                                  _p(ranks, F64P), C.byref(work), C.byref(iters), C.byref(ms)))
        return ranks, work.value, iters.value, ms.value
