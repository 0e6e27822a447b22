"""The C-ABI library: loads, exports every symbol include/lr_cuda.h declares,
host-only entry points behave like the reference, and the GPU path fails
loudly (no CPU fallback) when no device is present."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "lr_cuda.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lr_[a-z0-9_]+)\s*\(", text)))


def test_exports_every_declared_symbol(lr):
    so = C.CDLL(lr.library_path())
    syms = header_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(so, s)]
    assert not missing, missing
    assert set(syms) == set(lr.EXPORTS), set(syms) ^ set(lr.EXPORTS)


def test_no_oracle_in_product():
    # the product never links or loads the checker
    pkg = os.path.join(ROOT, "paper_1609_09068_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".cuh", ".hpp", ".h")) or f == "Makefile":
                txt = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "oracle" not in txt.lower().replace("oracle_r1_to_r3", ""), f


def test_helpers(lr):
    assert lr.lib().lr_version().decode().startswith("levelrank-b200")
    assert lr.iteration_cap(lr.SolverParams(0.85, 1e-9)) == 1280
    assert lr.iteration_cap(lr.SolverParams(0.85, 0.9)) == 16
    assert lr.iteration_cap(lr.SolverParams(0.5, 1e-9)) == 300
    tot, avg = lr.error_bound(1000, 10000, lr.SolverParams(0.85, 1e-9))
    assert abs(tot - 1000 * 1e-9 * 0.85 / 0.15) < 1e-18 and abs(avg - tot / 1e4) < 1e-22
    assert lr.error_bound(0, 100, lr.SolverParams()) == (0.0, 0.0)
    lr.validate_params(lr.SolverParams(0.5, 1e-9))
    for c, tol in [(0.0, 1e-9), (1.0, 1e-9), (-0.1, 1e-9), (1.5, 1e-9), (0.85, 0.0), (0.85, -1e-9)]:
        with pytest.raises(ValueError):
            lr.validate_params(lr.SolverParams(c, tol))


def test_plan_census(lr):
    from conftest import FIXTURE8
    p = lr.Plan(lr.Graph.from_edges(8, FIXTURE8), 100)
    c = p.census()
    assert (c["components"], c["scc_components"], c["cac_components"], c["singleton_cacs"], c["largest_component"],
            c["largest_is_scc"], c["max_level"], c["level_count"]) == (4, 2, 2, 1, 3, 0, 2, 3)


def _no_gpu():
    try:
        import torch
        return not torch.cuda.is_available()
    except Exception:
        return True


@pytest.mark.skipif(not _no_gpu(), reason="checks the no-GPU failure mode")
def test_fails_loudly_without_gpu(lr):
    from conftest import FIXTURE8
    g = lr.Graph.from_edges(8, FIXTURE8)
    with pytest.raises(lr.CudaError):
        lr.compute_pagerank(g, np.ones(8))
    with pytest.raises(lr.CudaError):
        lr.Engine(g)
    # argument validation still happens first, exactly like the reference
    with pytest.raises(ValueError):
        lr.compute_pagerank(g, np.ones(7))
    w = np.ones(8)
    w[2] = -1
    with pytest.raises(ValueError):
        lr.compute_pagerank(g, w)
    with pytest.raises(ValueError):
        lr.compute_pagerank(g, np.ones(8), lr.SolverParams(1.2, 1e-9))
