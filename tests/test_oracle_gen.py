"""The oracle-side generators (oracle/lr_gen.c, used by bench.py's CPU legs so
the reference arm never loads the product library) give the same graphs as
the product's (csrc/host/gen.cpp, lr.config_graph)."""
import numpy as np
import pytest


@pytest.mark.parametrize("cfg,shrink", [(1, 3), (1, 0), (2, 8), (3, 9), (4, 5), (5, 12)])
def test_oracle_generator_matches_product(lr, oracle, cfg, shrink):
    g = lr.config_graph(cfg, shrink)
    off, tgt, _, _ = g.csr()
    n, src, dst = oracle.gen_config(cfg, shrink, threads=3)
    assert n == g.n
    og = oracle.graph(n, src, dst)
    o_off, o_tgt, _, _ = og.csr()
    assert np.array_equal(off, o_off) and np.array_equal(tgt, o_tgt)
