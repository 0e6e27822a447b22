"""The multi-GPU path's host logic on CPU (gloo, world size 2).

The sharded solve in csrc/cuda/ctx.cu splits every grid SccLarge unit into
nnz-balanced row shards (lr_shard_rows), iterates only its own rows, then
exchanges the pushed-vector shards and all-reduces the shard maxima before the
common stop decision; the final rank shards are exchanged before lower levels
read them.  This test runs exactly that protocol over torch.distributed/gloo
with a scalar host SpMV standing in for the kernel, on the real layout, and
checks it reproduces the single-process oracle: same per-unit iteration
counts, bit-identical R3 (no SccSmall units in these graphs).
"""
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _emulate_sharded(L, w, c, tol, cap, rank, world, dist, lr):
    import torch
    n = L["n"]
    deg = L["deg"]
    vert = L["vertex_of"]
    kinds = L["unit_kind"]
    urb = L["unit_row_begin"]
    rankv = np.zeros(n)
    iters = np.zeros(L["n_units"], np.int64)
    for li in range(L["n_levels"]):
        rb, re = L["level_row_begin"][li], L["level_row_begin"][li + 1]
        kind_of_row = np.zeros(re - rb, np.int64)
        for u in range(L["level_unit_begin"][li], L["level_unit_begin"][li + 1]):
            kind_of_row[urb[u] - rb:urb[u + 1] - rb] = kinds[u]
        for r in range(rb, re):  # replicated on every rank
            acc = w[vert[r]]
            for e in range(L["xptr"][r], L["xptr"][r + 1]):
                s = L["xsrc"][e]
                acc += c * rankv[s] / float(deg[s])
            if kind_of_row[r - rb] == 0 and L["loop"][r]:
                acc /= 1.0 - c / float(deg[r])
            rankv[r] = acc
        for u in range(L["level_unit_begin"][li], L["level_unit_begin"][li + 1]):
            a, b = urb[u], urb[u + 1]
            if kinds[u] == 1:
                dp = L["depth_ptr"][L["cac_depth_begin"][u]:]
                d = 0
                while dp[d] < b:
                    for r in range(dp[d], dp[d + 1]):
                        acc = rankv[r]
                        for e in range(L["iptr"][r], L["iptr"][r + 1]):
                            s = L["isrc"][e]
                            acc += rankv[s] * c / float(deg[s])
                        if L["loop"][r]:
                            acc /= 1.0 - c / float(deg[r])
                        rankv[r] = acc
                    d += 1
                continue
            if kinds[u] != 3:
                continue
            # sharded power series of one SccLarge unit
            bounds = lr.shard_rows(L["iptr"], a, b, world)
            o0, o1 = bounds[rank], bounds[rank + 1]
            pf = np.array([c / float(deg[r]) for r in range(a, b)])
            s_cur = pf * rankv[a:b]
            pad = int(np.max(np.diff(bounds)))
            it = 0
            while True:
                y = np.zeros(o1 - o0)
                for r in range(o0, o1):
                    acc = 0.0
                    for e in range(L["iptr"][r], L["iptr"][r + 1]):
                        acc += s_cur[L["isrc"][e] - a]
                    y[r - o0] = acc
                rankv[o0:o1] = rankv[o0:o1] + y
                shard = np.zeros(pad)
                shard[:o1 - o0] = pf[o0 - a:o1 - a] * y
                parts = [torch.zeros(pad, dtype=torch.float64) for _ in range(world)]
                dist.all_gather(parts, torch.from_numpy(shard))
                s_cur = np.concatenate([parts[q].numpy()[:bounds[q + 1] - bounds[q]] for q in range(world)])
                mx = torch.tensor([y.max() if len(y) else 0.0], dtype=torch.float64)
                dist.all_reduce(mx, op=dist.ReduceOp.MAX)
                it += 1
                if it > cap:
                    raise RuntimeError("power series failed to converge")
                if not (mx.item() >= tol):
                    break
            iters[u] = it
            # replicate the final ranks of the unit
            shard = np.zeros(pad)
            shard[:o1 - o0] = rankv[o0:o1]
            parts = [torch.zeros(pad, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(parts, torch.from_numpy(shard))
            rankv[a:b] = np.concatenate([parts[q].numpy()[:bounds[q + 1] - bounds[q]] for q in range(world)])
    r3 = np.zeros(n)
    r3[vert] = rankv
    return r3, iters


def _worker(rank, world, port, cfg, shrink, result_path):
    import sys
    sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
    import torch.distributed as dist

    import paper_1609_09068_b200 as lr
    from oracle_py import Oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = lr.config_graph(cfg, shrink)
        L = lr.Plan(g, 100).layout()
        w = np.full(g.n, 1.0 / g.n)
        o = Oracle()
        cap = o.iteration_cap(0.85, 1e-12)
        r3, it = _emulate_sharded(L, w, 0.85, 1e-12, cap, rank, world, dist, lr)
        if rank == 0:
            off, tgt, _, _ = g.csr()
            ref = o.graph_from_csr(g.n, off, tgt).compute_pagerank(w, 0.85, 1e-12, 100)
            np.savez(result_path, r3=r3, it=it, ref=ref.ranks, ref_it=ref.unit_iters,
                     has_small=np.int64((L["unit_kind"] == 2).any()), n_large=np.int64((L["unit_kind"] == 3).sum()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg,shrink", [(2, 9), (3, 12)])
def test_sharded_power_series_matches_single_process(lr, tmp_path, cfg, shrink):
    import torch.multiprocessing as mp
    out = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(2, _free_port(), cfg, shrink, out), nprocs=2, join=True)
    z = np.load(out)
    assert int(z["n_large"]) >= 1, "the graph must have an iterated SCC"
    assert np.array_equal(z["it"], z["ref_it"])
    if int(z["has_small"]):
        np.testing.assert_allclose(z["r3"], z["ref"], rtol=1e-12)
    else:
        assert np.array_equal(z["r3"], z["ref"])


def test_shard_bounds_balanced(lr):
    rng = np.random.default_rng(3)
    deg = rng.zipf(1.8, 5000).clip(1, 5000)
    iptr = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
    for world in (1, 2, 3, 8):
        b = lr.shard_rows(iptr, 100, 4900, world)
        assert b[0] == 100 and b[-1] == 4900 and np.all(np.diff(b) >= 0)
        nnz = iptr[b[1:]] - iptr[b[:-1]]
        assert nnz.max() <= (iptr[4900] - iptr[100]) / world + deg.max()
