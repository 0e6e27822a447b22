"""The multi-GPU path's host logic on CPU (gloo, world size 2).

Per level the rows of the CTA-solved units are split over the ranks
(lr_split_level_rows), each rank solving its range, and the ranges are
broadcast from their owners (exchange_level).  The sharded solve in
csrc/cuda/ctx.cu splits every grid SccLarge unit into
nnz-balanced row shards, each cut into exchange chunks (lr_exchange_cuts);
per iteration it computes chunk j of its own rows and broadcasts every rank's
chunk j (roots in rank order) while the next chunk computes, all-reduces the
shard maxima after the last chunk, and only then takes the common stop
decision; the final rank shards are broadcast before lower levels read them.
This test replays that exact schedule (the library's cuts, the same
collective order) over torch.distributed/gloo with a scalar host SpMV standing
in for the kernel, on the real layout, and checks it reproduces the
single-process oracle: same per-unit iteration counts, bit-identical R3 (no
SccSmall units in these graphs).
"""
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHUNKS = 3  # exchange chunks per shard (LR_XCHG_CHUNKS on the GPU path)


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
        # the level's rows split over the ranks (lr_split_level_rows, as the
        # device does with LR_DIST_MIN_ROWS=0): each rank computes the start
        # weights and solves the one-pass units of its range ...
        split = lr.split_level_rows(L, li, world)
        my0, my1 = int(split[rank]), int(split[rank + 1])
        for r in range(my0, my1):
            acc = w[vert[r]]
            for e in range(L["xptr"][r], L["xptr"][r + 1]):
                s = L["xsrc"][e]
                acc += c * rankv[s] / float(deg[s])
            if kind_of_row[r - rb] == 0 and L["loop"][r]:
                acc /= 1.0 - c / float(deg[r])
            rankv[r] = acc
        for u in range(L["level_unit_begin"][li], L["level_unit_begin"][li + 1]):
            a, b = urb[u], urb[u + 1]
            if kinds[u] == 1 and not my0 <= a < my1:
                continue
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
        # ... then every range is broadcast from its owner (ctx.cu exchange_level)
        for q in range(world):
            q0, q1 = int(split[q]), int(split[q + 1])
            if q1 > q0:
                t = torch.from_numpy(rankv[q0:q1].copy())
                dist.broadcast(t, src=q)
                rankv[q0:q1] = t.numpy()
        for u in range(L["level_unit_begin"][li], L["level_unit_begin"][li + 1]):
            a, b = urb[u], urb[u + 1]
            if kinds[u] != 3:
                continue
            # sharded power series of one SccLarge unit, on the library's own
            # schedule: lr_exchange_cuts gives every rank's shard cut into
            # exchange chunks; per iteration chunk j is computed, then every
            # rank's chunk j is broadcast (roots in rank order), the last chunk
            # followed by the all-reduce of the maxima (ctx.cu chunked_iteration)
            cuts = lr.exchange_cuts(L["iptr"], a, b, world, CHUNKS)
            bounds = [int(cuts[q * CHUNKS]) for q in range(world)] + [int(b)]
            assert np.array_equal(bounds, lr.shard_rows(L["iptr"], a, b, world))
            pf = np.array([c / float(deg[r]) for r in range(a, b)])
            s_cur = pf * rankv[a:b]
            it = 0
            while True:
                s_next = np.zeros(b - a)
                mx_local = 0.0
                for j in range(CHUNKS):
                    for r in range(cuts[rank * CHUNKS + j], cuts[rank * CHUNKS + j + 1]):
                        acc = 0.0
                        for e in range(L["iptr"][r], L["iptr"][r + 1]):
                            acc += s_cur[L["isrc"][e] - a]
                        rankv[r] = rankv[r] + acc
                        s_next[r - a] = pf[r - a] * acc
                        mx_local = max(mx_local, acc)
                    for q in range(world):
                        q0, q1 = int(cuts[q * CHUNKS + j]), int(cuts[q * CHUNKS + j + 1])
                        if q1 > q0:
                            t = torch.from_numpy(s_next[q0 - a:q1 - a].copy())
                            dist.broadcast(t, src=q)
                            s_next[q0 - a:q1 - a] = t.numpy()
                mx = torch.tensor([mx_local], dtype=torch.float64)
                dist.all_reduce(mx, op=dist.ReduceOp.MAX)
                s_cur = s_next
                it += 1
                if it > cap:
                    raise RuntimeError("power series failed to converge")
                if not (mx.item() >= tol):
                    break
            iters[u] = it
            # replicate the final ranks of the unit: each rank's shard broadcast
            for q in range(world):
                t = torch.from_numpy(rankv[bounds[q]:bounds[q + 1]].copy())
                if len(t):
                    dist.broadcast(t, src=q)
                    rankv[bounds[q]:bounds[q + 1]] = t.numpy()
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
