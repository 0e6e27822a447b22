"""Test helper: a literal pure-Python execution of the device Layout.

Runs the level loop exactly as the CUDA kernels do (pull CSRs, per-row
accumulation order, depth slices, row blocks) but scalar on the host, so the
layout's ordering claims can be checked bit-for-bit against the oracle
without a GPU.  Small graphs only.  Dense small-SCC units use numpy.linalg
(not bit-exact; that path is checked within tolerance).
"""
import numpy as np


def emulate(L, w, c, tol, cap, long_row=None):
    n = L["n"]
    rank = np.zeros(n)
    iters = np.zeros(L["n_units"], np.int64)
    deg = L["deg"]
    vert = L["vertex_of"]
    kinds = L["unit_kind"]
    urb = L["unit_row_begin"]
    for li in range(L["n_levels"]):
        rb, re = L["level_row_begin"][li], L["level_row_begin"][li + 1]
        kind_of_row = {}
        for u in range(L["level_unit_begin"][li], L["level_unit_begin"][li + 1]):
            for r in range(urb[u], urb[u + 1]):
                kind_of_row[r] = kinds[u]
        for r in range(rb, re):  # k_cross
            acc = w[vert[r]]
            for e in range(L["xptr"][r], L["xptr"][r + 1]):
                s = L["xsrc"][e]
                acc += c * rank[s] / float(deg[s])
            if kind_of_row[r] == 0 and L["loop"][r]:
                acc /= 1.0 - c / float(deg[r])
            rank[r] = acc
        for u in range(L["level_unit_begin"][li], L["level_unit_begin"][li + 1]):
            a, b = urb[u], urb[u + 1]
            if kinds[u] == 1:  # CAC by depth slices
                dp = L["depth_ptr"][L["cac_depth_begin"][u]:]
                d = 0
                while dp[d] < b:
                    for r in range(dp[d], dp[d + 1]):
                        acc = rank[r]
                        for e in range(L["iptr"][r], L["iptr"][r + 1]):
                            s = L["isrc"][e]
                            acc += rank[s] * c / float(deg[s])
                        if L["loop"][r]:
                            acc /= 1.0 - c / float(deg[r])
                        rank[r] = acc
                    d += 1
            elif kinds[u] == 2:
                m = b - a
                M = np.eye(m)
                for r in range(a, b):
                    for e in range(L["iptr"][r], L["iptr"][r + 1]):
                        s = L["isrc"][e]
                        M[r - a, s - a] -= c / float(deg[s])
                rank[a:b] = np.linalg.solve(M, rank[a:b].copy())
            elif kinds[u] == 3:
                pf = np.array([c / float(deg[r]) for r in range(a, b)])
                s_cur = pf * rank[a:b]
                it = 0
                while True:
                    y = np.zeros(b - a)
                    for r in range(a, b):
                        acc = 0.0
                        for e in range(L["iptr"][r], L["iptr"][r + 1]):
                            acc += s_cur[L["isrc"][e] - a]
                        y[r - a] = acc
                    rank[a:b] = rank[a:b] + y
                    s_cur = pf * y
                    it += 1
                    if it > cap:
                        raise RuntimeError("power series failed to converge")
                    if not (y.max() >= tol):
                        break
                iters[u] = it
    r3 = np.zeros(n)
    r3[vert] = rank
    return r3, iters
