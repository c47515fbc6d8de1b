"""Algorithmic (compulsory) bytes of a GCN / GAT layer step: the sum of its
kernels' compulsory traffic, DESIGN.md §3 (SpMM 4(n+1)+8q'+8nf, GEMM
4(rows K + K N + rows N), the GAT kernels as listed there).  Pure functions,
used by scripts/sweep.py and bench.py's large-graph lines."""


def spmm_b(n, q, f):
    return 4 * (n + 1) + 8 * q + 8 * n * f


def gemm_b(r, kk, c):
    return 4 * (r * kk + kk * c + r * c)


def gcn_step_bytes(s, n, q, m, k, fg):
    f, b = s.forward, s.backward
    by = gemm_b(n, m, k) + (spmm_b(n, q, k) if f == 0 else spmm_b(n, q, m))
    if b == 0:  # fused: colsum, S = A'^T G, X^T S, S Theta^T
        by += 4 * n * k + spmm_b(n, q, k) + 4 * (n * m + n * k + m * k)
        by += gemm_b(n, k, m) if fg else 0
    else:  # split (P recomputed) / cached: P^T G (+colsum), G Theta^T, A'^T G2
        by += spmm_b(n, q, m) if b == 1 else 0
        by += 4 * (n * m + n * k + m * k)
        by += (gemm_b(n, k, m) + spmm_b(n, q, m)) if fg else 0
    return by


def gat_step_bytes(level, n, q, m, h, k):
    hk = h * k
    pat = 4 * (n + 1) + 4 * q
    attn = pat + 8 * n * h + 4 * q * h + q * h  # s, d in; alpha (+ mask) out
    fwd = gemm_b(n, m, hk) + 8 * n * h + attn + pat + 4 * q * h + 8 * n * hk
    lv = ["none", "features", "node-attn", "full"].index(level)
    rec = 0
    if lv < 1:
        rec += gemm_b(n, m, hk) + 8 * n * h
    elif lv < 2:
        rec += 4 * n * hk + 8 * n * h  # node scores from the cached M
    if lv < 3:
        rec += attn
    bwd = rec + (pat + 8 * n * hk + 4 * q * h)  # SDDMM
    bwd += 4 * (n + 1) + 13 * q * h + 4 * n * h  # softmax / LeakyReLU backward, dS
    bwd += 4 * (n + 1) + 8 * q + 8 * q * h + 8 * n * hk + 8 * n * h  # column pass
    bwd += 8 * n * hk + 8 * n * h  # d_bias, d_a_src, d_a_dst
    bwd += 4 * (n * m + n * hk + m * hk) + gemm_b(n, hk, m)  # dTheta, dX
    return fwd + bwd
