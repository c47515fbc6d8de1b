"""Vectorised float64 GAT layer (numpy + scipy.sparse) -- TEST INFRASTRUCTURE ONLY.

A restatement of the reference's GAT layer for full-size parity checks
(gat.hpp:89-139 forward, gat.hpp:172-219 backward; kernels.hpp:385-658 for the
node/edge scores, LeakyReLU, edge softmax, semibatched SpMM/SDDMM, row/column
sums and attention-parameter gradients).  It differs from oracle/sgnn_oracle.c
(the loop-order-exact restatement, bit-identical to the reference) only in
float64 summation order, ~1e-15 relative; tests/test_oracle_golden.py pins it
to the reference at 1e-12.

Why it exists: the LeakyReLU derivative is discontinuous at y = s_i + d_j = 0,
so an edge whose float32 score lands on the other side of zero than the float64
one (|y| ~ 1e-7) takes the other slope (1 vs beta) in the backward pass --
an O(1) change of that edge's dy that no precision bar can absorb.  Such
edges are ill-conditioned, not wrong.  `backward(..., mask=device_mask)`
evaluates the float64 gradients with the device's LeakyReLU decisions, so the
1e-4 bar measures everything else; the tests separately assert that every
decision that differs from the float64 one sits at |y| below 1e-5 of the
scores' scale.

Layouts follow the device / reference: M is n x (h*k) with the head in the
middle; edge values are edge-major q x h here (the reference's head-major
h x q is its transpose).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

_CHUNK = 1 << 17  # edges per block in the per-edge dots (bounds the temporaries)


def _rows_of(rowptr):
    n = rowptr.size - 1
    return np.repeat(np.arange(n, dtype=np.int64), np.diff(rowptr))


def forward(rowptr, cols, X, theta, a_src, a_dst, bias, heads, beta=0.2, mask=None):
    """Returns (out, state): state holds M, s, d, y, mask, alpha (edge-major)."""
    rowptr = np.asarray(rowptr, np.int64)
    cols = np.asarray(cols, np.int64)
    n = rowptr.size - 1
    hk = theta.shape[1]
    k = hk // heads
    M = np.asarray(X, np.float64) @ np.asarray(theta, np.float64)
    M3 = M.reshape(n, heads, k)
    s = np.einsum("nhk,hk->nh", M3, a_src)
    d = np.einsum("nhk,hk->nh", M3, a_dst)
    rows = _rows_of(rowptr)
    y = s[rows] + d[cols]  # q x h
    mk = (y > 0) if mask is None else np.asarray(mask, bool)
    w = np.where(mk, y, beta * y)
    starts = rowptr[:-1]
    if np.any(np.diff(rowptr) == 0):
        raise ValueError("gat_forward: pattern must contain all self loops")
    wmax = np.maximum.reduceat(w, starts, axis=0)
    ex = np.exp(w - wmax[rows])
    den = np.add.reduceat(ex, starts, axis=0)
    alpha = ex * (1.0 / den)[rows]
    out = np.empty((n, hk))
    out3 = out.reshape(n, heads, k)
    for t in range(heads):
        A = sp.csr_matrix((alpha[:, t], cols, rowptr), shape=(n, n))
        out3[:, t, :] = A @ M3[:, t, :]
    out += np.asarray(bias, np.float64)[None, :]
    return out, {"M": M, "s": s, "d": d, "y": y, "mask": mk, "alpha": alpha, "rows": rows}


def backward(rowptr, cols, G, X, theta, a_src, a_dst, heads, beta=0.2, fg=True, mask=None,
             state=None):
    """(d_theta, d_a_src, d_a_dst, d_bias, d_input or None) in float64.
    mask (q x h bool, edge-major) overrides the LeakyReLU decisions."""
    rowptr = np.asarray(rowptr, np.int64)
    cols = np.asarray(cols, np.int64)
    n = rowptr.size - 1
    hk = theta.shape[1]
    k = hk // heads
    if state is None or mask is not None:
        _, state = forward(rowptr, cols, X, theta, a_src, a_dst, np.zeros(hk), heads, beta,
                           mask)
    M3 = state["M"].reshape(n, heads, k)
    alpha, mk, rows = state["alpha"], state["mask"], state["rows"]
    G = np.asarray(G, np.float64)
    G3 = G.reshape(n, heads, k)
    q = cols.size
    da = np.empty((q, heads))
    for e0 in range(0, q, _CHUNK):
        e1 = min(q, e0 + _CHUNK)
        da[e0:e1] = np.einsum("qhk,qhk->qh", G3[rows[e0:e1]], M3[cols[e0:e1]])
    starts = rowptr[:-1]
    dot = np.add.reduceat(alpha * da, starts, axis=0)
    dw = alpha * (da - dot[rows])
    dy = np.where(mk, dw, beta * dw)
    dS = np.add.reduceat(dy, starts, axis=0)
    dD = np.zeros((n, heads))
    for t in range(heads):
        dD[:, t] = np.bincount(cols, weights=dy[:, t], minlength=n)
    dM = np.empty((n, hk))
    dM3 = dM.reshape(n, heads, k)
    for t in range(heads):
        AT = sp.csr_matrix((alpha[:, t], cols, rowptr), shape=(n, n)).T.tocsr()
        dM3[:, t, :] = AT @ G3[:, t, :]
    dM3 += dS[:, :, None] * np.asarray(a_src)[None] + dD[:, :, None] * np.asarray(a_dst)[None]
    d_a_src = np.einsum("nh,nhk->hk", dS, M3)
    d_a_dst = np.einsum("nh,nhk->hk", dD, M3)
    Xd = np.asarray(X, np.float64)
    d_theta = Xd.T @ dM
    d_bias = G.sum(axis=0)
    d_input = dM @ np.asarray(theta, np.float64).T if fg else None
    return d_theta, d_a_src, d_a_dst, d_bias, d_input


def ill_conditioned_flips(y_ref, mask_dev, rel=1e-5):
    """Edges (edge-major q x h) whose device LeakyReLU decision differs from
    the float64 one: returns (count, count with |y| above rel * scale)."""
    flips = np.asarray(mask_dev, bool) != (y_ref > 0)
    scale = np.abs(y_ref).max() if y_ref.size else 1.0
    return int(flips.sum()), int((flips & (np.abs(y_ref) > rel * scale)).sum())
