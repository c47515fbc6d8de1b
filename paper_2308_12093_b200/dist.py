"""1-D destination-row partitioned GCN layer across the ranks of a
torch.distributed group (NCCL over NVLink on B200; gloo in the CPU tests).

North-star row (e) / SURVEY 8(e): destination rows are split into P contiguous
blocks balanced by nnz.  Rank p owns
  * A'_p   -- rows [r0, r1) of A' (all columns), CSR, for A' . B
  * A'T_p  -- rows [r0, r1) of A'^T (= columns [r0, r1) of A'), for A'^T . B
  * its row block of X / dX' / out, and replicated parameters.
Every propagation of a dense operand B needs all rows of B: one all-gather per
SpMM (the exchange step); parameter gradients are all-reduced.  Accumulation
order inside each output row is the reference's (ascending column), so the
SpMM blocks are bit-identical to the single-GPU product.

The compute backend is pluggable (`ops`): DeviceOps runs libsgnn_cuda.so on
the rank's GPU; tests inject a CPU implementation to exercise the partition
and collective logic under gloo.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


# ---------------------------------------------------------------------------
# host-side partition logic
# ---------------------------------------------------------------------------
def partition_rows(rowptr, parts):
    """nnz-balanced contiguous row blocks: bounds[p] .. bounds[p+1]."""
    rowptr = np.asarray(rowptr, dtype=np.int64)
    n = len(rowptr) - 1
    q = int(rowptr[-1])
    bounds = [0]
    for p in range(1, parts):
        target = (q * p) // parts
        r = int(np.searchsorted(rowptr, target, side="left"))
        r = min(max(r, bounds[-1]), n)
        bounds.append(r)
    bounds.append(n)
    return bounds


def row_block(rows, cols, vals, r0, r1):
    """Entries of canonical COO with row in [r0, r1): (local row, global col, val)."""
    rows = np.asarray(rows)
    lo = int(np.searchsorted(rows, r0, side="left"))
    hi = int(np.searchsorted(rows, r1, side="left"))
    return (rows[lo:hi] - r0).astype(np.int32), np.asarray(cols)[lo:hi].astype(np.int32), \
        np.asarray(vals)[lo:hi]


def transposed_block(rows, cols, vals, r0, r1):
    """Rows [r0, r1) of A^T = entries with col in [r0, r1), as canonical COO
    (local row = col - r0, global col = row), ordered by (col, row): the CSC
    order of the reference (rows ascend within a column, sparse.hpp:207-216)."""
    rows, cols, vals = np.asarray(rows), np.asarray(cols), np.asarray(vals)
    m = (cols >= r0) & (cols < r1)
    r, c, v = cols[m] - r0, rows[m], vals[m]
    order = np.lexsort((c, r))
    return r[order].astype(np.int32), c[order].astype(np.int32), v[order]


# ---------------------------------------------------------------------------
# compute backends
# ---------------------------------------------------------------------------
class DeviceOps:
    """libsgnn_cuda.so on this rank's GPU (fails loudly without it)."""

    def __init__(self, device):
        from . import device as d

        self.d = d
        self.dev = torch.device(device)

    def adjacency(self, n_rows, n_cols, rows, cols, vals, dtype):
        d = self.d
        t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(self.dev, dt)  # noqa: E731
        return d.Adjacency(n_rows, n_cols, t(rows, torch.int32), t(cols, torch.int32),
                           t(vals, dtype), "csr")

    def spmm(self, adj, B, bias=None):
        return adj.spmm(B.contiguous(), bias=bias)

    def gemm(self, A, B, ta=False, tb=False, bias=None):
        out = self.d.gemm(A, B, ta, tb)
        return out if bias is None else out + bias

    def colsum(self, X):
        return self.d.column_sums(X)


# ---------------------------------------------------------------------------
# collectives over uneven row blocks
# ---------------------------------------------------------------------------
def all_gather_rows(local, bounds, group=None):
    """Concatenate every rank's row block (padded to the largest block)."""
    world = len(bounds) - 1
    sizes = [bounds[p + 1] - bounds[p] for p in range(world)]
    mx = max(sizes)
    f = local.shape[1]
    pad = torch.zeros((mx, f), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    buf = torch.empty((world * mx, f), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(buf, pad, group=group)
    return torch.cat([buf[p * mx: p * mx + sizes[p]] for p in range(world)], 0)


def all_reduce_sum(t, group=None):
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


# ---------------------------------------------------------------------------
# partitioned GCN layer (gcn.hpp:91-193 over row blocks)
# ---------------------------------------------------------------------------
class DistGcnLayer:
    """One GCN layer over a row-partitioned normalized operator.

    rows/cols/vals: the full canonical normalized COO of A' (host arrays; every
    rank builds only its blocks).  scheme: (forward, backward, caching) ints of
    the reference's SchemeChoice (resolve with device.resolve_scheme).
    """

    def __init__(self, n, rows, cols, vals, ops, dtype=torch.float32, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        rowptr = np.zeros(n + 1, np.int64)
        np.add.at(rowptr, np.asarray(rows, np.int64) + 1, 1)
        rowptr = np.cumsum(rowptr)
        self.n = n
        self.bounds = partition_rows(rowptr, self.world)
        self.r0, self.r1 = self.bounds[self.rank], self.bounds[self.rank + 1]
        self.ops = ops
        nl = self.r1 - self.r0
        self.A = ops.adjacency(nl, n, *row_block(rows, cols, vals, self.r0, self.r1), dtype)
        self.AT = ops.adjacency(nl, n, *transposed_block(rows, cols, vals, self.r0, self.r1),
                                dtype)

    def forward(self, X_local, theta, bias, scheme):
        fwd = scheme[0]
        ops = self.ops
        cache = {"scheme": scheme}
        if fwd == 0:  # transform-first: M = X Theta, gather M, out = A'_p M + b
            M_local = ops.gemm(X_local, theta)
            M = all_gather_rows(M_local, self.bounds, self.group)
            out = ops.spmm(self.A, M, bias)
            cache["X"] = X_local
        else:  # propagate-first: gather X, P_p = A'_p X, out = P_p Theta + b
            X = all_gather_rows(X_local, self.bounds, self.group)
            P = ops.spmm(self.A, X)
            out = ops.gemm(P, theta, bias=bias)
            if fwd == 2:
                cache["P"] = P
            else:
                cache["X"] = X_local
        return out, cache

    def backward(self, G_local, theta, cache, needs_feature_grad):
        ops = self.ops
        bwd = cache["scheme"][1]
        d_bias = all_reduce_sum(ops.colsum(G_local), self.group)
        d_input = None
        if bwd == 0:  # fused: S = A'^T G (rows of my block), dTheta = X^T S
            G = all_gather_rows(G_local, self.bounds, self.group)
            S = ops.spmm(self.AT, G)
            d_theta = all_reduce_sum(ops.gemm(cache["X"], S, ta=True), self.group)
            if needs_feature_grad:
                d_input = ops.gemm(S, theta, tb=True)
        else:
            if bwd == 1:  # split: recompute P_p = A'_p X
                X = all_gather_rows(cache["X"], self.bounds, self.group)
                P = ops.spmm(self.A, X)
            else:
                P = cache["P"]
            d_theta = all_reduce_sum(ops.gemm(P, G_local, ta=True), self.group)
            if needs_feature_grad:
                G2 = all_gather_rows(ops.gemm(G_local, theta, tb=True), self.bounds, self.group)
                d_input = ops.spmm(self.AT, G2)
        return d_theta, d_bias, d_input
