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

import ctypes as C

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

    def empty(self, rows, cols, dtype):
        return torch.empty((rows, cols), dtype=dtype, device=self.dev)

    def spmm(self, adj, B, bias=None):
        return adj.spmm(B.contiguous(), bias=bias)

    def gemm(self, A, B, ta=False, tb=False, bias=None, out=None, colsum_b=None):
        """bias fused into the epilogue; colsum_b = 1^T B from the same read
        of B (C = A^T B); out may be a row range of a larger buffer."""
        return self.d.gemm(A, B, ta, tb, bias=bias, out=out, colsum_b=colsum_b)

    def colsum(self, X):
        return self.d.column_sums(X)


# ---------------------------------------------------------------------------
# partitioned GCN layer (gcn.hpp:91-193 over row blocks)
# ---------------------------------------------------------------------------
def padded_columns(cols, bounds, mx):
    """Global column j -> owner(j) * mx + (j - bounds[owner]): the row of j in
    the padded all-gather layout (world blocks of mx rows).  Monotonic in j,
    so the stored (ascending-column) order of every row is unchanged."""
    cols = np.asarray(cols, np.int64)
    b = np.asarray(bounds, np.int64)
    owner = np.searchsorted(b, cols, side="right") - 1
    return (owner * mx + (cols - b[owner])).astype(np.int32)


class DistGcnLayer:
    """One GCN layer over a row-partitioned normalized operator.

    rows/cols/vals: the full canonical normalized COO of A' (host arrays; every
    rank builds only its blocks).  scheme: (forward, backward, caching) ints of
    the reference's SchemeChoice (resolve with device.resolve_scheme).

    Gathered operands use a padded layout -- world blocks of mx = max block
    rows -- and the local operator blocks index it directly (their column ids
    are remapped once at setup), so a rank's producer (GEMM) writes its rows
    straight into its slot of the gather buffer and the all-gather is
    in place: no pad or concatenation copies, and none at all at world 1.
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
        self.mx = max(self.bounds[p + 1] - self.bounds[p] for p in range(self.world))
        self.ops, self.dtype = ops, dtype
        nl = self.r1 - self.r0
        wide = self.world * self.mx
        r, c, v = row_block(rows, cols, vals, self.r0, self.r1)
        self.A = ops.adjacency(nl, wide, r, padded_columns(c, self.bounds, self.mx), v, dtype)
        r, c, v = transposed_block(rows, cols, vals, self.r0, self.r1)
        self.AT = ops.adjacency(nl, wide, r, padded_columns(c, self.bounds, self.mx), v, dtype)
        self._static = None

    # -- padded in-place all-gather ------------------------------------------
    def _buffer(self, f, dtype):
        buf = self.ops.empty(self.world * self.mx, f, dtype)
        lo = self.rank * self.mx
        return buf, buf[lo: lo + (self.r1 - self.r0)]

    def _exchange(self, buf):
        if self.world > 1:
            lo = self.rank * self.mx
            dist.all_gather_into_tensor(buf, buf[lo: lo + self.mx], group=self.group)
        return buf

    def gather(self, local):
        """Every rank's row block of `local`, padded layout."""
        buf, mine = self._buffer(local.shape[1], local.dtype)
        mine.copy_(local)
        return self._exchange(buf)

    def gather_static(self, X_local):
        """Layer-1 input features are the same every step: gather them once
        ('free for layer 1, replicate once')."""
        self._static = self.gather(X_local)
        return self._static

    def _allreduce(self, *ts):
        if self.world == 1:
            return ts
        flat = torch.cat([t.reshape(-1) for t in ts])
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=self.group)
        out, o = [], 0
        for t in ts:
            out.append(flat[o: o + t.numel()].view_as(t))
            o += t.numel()
        return tuple(out)

    def forward(self, X_local, theta, bias, scheme, static_input=False):
        fwd = scheme[0]
        ops = self.ops
        cache = {"scheme": scheme}
        if fwd == 0:  # transform-first: M = X Theta into my slot, gather, out = A'_p M + b
            buf, mine = self._buffer(theta.shape[1], X_local.dtype)
            ops.gemm(X_local, theta, out=mine)
            out = ops.spmm(self.A, self._exchange(buf), bias)
            cache["X"] = X_local
        else:  # propagate-first: gather X, P_p = A'_p X, out = P_p Theta + b
            if static_input:
                X = self._static if self._static is not None else self.gather_static(X_local)
            else:
                X = self.gather(X_local)
            P = ops.spmm(self.A, X)
            out = ops.gemm(P, theta, bias=bias)
            if fwd == 2:
                cache["P"] = P
            else:
                cache["X"] = X_local
                cache["Xg"] = X if static_input else None
        return out, cache

    def backward(self, G_local, theta, cache, needs_feature_grad):
        ops = self.ops
        bwd = cache["scheme"][1]
        d_input = None
        if bwd == 0:  # fused: S = A'^T G (rows of my block), dTheta = X^T S
            d_bias = ops.colsum(G_local)
            S = ops.spmm(self.AT, self.gather(G_local))
            d_theta, d_bias = self._allreduce(ops.gemm(cache["X"], S, ta=True), d_bias)
            if needs_feature_grad:
                d_input = ops.gemm(S, theta, tb=True)
        else:
            if bwd == 1:  # split: recompute P_p = A'_p X
                X = cache.get("Xg")
                P = ops.spmm(self.A, X if X is not None else self.gather(cache["X"]))
            else:
                P = cache["P"]
            d_bias = ops.empty(1, G_local.shape[1], G_local.dtype).view(-1)
            d_theta = ops.gemm(P, G_local, ta=True, colsum_b=d_bias)
            d_theta, d_bias = self._allreduce(d_theta, d_bias)
            if needs_feature_grad:
                buf, mine = self._buffer(theta.shape[0], G_local.dtype)
                ops.gemm(G_local, theta, tb=True, out=mine)
                d_input = ops.spmm(self.AT, self._exchange(buf))
        return d_theta, d_bias, d_input

    def step_host(self, hX, theta, bias, scheme, hG, needs_feature_grad, h_out, h_d_theta,
                  h_d_bias, h_d_input=None, static_input=False):
        """Forward + backward of this rank's row block from HOST buffers
        (pinned), the counterpart of sgnn_gcn_step_host: X / dX' blocks are
        copied in and out / grads copied out on side streams, overlapped with
        compute and with each other.  Stream-ordered on the current stream."""
        cs = torch.cuda.current_stream()
        if not hasattr(self, "_s_in"):
            self._s_in, self._s_out = torch.cuda.Stream(), torch.cuda.Stream()
        s_in, s_out = self._s_in, self._s_out
        s_in.wait_stream(cs)
        s_out.wait_stream(cs)
        dev = cs.device
        with torch.cuda.stream(s_in):
            X = hX.to(dev, non_blocking=True)
            ev_x = torch.cuda.Event()
            ev_x.record(s_in)
            G = hG.to(dev, non_blocking=True)
            ev_g = torch.cuda.Event()
            ev_g.record(s_in)
        X.record_stream(cs)
        G.record_stream(cs)
        cs.wait_event(ev_x)
        out, cache = self.forward(X, theta, bias, scheme, static_input=static_input)
        ev_o = torch.cuda.Event()
        ev_o.record(cs)
        s_out.wait_event(ev_o)
        with torch.cuda.stream(s_out):
            h_out.copy_(out, non_blocking=True)
        out.record_stream(s_out)
        cs.wait_event(ev_g)
        d_theta, d_bias, d_input = self.backward(G, theta, cache, needs_feature_grad)
        ev_b = torch.cuda.Event()
        ev_b.record(cs)
        s_out.wait_event(ev_b)
        with torch.cuda.stream(s_out):
            h_d_theta.copy_(d_theta, non_blocking=True)
            h_d_bias.copy_(d_bias, non_blocking=True)
            if needs_feature_grad:
                h_d_input.copy_(d_input, non_blocking=True)
        for t in (d_theta, d_bias) + ((d_input,) if needs_feature_grad else ()):
            t.record_stream(s_out)
        cs.wait_stream(s_out)


class DistGcn2:
    """Gcn2Model (model.hpp:40-115: GCN -> ReLU -> GCN, MSE step) over the
    row partition: both layers share the rank's operator blocks; the hidden
    activation, the loss and its gradient are computed on the rank's rows
    (the loss sum is all-reduced, the gradient normalised by the global
    size); parameter gradients are all-reduced inside the layers.  Parameters
    are replicated, initialised like the reference (seed, seed + 101)."""

    def __init__(self, layer: DistGcnLayer, m, hidden, out, seed, policy="adaptive",
                 caching=True, input_grad=False, dtype=torch.float32):
        from . import device as d

        self.d, self.layer = d, layer
        self.p = list(d.gcn_params(m, hidden, seed, dtype=dtype)) + \
            list(d.gcn_params(hidden, out, seed + 101, dtype=dtype))
        s1 = d.resolve_scheme(policy, m, hidden, input_grad, caching)
        s2 = d.resolve_scheme(policy, hidden, out, True, caching)  # model.hpp:61-62
        self.s1 = (s1.forward, s1.backward, s1.caching)
        self.s2 = (s2.forward, s2.backward, s2.caching)
        self.input_grad, self.out = input_grad, out

    def train_step(self, X_local, target_local, static_input=True):
        d, L = self.d, self.layer
        th1, b1, th2, b2 = self.p
        h, c1 = L.forward(X_local, th1, b1, self.s1, static_input=static_input)
        h, mask = d.activation(h, "relu", out=h)
        o, c2 = L.forward(h, th2, b2, self.s2)
        loss, g = d.loss_mse(o, target_local, total=L.n * self.out)
        if L.world > 1:
            dist.all_reduce(loss, op=dist.ReduceOp.SUM, group=L.group)
        dth2, db2, dh = L.backward(g, th2, c2, True)
        dh = d.activation_backward(dh, mask, "relu", out=dh)
        dth1, db1, dx = L.backward(dh, th1, c1, self.input_grad)
        return loss, o, [dth1, db1, dth2, db2], dx


# ---------------------------------------------------------------------------
# partitioned GAT layer (gat.hpp:89-219 over row blocks)
# ---------------------------------------------------------------------------
def gat_blocks(rowptr, cols, bounds, rank):
    """Host-side index arrays of rank's blocks of a GAT pattern (CSR with all
    self loops, canonical order).  Row block: local rowptr and the columns
    remapped to the padded node layout.  Column block (columns [r0, r1), i.e.
    rows of A^T, rows ascending within a column like the reference's CSC,
    sparse.hpp:207-216): local colptr, the rows remapped to the padded node
    layout, and perm = the padded edge index of each entry -- the edges of
    rank p's rows occupy slot p (emx entries) of a gathered edge-major array."""
    rowptr = np.asarray(rowptr, np.int64)
    cols = np.asarray(cols, np.int64)
    world = len(bounds) - 1
    mx = max(bounds[p + 1] - bounds[p] for p in range(world))
    ebounds = [int(rowptr[b]) for b in bounds]
    emx = max(ebounds[p + 1] - ebounds[p] for p in range(world))
    r0, r1 = bounds[rank], bounds[rank + 1]
    e0, e1 = ebounds[rank], ebounds[rank + 1]
    rp = (rowptr[r0:r1 + 1] - e0).astype(np.int32)
    cl = padded_columns(cols[e0:e1], bounds, mx)
    n = len(rowptr) - 1
    rows_of = np.repeat(np.arange(n, dtype=np.int64), np.diff(rowptr))
    sel = np.nonzero((cols >= r0) & (cols < r1))[0]  # canonical edge ids, row-major
    lc = cols[sel] - r0
    order = np.argsort(lc, kind="stable")  # rows stay ascending within a column
    e = sel[order]
    r = rows_of[e]
    colptr = np.zeros(r1 - r0 + 1, np.int64)
    np.add.at(colptr, lc[order] + 1, 1)
    colptr = np.cumsum(colptr).astype(np.int32)
    owner = np.searchsorted(np.asarray(bounds, np.int64), r, side="right") - 1
    perm = (owner * emx + (e - np.asarray(ebounds, np.int64)[owner])).astype(np.int32)
    return {"rowptr": rp, "cols": cl, "colptr": colptr,
            "rows": padded_columns(r, bounds, mx), "perm": perm, "mx": mx, "emx": emx,
            "edges": e1 - e0}


class DistGatLayer:
    """One GAT layer (float32, h in {1,2,4,8}, k % 4 == 0) over the row
    partition.  Forward: M = X_p Theta with the node scores (own rows) into
    the rank's slots of the padded M / d gather buffers, all-gather, then
    attention and aggregation of the rank's rows.  Backward: SDDMM and the
    softmax backward on the rank's rows, all-gather of dX', alpha and dy
    (edge-major; each rank's edges are one contiguous slot), the column pass
    over the rank's columns (rows of A^T), parameter gradients on the rank's
    rows, one packed all-reduce.  Every piece is a libsgnn_cuda.so kernel
    (the sgnn_gat_* block entry points)."""

    def __init__(self, n, rowptr, cols, heads, k, device, group=None):
        from . import _capi
        from .device import Context

        self.c = _capi
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.n, self.h, self.k = n, heads, k
        self.dev = torch.device(device)
        self.bounds = partition_rows(rowptr, self.world)
        self.r0, self.r1 = self.bounds[self.rank], self.bounds[self.rank + 1]
        b = gat_blocks(rowptr, cols, self.bounds, self.rank)
        self.mx, self.emx, self.ne = b["mx"], b["emx"], b["edges"]
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(self.dev)  # noqa: E731
        self.rowptr, self.cols = t(b["rowptr"]), t(b["cols"])
        self.colptr, self.crows, self.perm = t(b["colptr"]), t(b["rows"]), t(b["perm"])
        self.ctx = Context.default(self.dev.index)
        # hub-row plans of the rank's row and column blocks (power-law graphs)
        nl = self.r1 - self.r0
        self.rplan, self.cplan = C.c_void_p(), C.c_void_p()
        _capi.check(_capi.lib.sgnn_rowplan_create(self.ctx.handle, nl, self.rowptr.data_ptr(),
                                                  C.byref(self.rplan)))
        _capi.check(_capi.lib.sgnn_rowplan_create(self.ctx.handle, nl, self.colptr.data_ptr(),
                                                  C.byref(self.cplan)))

    def __del__(self):
        lib = self.c.lib if hasattr(self, "c") else None
        for nm in ("rplan", "cplan"):
            h = getattr(self, nm, None)
            if lib is not None and h:
                lib.sgnn_rowplan_destroy(h)

    def _buf(self, slots, width, used, dtype=torch.float32):
        buf = torch.empty((self.world * slots, width), dtype=dtype, device=self.dev)
        lo = self.rank * slots
        return buf, buf[lo: lo + used]

    def _exchange(self, buf, slots):
        if self.world > 1:
            lo = self.rank * slots
            dist.all_gather_into_tensor(buf, buf[lo: lo + slots], group=self.group)
        return buf

    @staticmethod
    def _p(t):
        return None if t is None else t.data_ptr()

    def forward(self, X_local, theta, a_src, a_dst, bias, beta=0.2):
        c, lib, P = self.c, self.c.lib, self._p
        h, k, nl = self.h, self.k, self.r1 - self.r0
        X_local = X_local.contiguous()
        Mbuf, Mmine = self._buf(self.mx, h * k, nl)
        dbuf, dmine = self._buf(self.mx, h, nl)
        s_loc = torch.empty((nl, h), dtype=torch.float32, device=self.dev)
        c.check(lib.sgnn_gat_transform(self.ctx.handle, P(X_local), nl, X_local.shape[1],
                                       P(theta), h, k, P(a_src), P(a_dst), P(Mmine), P(s_loc),
                                       P(dmine)))
        self._exchange(Mbuf, self.mx)
        self._exchange(dbuf, self.mx)
        abuf, amine = self._buf(self.emx, h, self.ne)
        mask = torch.empty((self.ne, h), dtype=torch.uint8, device=self.dev)
        c.check(lib.sgnn_gat_attention(self.ctx.handle, nl, P(self.rowptr), P(self.cols), h,
                                       P(s_loc), P(dbuf), float(beta), P(amine), P(mask),
                                       self.rplan))
        out = torch.empty((nl, h * k), dtype=torch.float32, device=self.dev)
        c.check(lib.sgnn_gat_aggregate(self.ctx.handle, nl, P(self.rowptr), P(self.cols), h, k,
                                       P(amine), P(Mbuf), P(bias), P(out), self.rplan))
        return out, {"X": X_local, "M": Mbuf, "Mmine": Mmine, "alpha": abuf, "amine": amine,
                     "mask": mask, "beta": beta}

    def backward(self, G_local, theta, a_src, a_dst, cache, needs_feature_grad):
        from . import device as d

        c, lib, P = self.c, self.c.lib, self._p
        h, k, nl = self.h, self.k, self.r1 - self.r0
        hk = h * k
        beta = cache["beta"]
        Gbuf, Gmine = self._buf(self.mx, hk, nl)
        Gmine.copy_(G_local)
        da = torch.empty((self.ne, h), dtype=torch.float32, device=self.dev)
        c.check(lib.sgnn_gat_sddmm(self.ctx.handle, nl, P(self.rowptr), P(self.cols), h, k,
                                   P(cache["M"]), P(Gmine), P(da), self.rplan))
        dybuf, dymine = self._buf(self.emx, h, self.ne)
        dS = torch.empty((nl, h), dtype=torch.float32, device=self.dev)
        c.check(lib.sgnn_gat_softmax_backward(self.ctx.handle, nl, P(self.rowptr), h,
                                              P(cache["amine"]), P(cache["mask"]), P(da),
                                              float(beta), P(dymine), P(dS), self.rplan))
        self._exchange(Gbuf, self.mx)
        self._exchange(cache["alpha"], self.emx)
        self._exchange(dybuf, self.emx)
        dD = torch.empty((nl, h), dtype=torch.float32, device=self.dev)
        dM = torch.empty((nl, hk), dtype=torch.float32, device=self.dev)
        c.check(lib.sgnn_gat_column_pass(self.ctx.handle, nl, P(self.colptr), P(self.crows),
                                         P(self.perm), h, k, P(Gbuf), P(cache["alpha"]),
                                         P(dybuf), P(dS), P(a_src), P(a_dst), P(dD), P(dM),
                                         self.cplan))
        flat = torch.empty(theta.numel() + 3 * hk, dtype=torch.float32, device=self.dev)
        d_theta = flat[:theta.numel()].view_as(theta)
        d_b = flat[theta.numel():theta.numel() + hk]
        d_as = flat[theta.numel() + hk:theta.numel() + 2 * hk].view(h, k)
        d_ad = flat[theta.numel() + 2 * hk:].view(h, k)
        c.check(lib.sgnn_gat_param_grads(self.ctx.handle, nl, h, k, P(Gmine),
                                         P(cache["Mmine"]), P(dS), P(dD), P(d_b), P(d_as),
                                         P(d_ad)))
        d.gemm(cache["X"], dM, True, False, out=d_theta)
        d_x = d.gemm(dM, theta, False, True) if needs_feature_grad else None
        if self.world > 1:
            dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=self.group)
        return d_theta, d_as, d_ad, d_b, d_x
