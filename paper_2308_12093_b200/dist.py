"""1-D destination-row partitioned GCN / GAT layers and 2-layer models across
the ranks of a torch.distributed group (NCCL over NVLink on B200; gloo in the
CPU tests).

North-star row (e) / SURVEY 8(e): destination rows are split into P contiguous
blocks balanced by nnz.  Rank p owns
  * A'_p   -- rows [r0, r1) of A' (all columns), CSR, for A' . B
  * A'T_p  -- rows [r0, r1) of A'^T (= columns [r0, r1) of A'), for A'^T . B
  * its row block of X / dX' / out, and replicated parameters.
Every propagation of a dense operand B needs all rows of B: one all-gather per
SpMM (the exchange step); parameter gradients are all-reduced.  Accumulation
order inside each output row is the reference's (ascending column), so the
SpMM blocks are bit-identical to the single-GPU product.

The GAT layer exchanges node-sized data only: M and the destination scores d
in the forward pass; dX' and four per-row statistics (s, softmax max, 1 / sum,
sum alpha dAlpha) in the backward pass, from which the column pass rebuilds
every edge's alpha and dy (sgnn_gat_column_pass_stats).  Shipping alpha and
dy instead costs 2 q' h values per layer -- 4.1 GB at config 5 -- against
4 n h (0.31 GB).

All-gathers are issued asynchronously and overlap the compute that does not
need them (the GAT attention with the M gather, the SDDMM and softmax backward
with the dX' gather, the dTheta GEMM with the G.Theta^T gather).

The compute backend is pluggable (`ops`): DeviceOps / GatDeviceOps run
libsgnn_cuda.so on the rank's GPU; tests inject CPU implementations to
exercise the partition and collective logic under gloo.
"""
from __future__ import annotations

import contextlib
import ctypes as C

import numpy as np
import torch
import torch.distributed as dist


# ---------------------------------------------------------------------------
# host-side partition logic (numpy or torch inputs; torch tensors stay on
# their device, so a 64M-edge graph is partitioned on the GPU)
# ---------------------------------------------------------------------------
def _np(a):
    return a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)


def _t(a, dtype=None):
    t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
    return t if dtype is None else t.to(dtype)


def partition_rows(rowptr, parts):
    """nnz-balanced contiguous row blocks: bounds[p] .. bounds[p+1]."""
    rowptr = _np(rowptr).astype(np.int64)
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
    if isinstance(rows, torch.Tensor):
        lo = int(torch.searchsorted(rows, torch.tensor(r0, dtype=rows.dtype, device=rows.device)))
        hi = int(torch.searchsorted(rows, torch.tensor(r1, dtype=rows.dtype, device=rows.device)))
        return (rows[lo:hi] - r0).to(torch.int32), cols[lo:hi].to(torch.int32), vals[lo:hi]
    rows = np.asarray(rows)
    lo = int(np.searchsorted(rows, r0, side="left"))
    hi = int(np.searchsorted(rows, r1, side="left"))
    return (rows[lo:hi] - r0).astype(np.int32), np.asarray(cols)[lo:hi].astype(np.int32), \
        np.asarray(vals)[lo:hi]


def transposed_block(rows, cols, vals, r0, r1):
    """Rows [r0, r1) of A^T = entries with col in [r0, r1), as canonical COO
    (local row = col - r0, global col = row), ordered by (col, row): the CSC
    order of the reference (rows ascend within a column, sparse.hpp:207-216)."""
    if isinstance(rows, torch.Tensor):
        m = (cols >= r0) & (cols < r1)
        r, c, v = (cols[m] - r0).to(torch.int64), rows[m].to(torch.int64), vals[m]
        # canonical COO is row-major, so c ascends already: a stable sort by r
        order = torch.argsort(r, stable=True)
        return r[order].to(torch.int32), c[order].to(torch.int32), v[order]
    rows, cols, vals = np.asarray(rows), np.asarray(cols), np.asarray(vals)
    m = (cols >= r0) & (cols < r1)
    r, c, v = cols[m] - r0, rows[m], vals[m]
    order = np.lexsort((c, r))
    return r[order].astype(np.int32), c[order].astype(np.int32), v[order]


def padded_columns(cols, bounds, mx):
    """Global column j -> owner(j) * mx + (j - bounds[owner]): the row of j in
    the padded all-gather layout (world blocks of mx rows).  Monotonic in j,
    so the stored (ascending-column) order of every row is unchanged."""
    if isinstance(cols, torch.Tensor):
        b = torch.tensor(bounds, dtype=torch.int64, device=cols.device)
        c = cols.to(torch.int64).contiguous()
        owner = torch.searchsorted(b, c, right=True) - 1
        return (owner * mx + (c - b[owner])).to(torch.int32)
    cols = np.asarray(cols, np.int64)
    b = np.asarray(bounds, np.int64)
    owner = np.searchsorted(b, cols, side="right") - 1
    return (owner * mx + (cols - b[owner])).astype(np.int32)


# ---------------------------------------------------------------------------
# stream discipline and asynchronous exchanges
# ---------------------------------------------------------------------------
@contextlib.contextmanager
def ordered_on(stream):
    """Run the body with `stream` as torch's current stream, ordered after the
    caller's current stream and before whatever the caller enqueues next:
    libsgnn_cuda.so kernels (the context's stream), torch allocations and
    NCCL collectives (which follow torch's current stream) then share one
    stream whatever stream the caller is on."""
    if stream is None:
        yield
        return
    cur = torch.cuda.current_stream(stream.device)
    if cur == stream:
        yield
        return
    stream.wait_stream(cur)
    with torch.cuda.stream(stream):
        yield
    cur.wait_stream(stream)


class _Exchange:
    """Padded in-place all-gather of rank slots, issued asynchronously."""

    def __init__(self, group, rank, world):
        self.group, self.rank, self.world = group, rank, world

    def start(self, buf, slots):
        if self.world == 1:
            return None
        lo = self.rank * slots
        return dist.all_gather_into_tensor(buf, buf[lo: lo + slots], group=self.group,
                                           async_op=True)

    @staticmethod
    def wait(work):
        if work is not None:
            work.wait()

    def allreduce(self, flat):
        if self.world > 1:
            dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=self.group)
        return flat


def _rank_world(group):
    """(rank, world) of a process group; a group object may instead carry its
    own (`rank_world()`: the single-GPU multi-rank simulation of the tests)."""
    if hasattr(group, "rank_world"):
        return group.rank_world()
    return dist.get_rank(group), dist.get_world_size(group)


def _exchange_for(group, rank, world):
    if hasattr(group, "exchange"):  # simulated group: its own collectives
        return group.exchange(rank, world)
    return _Exchange(group, rank, world)


# ---------------------------------------------------------------------------
# compute backends
# ---------------------------------------------------------------------------
class DeviceOps:
    """libsgnn_cuda.so on this rank's GPU (fails loudly without it)."""

    def __init__(self, device):
        from . import device as d

        self.d = d
        self.dev = torch.device(device)
        self.ctx = d.Context.default(self.dev.index)

    def scope(self):
        return ordered_on(self.ctx.stream)

    def adjacency(self, n_rows, n_cols, rows, cols, vals, dtype):
        d = self.d
        t = lambda a, dt: _t(a).to(self.dev, dt)  # noqa: E731
        return d.Adjacency(n_rows, n_cols, t(rows, torch.int32), t(cols, torch.int32),
                           t(vals, dtype), "csr", ctx=self.ctx)

    def empty(self, rows, cols, dtype):
        return torch.empty((rows, cols), dtype=dtype, device=self.dev)

    def spmm(self, adj, B, bias=None):
        return adj.spmm(B.contiguous(), bias=bias)

    def gemm(self, A, B, ta=False, tb=False, bias=None, out=None, colsum_b=None):
        """bias fused into the epilogue; colsum_b = 1^T B from the same read
        of B (C = A^T B); out may be a row range of a larger buffer."""
        return self.d.gemm(A, B, ta, tb, ctx=self.ctx, bias=bias, out=out, colsum_b=colsum_b)

    def colsum(self, X):
        return self.d.column_sums(X, ctx=self.ctx)

    def gemm_act(self, A, B, act, mask, ta=False, tb=False, bias=None, saved=None):
        """gemm + activation, fused into the tcgen05 epilogue where possible"""
        return self.d.gemm_act(A, B, act, mask, ta, tb, bias=bias, saved=saved, ctx=self.ctx)

    def mask(self, rows, cols):
        return torch.empty((rows, cols), dtype=torch.uint8, device=self.dev)

    # model pieces (dense.hpp:196-270, model.hpp loss_mse)
    def activation(self, X, kind, out=None):
        return self.d.activation(X, kind, out=out, ctx=self.ctx)

    def activation_backward(self, g, mask, kind, saved=None, out=None):
        return self.d.activation_backward(g, mask, kind, saved=saved, out=out, ctx=self.ctx)

    def loss_mse(self, out, target, total):
        return self.d.loss_mse(out, target, total=total, ctx=self.ctx)


class GatDeviceOps(DeviceOps):
    """The GAT block entry points of libsgnn_cuda.so (sgnn_gat_*; float32,
    h in {1,2,4,8}, k % 4 == 0)."""

    def __init__(self, device):
        super().__init__(device)
        from . import _capi

        self.c = _capi

    def index(self, a):
        return _t(a, torch.int32).to(self.dev).contiguous()

    def rowplan(self, n_rows, rowptr):
        h = C.c_void_p()
        self.c.check(self.c.lib.sgnn_rowplan_create(self.ctx.handle, n_rows, rowptr.data_ptr(),
                                                    C.byref(h)))
        return h

    def free_rowplan(self, h):
        if h:
            self.c.lib.sgnn_rowplan_destroy(h)

    def stats_supported(self, h, k):
        return bool(self.c.lib.sgnn_gat_column_stats_supported(h, k))

    @staticmethod
    def _p(t):
        return None if t is None else t.data_ptr()

    def transform(self, X, theta, h, k, a_src, a_dst, M, s, d):
        P = self._p
        self.c.check(self.c.lib.sgnn_gat_transform(self.ctx.handle, P(X), X.shape[0], X.shape[1],
                                                   P(theta), h, k, P(a_src), P(a_dst), P(M),
                                                   P(s), P(d)))

    def attention(self, nl, rowptr, cols, h, s, d, beta, alpha, mask, stats, plan):
        P = self._p
        self.c.check(self.c.lib.sgnn_gat_attention_ex(self.ctx.handle, nl, P(rowptr), P(cols), h,
                                                      P(s), P(d), float(beta), P(alpha), P(mask),
                                                      P(stats), plan))

    def aggregate(self, nl, rowptr, cols, h, k, alpha, M, bias, out, plan):
        P = self._p
        self.c.check(self.c.lib.sgnn_gat_aggregate(self.ctx.handle, nl, P(rowptr), P(cols), h, k,
                                                   P(alpha), P(M), P(bias), P(out), plan))

    def sddmm(self, nl, rowptr, cols, h, k, M, G, da, plan):
        P = self._p
        self.c.check(self.c.lib.sgnn_gat_sddmm(self.ctx.handle, nl, P(rowptr), P(cols), h, k,
                                               P(M), P(G), P(da), plan))

    def softmax_backward(self, nl, rowptr, h, alpha, mask, da, beta, dy, dS, stats, plan):
        P = self._p
        self.c.check(self.c.lib.sgnn_gat_softmax_backward_ex(
            self.ctx.handle, nl, P(rowptr), h, P(alpha), P(mask), P(da), float(beta), P(dy),
            P(dS), P(stats), plan))

    def column_pass(self, nl, colptr, rows, perm, h, k, G, alpha, dy, dS, a_src, a_dst, dD,
                    dM, plan):
        P = self._p
        self.c.check(self.c.lib.sgnn_gat_column_pass(
            self.ctx.handle, nl, P(colptr), P(rows), P(perm), h, k, P(G), P(alpha), P(dy),
            P(dS), P(a_src), P(a_dst), P(dD), P(dM), plan))

    def column_pass_stats(self, nl, colptr, rows, h, k, G, stats, d_own, M_own, beta, dS,
                          a_src, a_dst, dD, dM, plan):
        P = self._p
        self.c.check(self.c.lib.sgnn_gat_column_pass_stats(
            self.ctx.handle, nl, P(colptr), P(rows), h, k, P(G), P(stats), P(d_own), P(M_own),
            float(beta), P(dS), P(a_src), P(a_dst), P(dD), P(dM), plan))

    def param_grads(self, nl, h, k, G, M, dS, dD, d_b, d_as, d_ad):
        P = self._p
        self.c.check(self.c.lib.sgnn_gat_param_grads(self.ctx.handle, nl, h, k, P(G), P(M),
                                                     P(dS), P(dD), P(d_b), P(d_as), P(d_ad)))


def _scope(ops):
    return ops.scope() if hasattr(ops, "scope") else contextlib.nullcontext()


# ---------------------------------------------------------------------------
# partitioned GCN layer (gcn.hpp:91-193 over row blocks)
# ---------------------------------------------------------------------------
class DistGcnLayer:
    """One GCN layer over a row-partitioned normalized operator.

    rows/cols/vals: the full canonical normalized COO of A' (host arrays or
    device tensors; every rank builds only its blocks).  scheme: (forward,
    backward, caching) ints of the reference's SchemeChoice (resolve with
    device.resolve_scheme).

    Gathered operands use a padded layout -- world blocks of mx = max block
    rows -- and the local operator blocks index it directly (their column ids
    are remapped once at setup), so a rank's producer (GEMM) writes its rows
    straight into its slot of the gather buffer and the all-gather is
    in place: no pad or concatenation copies, and none at all at world 1.
    """

    def __init__(self, n, rows, cols, vals, ops, dtype=torch.float32, group=None):
        self.group = group
        self.rank, self.world = _rank_world(group)
        r_np = _np(rows).astype(np.int64) if not isinstance(rows, torch.Tensor) else None
        if r_np is not None:
            rowptr = np.zeros(n + 1, np.int64)
            np.add.at(rowptr, r_np + 1, 1)
            rowptr = np.cumsum(rowptr)
        else:
            rowptr = torch.zeros(n + 1, dtype=torch.int64, device=rows.device)
            rowptr[1:] = torch.cumsum(torch.bincount(rows.to(torch.int64), minlength=n), 0)
        self.n = n
        self.nnz = int(rowptr[-1])
        self.bounds = partition_rows(rowptr, self.world)
        self.r0, self.r1 = self.bounds[self.rank], self.bounds[self.rank + 1]
        self.mx = max(self.bounds[p + 1] - self.bounds[p] for p in range(self.world))
        self.ops, self.dtype = ops, dtype
        self.x = _exchange_for(group, self.rank, self.world)
        nl = self.r1 - self.r0
        wide = self.world * self.mx
        r, c, v = row_block(rows, cols, vals, self.r0, self.r1)
        self.local_nnz = int(r.shape[0])
        self.A = ops.adjacency(nl, wide, r, padded_columns(c, self.bounds, self.mx), v, dtype)
        r, c, v = transposed_block(rows, cols, vals, self.r0, self.r1)
        self.AT = ops.adjacency(nl, wide, r, padded_columns(c, self.bounds, self.mx), v, dtype)
        self._static = None
        self._static_key = None

    # -- padded in-place all-gather ------------------------------------------
    def _buffer(self, f, dtype):
        buf = self.ops.empty(self.world * self.mx, f, dtype)
        lo = self.rank * self.mx
        return buf, buf[lo: lo + (self.r1 - self.r0)]

    def _exchange(self, buf):
        self.x.wait(self.x.start(buf, self.mx))
        return buf

    def gather(self, local):
        """Every rank's row block of `local`, padded layout."""
        buf, mine = self._buffer(local.shape[1], local.dtype)
        mine.copy_(local)
        return self._exchange(buf)

    @staticmethod
    def _key(X):
        return (X.data_ptr(), X._version, tuple(X.shape), X.dtype)

    def gather_static(self, X_local):
        """Layer-1 input features are the same every step: gather them once
        ('free for layer 1, replicate once').  The cached copy is
        keyed on the tensor's storage and version, so new or modified
        features are gathered again."""
        key = self._key(X_local)
        if self._static is None or self._static_key != key:
            self._static = self.gather(X_local)
            self._static_key = key
        return self._static

    def _allreduce(self, *ts):
        if self.world == 1:
            return ts
        flat = torch.cat([t.reshape(-1) for t in ts])
        self.x.allreduce(flat)
        out, o = [], 0
        for t in ts:
            out.append(flat[o: o + t.numel()].view_as(t))
            o += t.numel()
        return tuple(out)

    def forward(self, X_local, theta, bias, scheme, static_input=False):
        with _scope(self.ops):
            return self._forward(X_local, theta, bias, scheme, static_input)

    def _forward(self, X_local, theta, bias, scheme, static_input, relu_mask=None):
        """relu_mask (optional, uint8 like out): out = ReLU(layer) with its
        mask (dense.hpp:197-228), fused into the output GEMM's epilogue for
        the propagate-first schemes."""
        fwd = scheme[0]
        ops = self.ops
        cache = {"scheme": scheme}
        if fwd == 0:  # transform-first: M = X Theta into my slot, gather, out = A'_p M + b
            buf, mine = self._buffer(theta.shape[1], X_local.dtype)
            ops.gemm(X_local, theta, out=mine)
            out = ops.spmm(self.A, self._exchange(buf), bias)
            if relu_mask is not None:
                out, m = ops.activation(out, "relu", out=out)
                relu_mask.copy_(m)
            cache["X"] = X_local
        else:  # propagate-first: gather X, P_p = A'_p X, out = P_p Theta + b
            X = self.gather_static(X_local) if static_input else self.gather(X_local)
            P = ops.spmm(self.A, X)
            if relu_mask is not None:
                out = ops.gemm_act(P, theta, "relu", relu_mask, bias=bias)
            else:
                out = ops.gemm(P, theta, bias=bias)
            if fwd == 2:
                cache["P"] = P
            else:
                cache["X"] = X_local
                cache["Xg"] = X if static_input else None
        return out, cache

    def backward(self, G_local, theta, cache, needs_feature_grad):
        with _scope(self.ops):
            return self._backward(G_local, theta, cache, needs_feature_grad)

    def _backward(self, G_local, theta, cache, needs_feature_grad, relu_mask=None):
        """relu_mask (optional): d_input gets the ReLU backward of the layer
        below applied (fused into the d_input GEMM for the fused scheme)."""
        ops = self.ops
        bwd = cache["scheme"][1]
        d_input = None
        if bwd == 0:  # fused: S = A'^T G (rows of my block), dTheta = X^T S
            buf, mine = self._buffer(G_local.shape[1], G_local.dtype)
            mine.copy_(G_local)
            w = self.x.start(buf, self.mx)
            d_bias = ops.colsum(G_local)  # overlaps the exchange
            self.x.wait(w)
            S = ops.spmm(self.AT, buf)
            d_theta, d_bias = self._allreduce(ops.gemm(cache["X"], S, ta=True), d_bias)
            if needs_feature_grad:
                if relu_mask is not None:
                    return d_theta, d_bias, ops.gemm_act(S, theta, "relu_backward", relu_mask,
                                                         tb=True)
                d_input = ops.gemm(S, theta, tb=True)
        else:
            w, buf = None, None
            if needs_feature_grad:  # G Theta^T into my slot first: its exchange
                buf, mine = self._buffer(theta.shape[0], G_local.dtype)  # overlaps dTheta
                ops.gemm(G_local, theta, tb=True, out=mine)
                w = self.x.start(buf, self.mx)
            if bwd == 1:  # split: recompute P_p = A'_p X
                X = cache.get("Xg")
                P = ops.spmm(self.A, X if X is not None else self.gather(cache["X"]))
            else:
                P = cache["P"]
            d_bias = ops.empty(1, G_local.shape[1], G_local.dtype).view(-1)
            d_theta = ops.gemm(P, G_local, ta=True, colsum_b=d_bias)
            self.x.wait(w)
            d_theta, d_bias = self._allreduce(d_theta, d_bias)
            if needs_feature_grad:
                d_input = ops.spmm(self.AT, buf)
        if relu_mask is not None and d_input is not None:
            d_input = ops.activation_backward(d_input, relu_mask, "relu", out=d_input)
        return d_theta, d_bias, d_input

    def step_host(self, hX, theta, bias, scheme, hG, needs_feature_grad, h_out, h_d_theta,
                  h_d_bias, h_d_input=None, static_input=False):
        """Forward + backward of this rank's row block from HOST buffers
        (pinned), the counterpart of sgnn_gcn_step_host: X / dX' blocks are
        copied in and out / grads copied out on side streams, overlapped with
        compute and with each other.  Ordered after the caller's current
        stream; the compute runs on the context's stream."""
        with _scope(self.ops):
            self._step_host(hX, theta, bias, scheme, hG, needs_feature_grad, h_out, h_d_theta,
                            h_d_bias, h_d_input, static_input)

    def _step_host(self, hX, theta, bias, scheme, hG, needs_feature_grad, h_out, h_d_theta,
                   h_d_bias, h_d_input, static_input):
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
        out, cache = self._forward(X, theta, bias, scheme, static_input)
        ev_o = torch.cuda.Event()
        ev_o.record(cs)
        s_out.wait_event(ev_o)
        with torch.cuda.stream(s_out):
            h_out.copy_(out, non_blocking=True)
        out.record_stream(s_out)
        cs.wait_event(ev_g)
        d_theta, d_bias, d_input = self._backward(G, theta, cache, needs_feature_grad)
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
                 caching=True, input_grad=False, dtype=torch.float32, params=None):
        from . import device as d

        self.layer = layer
        if params is None:
            params = list(d.gcn_params(m, hidden, seed, dtype=dtype)) + \
                list(d.gcn_params(hidden, out, seed + 101, dtype=dtype))
        self.p = list(params)
        s1 = d.resolve_scheme(policy, m, hidden, input_grad, caching)
        s2 = d.resolve_scheme(policy, hidden, out, True, caching)  # model.hpp:61-62
        self.s1 = (s1.forward, s1.backward, s1.caching)
        self.s2 = (s2.forward, s2.backward, s2.caching)
        self.input_grad, self.out = input_grad, out

    def train_step(self, X_local, target_local, static_input=True):
        L = self.layer
        with _scope(L.ops):
            ops = L.ops
            th1, b1, th2, b2 = self.p
            # ReLU fused into the layer-1 output GEMM and, backwards, into the
            # layer-2 d_input GEMM where the schemes allow it (as model.cu)
            mask = ops.mask(L.r1 - L.r0, th1.shape[1])
            h, c1 = L._forward(X_local, th1, b1, self.s1, static_input, relu_mask=mask)
            o, c2 = L._forward(h, th2, b2, self.s2, False)
            loss, g = ops.loss_mse(o, target_local, L.n * self.out)
            L.x.allreduce(loss)
            dth2, db2, dh = L._backward(g, th2, c2, True, relu_mask=mask)
            dth1, db1, dx = L._backward(dh, th1, c1, self.input_grad)
        return loss, o, [dth1, db1, dth2, db2], dx


# ---------------------------------------------------------------------------
# partitioned GAT layer (gat.hpp:89-219 over row blocks)
# ---------------------------------------------------------------------------
def gat_blocks(rowptr, cols, bounds, rank):
    """Index arrays of rank's blocks of a GAT pattern (CSR with all self
    loops, canonical order).  Row block: local rowptr and the columns
    remapped to the padded node layout.  Column block (columns [r0, r1), i.e.
    rows of A^T, rows ascending within a column like the reference's CSC,
    sparse.hpp:207-216): local colptr, the rows remapped to the padded node
    layout, and perm = the padded edge index of each entry -- the edges of
    rank p's rows occupy slot p (emx entries) of a gathered edge-major array.
    numpy inputs give numpy arrays; torch tensors stay on their device."""
    if not isinstance(rowptr, torch.Tensor):
        out = gat_blocks(torch.from_numpy(np.asarray(rowptr, np.int64)),
                         torch.from_numpy(np.asarray(cols, np.int64)), bounds, rank)
        return {k: (v.numpy() if isinstance(v, torch.Tensor) else v) for k, v in out.items()}
    rowptr = rowptr.to(torch.int64)
    cols = cols.to(torch.int64)
    dev = rowptr.device
    world = len(bounds) - 1
    mx = max(bounds[p + 1] - bounds[p] for p in range(world))
    rp_h = _np(rowptr[torch.tensor(bounds, device=dev)])
    ebounds = [int(x) for x in rp_h]
    emx = max(ebounds[p + 1] - ebounds[p] for p in range(world))
    r0, r1 = bounds[rank], bounds[rank + 1]
    e0, e1 = ebounds[rank], ebounds[rank + 1]
    rp = (rowptr[r0:r1 + 1] - e0).to(torch.int32)
    cl = padded_columns(cols[e0:e1], bounds, mx)
    n = rowptr.numel() - 1
    sel = torch.nonzero((cols >= r0) & (cols < r1)).view(-1)  # canonical edge ids, row-major
    lc = cols[sel] - r0
    order = torch.argsort(lc, stable=True)  # rows stay ascending within a column
    e = sel[order]
    # row of canonical edge e: the last rowptr entry <= e
    r = torch.searchsorted(rowptr, e, right=True) - 1
    colptr = torch.zeros(r1 - r0 + 1, dtype=torch.int64, device=dev)
    colptr[1:] = torch.cumsum(torch.bincount(lc, minlength=r1 - r0), 0)
    eb = torch.tensor(ebounds, dtype=torch.int64, device=dev)
    owner = torch.searchsorted(torch.tensor(bounds, dtype=torch.int64, device=dev), r,
                               right=True) - 1
    perm = (owner * emx + (e - eb[owner])).to(torch.int32)
    del n
    return {"rowptr": rp, "cols": cl, "colptr": colptr.to(torch.int32),
            "rows": padded_columns(r, bounds, mx), "perm": perm, "mx": mx, "emx": emx,
            "edges": e1 - e0}


class DistGatLayer:
    """One GAT layer (float32, h in {1,2,4,8}, k % 4 == 0) over the row
    partition.

    Forward: M = X_p Theta with the node scores (own rows) into the rank's
    slots of the padded M / d gather buffers; all-gather d, then the M
    all-gather overlapped with the attention of the rank's rows (which only
    needs d); aggregation.  Backward: the dX' all-gather overlapped with the
    SDDMM and softmax backward of the rank's rows; all-gather of the per-row
    statistics; the column pass over the rank's columns (rows of A^T)
    rebuilding alpha / dy from them; parameter gradients on the rank's rows;
    one packed all-reduce.

    exchange="stats" (default on more than one rank where
    sgnn_gat_column_stats_supported) ships 4 n h statistics; "edges" ships
    alpha and dy (2 q' h values) -- the default on one rank, where nothing is
    shipped and the single-GPU column pass (no dAlpha recompute) is 0.3 ms
    faster at Arxiv h=8 k=32 -- and for head widths the statistics kernel
    does not cover.

    `ops` is GatDeviceOps (or a device string); the CPU tests inject their
    own backend."""

    def __init__(self, n, rowptr, cols, heads, k, ops, group=None, exchange=None):
        if isinstance(ops, (str, torch.device)):
            ops = GatDeviceOps(ops)
        self.ops = ops
        self.group = group
        self.rank, self.world = _rank_world(group)
        self.x = _exchange_for(group, self.rank, self.world)
        self.n, self.h, self.k = n, heads, k
        self.bounds = partition_rows(rowptr, self.world)
        self.r0, self.r1 = self.bounds[self.rank], self.bounds[self.rank + 1]
        b = gat_blocks(rowptr, cols, self.bounds, self.rank)
        self.mx, self.emx, self.ne = b["mx"], b["emx"], b["edges"]
        self.nnz = int(_np(rowptr[-1:])[0])
        self.rowptr, self.cols = ops.index(b["rowptr"]), ops.index(b["cols"])
        self.colptr, self.crows, self.perm = (ops.index(b["colptr"]), ops.index(b["rows"]),
                                              ops.index(b["perm"]))
        if exchange is None:  # one rank exchanges nothing: keep the single-GPU column pass
            exchange = "stats" if self.world > 1 and ops.stats_supported(heads, k) else "edges"
        if exchange == "stats" and not ops.stats_supported(heads, k):
            raise ValueError(f"gat block: no statistics column pass for h={heads}, k={k}")
        self.exchange = exchange
        # hub-row plans of the rank's row and column blocks (power-law graphs)
        nl = self.r1 - self.r0
        self.rplan = ops.rowplan(nl, self.rowptr)
        self.cplan = ops.rowplan(nl, self.colptr)

    def __del__(self):
        ops = getattr(self, "ops", None)
        if ops is not None:
            for nm in ("rplan", "cplan"):
                h = getattr(self, nm, None)
                if h is not None:
                    ops.free_rowplan(h)

    def _buf(self, slots, width, used, dtype=torch.float32):
        buf = self.ops.empty(self.world * slots, width, dtype)
        lo = self.rank * slots
        return buf, buf[lo: lo + used]

    def forward(self, X_local, theta, a_src, a_dst, bias, beta=0.2):
        with _scope(self.ops):
            return self._forward(X_local, theta, a_src, a_dst, bias, beta)

    def _forward(self, X_local, theta, a_src, a_dst, bias, beta):
        ops, x = self.ops, self.x
        h, k, nl = self.h, self.k, self.r1 - self.r0
        X_local = X_local.contiguous()
        Mbuf, Mmine = self._buf(self.mx, h * k, nl)
        dbuf, dmine = self._buf(self.mx, h, nl)
        s_loc = ops.empty(nl, h, torch.float32)
        ops.transform(X_local, theta, h, k, a_src, a_dst, Mmine, s_loc, dmine)
        x.wait(x.start(dbuf, self.mx))
        wM = x.start(Mbuf, self.mx)  # overlaps the attention, which needs d only
        cache = {"X": X_local, "M": Mbuf, "Mmine": Mmine, "dbuf": dbuf, "dmine": dmine,
                 "beta": beta}
        mask = ops.mask(self.ne, h)
        if self.exchange == "stats":
            alpha = ops.empty(self.ne, h, torch.float32)
            sbuf, smine = self._buf(self.mx, 4 * h, nl)
            ops.attention(nl, self.rowptr, self.cols, h, s_loc, dbuf, beta, alpha, mask, smine,
                          self.rplan)
            cache.update(amine=alpha, stats=sbuf, smine=smine)
        else:
            abuf, amine = self._buf(self.emx, h, self.ne)
            ops.attention(nl, self.rowptr, self.cols, h, s_loc, dbuf, beta, amine, mask, None,
                          self.rplan)
            cache.update(alpha=abuf, amine=amine)
        cache["mask"] = mask
        x.wait(wM)
        out = ops.empty(nl, h * k, torch.float32)
        ops.aggregate(nl, self.rowptr, self.cols, h, k, cache["amine"], Mbuf, bias, out,
                      self.rplan)
        return out, cache

    def backward(self, G_local, theta, a_src, a_dst, cache, needs_feature_grad):
        with _scope(self.ops):
            return self._backward(G_local, theta, a_src, a_dst, cache, needs_feature_grad)

    def _backward(self, G_local, theta, a_src, a_dst, cache, needs_feature_grad, elu=None):
        """elu (optional): (mask, saved) of an ELU(1) below the layer; d_input
        gets its backward, fused into the d_input GEMM epilogue."""
        ops, x = self.ops, self.x
        h, k, nl = self.h, self.k, self.r1 - self.r0
        hk = h * k
        beta = cache["beta"]
        Gbuf, Gmine = self._buf(self.mx, hk, nl)
        Gmine.copy_(G_local)
        wG = x.start(Gbuf, self.mx)  # overlaps the SDDMM and the softmax backward
        da = ops.empty(self.ne, h, torch.float32)
        ops.sddmm(nl, self.rowptr, self.cols, h, k, cache["M"], Gmine, da, self.rplan)
        dS = ops.empty(nl, h, torch.float32)
        dD = ops.empty(nl, h, torch.float32)
        dM = ops.empty(nl, hk, torch.float32)
        if self.exchange == "stats":
            dy = ops.empty(self.ne, h, torch.float32)
            ops.softmax_backward(nl, self.rowptr, h, cache["amine"], cache["mask"], da, beta, dy,
                                 dS, cache["smine"], self.rplan)
            x.wait(x.start(cache["stats"], self.mx))
            x.wait(wG)
            ops.column_pass_stats(nl, self.colptr, self.crows, h, k, Gbuf, cache["stats"],
                                  cache["dmine"], cache["Mmine"], beta, dS, a_src, a_dst, dD, dM,
                                  self.cplan)
        else:
            dybuf, dymine = self._buf(self.emx, h, self.ne)
            ops.softmax_backward(nl, self.rowptr, h, cache["amine"], cache["mask"], da, beta,
                                 dymine, dS, None, self.rplan)
            wa = x.start(cache["alpha"], self.emx)
            x.wait(x.start(dybuf, self.emx))
            x.wait(wa)
            x.wait(wG)
            ops.column_pass(nl, self.colptr, self.crows, self.perm, h, k, Gbuf, cache["alpha"],
                            dybuf, dS, a_src, a_dst, dD, dM, self.cplan)
        flat = ops.empty(1, theta.numel() + 3 * hk, torch.float32).view(-1)
        d_theta = flat[:theta.numel()].view_as(theta)
        d_b = flat[theta.numel():theta.numel() + hk]
        d_as = flat[theta.numel() + hk:theta.numel() + 2 * hk].view(h, k)
        d_ad = flat[theta.numel() + 2 * hk:].view(h, k)
        ops.param_grads(nl, h, k, Gmine, cache["Mmine"], dS, dD, d_b, d_as, d_ad)
        ops.gemm(cache["X"], dM, True, False, out=d_theta)
        d_x = None
        if needs_feature_grad:
            d_x = ops.gemm(dM, theta, False, True) if elu is None else \
                ops.gemm_act(dM, theta, "elu_backward", elu[0], tb=True, saved=elu[1])
        x.allreduce(flat)
        return d_theta, d_as, d_ad, d_b, d_x


class DistGat2:
    """Gat2Model (model.hpp:123-201: GAT -> ELU(1) -> GAT, MSE step) over the
    row partition; both layers share the rank's pattern blocks (one
    DistGatLayer per width).  Parameters replicated, initialised like the
    reference (layer 1 GatParams(m, h, hidden, seed), layer 2
    GatParams(h * hidden, h, out, seed + 201))."""

    def __init__(self, l1: DistGatLayer, l2: DistGatLayer, m, hidden, out, heads, seed,
                 input_grad=False, beta=0.2, params=None):
        from . import device as d

        if params is None:
            params = list(d.gat_params(m, heads, hidden, seed)) + \
                list(d.gat_params(heads * hidden, heads, out, seed + 201))
        self.p = list(params)
        self.l1, self.l2 = l1, l2
        self.heads, self.out, self.beta, self.input_grad = heads, out, beta, input_grad

    def train_step(self, X_local, target_local):
        L1, L2 = self.l1, self.l2
        ops = L1.ops
        th1, as1, ad1, b1, th2, as2, ad2, b2 = self.p
        with _scope(ops):
            h, c1 = L1._forward(X_local, th1, as1, ad1, b1, self.beta)
            h, mask = ops.activation(h, "elu", out=h)
            o, c2 = L2._forward(h, th2, as2, ad2, b2, self.beta)
            loss, g = ops.loss_mse(o, target_local, L2.n * self.heads * self.out)
            L2.x.allreduce(loss)
            # the ELU backward fused into the layer-2 d_input GEMM (as model.cu)
            g2 = L2._backward(g, th2, as2, ad2, c2, True, elu=(mask, h))
            g1 = L1._backward(g2[4], th1, as1, ad1, c1, self.input_grad)
        return loss, o, list(g1[:4]) + list(g2[:4]), g1[4]
