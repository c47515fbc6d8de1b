"""Device-resident API over the C-ABI: torch tensors for memory and streams,
libsgnn_cuda.so for every computation.

Mirrors the reference's C++ layer API (gcn.hpp / gat.hpp / kernels.hpp /
sparse.hpp / pattern.hpp): `Adjacency` is AdjacencyOp, `Pattern` is
SparsePattern, `gcn_forward`/`gcn_backward`/`gat_forward`/`gat_backward`
take and return the same operands, caches are consume-once and the cache
levels / scheme choices are the reference's.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _capi as _c
from ._capi import Scheme, check, lib

_DT = {torch.float32: _c.F32, torch.float64: _c.F64}


def _p(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _dt(t):
    try:
        return _DT[t.dtype]
    except KeyError:
        raise ValueError(f"unsupported dtype {t.dtype}: float32 or float64 expected") from None


class _CudaArray:
    """Zero-copy view of a raw device pointer for torch.as_tensor."""

    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr,
                                         "data": (int(ptr or 0), False), "version": 3,
                                         "strides": None}


def _view(ptr, n, dtype, device):
    ts = {torch.int32: "<i4", torch.float32: "<f4", torch.float64: "<f8"}[dtype]
    if n == 0:
        return torch.empty(0, dtype=dtype, device=device)
    return torch.as_tensor(_CudaArray(ptr, n, ts), device=device).clone()


class Context:
    """One device + stream (sgnn_ctx).  Work is enqueued on torch's current
    stream at creation time so torch allocations and kernels stay ordered."""

    _default = {}

    def __init__(self, device=None, stream=None):
        if not torch.cuda.is_available():
            raise RuntimeError("sgnn-b200 needs a CUDA device (B200, sm_100a); no CPU fallback")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else int(device))
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.stream = s
        h = C.c_void_p()
        check(lib.sgnn_ctx_create(self.device.index, C.c_void_p(s.cuda_stream), C.byref(h)))
        self.handle = h

    @classmethod
    def default(cls, device=None):
        idx = torch.cuda.current_device() if device is None else int(device)
        ctx = cls._default.get(idx)
        if ctx is None:
            with torch.cuda.device(idx):
                ctx = cls._default[idx] = cls(idx)
        return ctx

    def set_stream(self, stream):
        """Enqueue subsequent work on `stream` (a torch.cuda.Stream), e.g. the
        capture stream of torch.cuda.graph: layer calls contain no host
        synchronisation, so a whole fwd+bwd step can be captured and replayed."""
        check(lib.sgnn_ctx_set_stream(self.handle, C.c_void_p(stream.cuda_stream)))
        self.stream = stream

    @property
    def launch_count(self):
        v = C.c_int64()
        check(lib.sgnn_ctx_launch_count(self.handle, C.byref(v)))
        return v.value

    def synchronize(self):
        check(lib.sgnn_ctx_synchronize(self.handle))

    def __del__(self, _destroy=lib.sgnn_ctx_destroy):
        if getattr(self, "handle", None):
            _destroy(self.handle)
            self.handle = None


MEM_CLASSES = {"untracked": 0, "transient": 1, "cache": 2, "output": 3, "all": 4}


def memory_stats(mem_class):
    """(live, peak, total) device bytes of a class (memtrack.hpp:19-94 on the
    device engine: layer intermediates charged with their logical sizes)."""
    live, peak, total = C.c_int64(), C.c_int64(), C.c_int64()
    check(lib.sgnn_mem_stats(MEM_CLASSES[mem_class], C.byref(live), C.byref(peak),
                             C.byref(total)))
    return live.value, peak.value, total.value


def reset_memory_peaks():
    """Peaks restart from the live level (memtrack.hpp:79-87)."""
    check(lib.sgnn_mem_reset_peaks())


def _ctx(ctx):
    return ctx if ctx is not None else Context.default()


class StepGraph:
    """A stream-ordered step (layer or model calls without host
    synchronisation) captured once into a CUDA graph and replayed: the same
    kernels with the per-launch CPU overhead removed.  `fn` is warmed up,
    captured on a side stream (the context's stream is switched for the
    capture), and its return value -- tensors from the graph's memory pool,
    rewritten by every replay -- is `outputs`."""

    def __init__(self, fn, ctx=None, warmup=1):
        self.ctx = ctx = _ctx(ctx)
        dev = ctx.device
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        prev = ctx.stream
        ctx.set_stream(side)
        try:
            with torch.cuda.stream(side):
                for _ in range(warmup):
                    fn()
                side.synchronize()
                self.graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(self.graph, stream=side):
                    self.outputs = fn()
        finally:
            ctx.set_stream(prev)
        torch.cuda.current_stream(dev).wait_stream(side)

    def replay(self):
        self.graph.replay()
        return self.outputs


# ---- selector / model (host-pure) -----------------------------------------
def resolve_scheme(policy, m, k, needs_feature_grad=False, caching=False) -> Scheme:
    """gcn.hpp:34-47; policy 'adaptive' | 'transform-first' | 'propagate-first'."""
    if isinstance(policy, str):
        if policy not in _c.POLICIES:
            raise ValueError("unknown scheme")
        policy = _c.POLICIES[policy]
    s = Scheme()
    check(lib.sgnn_resolve_scheme(int(policy), int(m), int(k), int(bool(needs_feature_grad)),
                                  int(bool(caching)), C.byref(s)))
    return s


def make_scheme(forward, backward, caching):
    names_f = {n: i for i, n in enumerate(_c.FWD_NAMES)}
    names_b = {n: i for i, n in enumerate(_c.BWD_NAMES)}
    return Scheme(names_f.get(forward, forward), names_b.get(backward, backward), int(caching))


# ---- deterministic inputs --------------------------------------------------
def random_uniform(rows, cols, seed, lo=-1.0, hi=1.0, dtype=torch.float32, ctx=None):
    """dense.hpp:45-53 DenseMatrix::random_uniform, generated on the device."""
    ctx = _ctx(ctx)
    out = torch.empty((rows, cols), dtype=dtype, device=ctx.device)
    check(lib.sgnn_random_uniform(ctx.handle, rows, cols, seed, lo, hi, _dt(out), _p(out)))
    return out


def gcn_params(m, k, seed, dtype=torch.float32, ctx=None):
    ctx = _ctx(ctx)
    th = torch.empty((m, k), dtype=dtype, device=ctx.device)
    b = torch.empty(k, dtype=dtype, device=ctx.device)
    check(lib.sgnn_gcn_params_init(ctx.handle, m, k, seed, _dt(th), _p(th), _p(b)))
    return th, b


def gat_params(m, h, k, seed, dtype=torch.float32, ctx=None):
    ctx = _ctx(ctx)
    dev = ctx.device
    th = torch.empty((m, h * k), dtype=dtype, device=dev)
    a_s = torch.empty((h, k), dtype=dtype, device=dev)
    a_d = torch.empty((h, k), dtype=dtype, device=dev)
    b = torch.empty(h * k, dtype=dtype, device=dev)
    check(lib.sgnn_gat_params_init(ctx.handle, m, h, k, seed, _dt(th), _p(th), _p(a_s), _p(a_d),
                                   _p(b)))
    return th, a_s, a_d, b


def synthetic_graph(n, avg_degree, seed):
    """graph.hpp:160-190 (host; sequential rejection sampler).  Returns int32
    CPU tensors (src, dst) in canonical order."""
    ne = lib.sgnn_synthetic_graph_edges(n, float(avg_degree))
    src = torch.empty(max(ne, 0), dtype=torch.int32)
    dst = torch.empty(max(ne, 0), dtype=torch.int32)
    check(lib.sgnn_synthetic_graph(n, float(avg_degree), seed, _p(src), _p(dst)))
    return src, dst


def powerlaw_graph(n, avg_degree, exponent=3.0, seed=1, ctx=None):
    """Chung-Lu power-law graph generated on the device (sgnn_powerlaw_graph):
    int32 device tensors (src, dst), undirected, canonical order."""
    ctx = _ctx(ctx)
    cap = lib.sgnn_powerlaw_graph_capacity(n, float(avg_degree))
    src = torch.empty(max(cap, 1), dtype=torch.int32, device=ctx.device)
    dst = torch.empty(max(cap, 1), dtype=torch.int32, device=ctx.device)
    cnt = C.c_int64()
    check(lib.sgnn_powerlaw_graph(ctx.handle, n, float(avg_degree), float(exponent), seed,
                                  _p(src), _p(dst), C.byref(cnt)))
    return src[:cnt.value], dst[:cnt.value]


# ---- sparse-format layer ---------------------------------------------------
def _i32(t, dev):
    return t.to(device=dev, dtype=torch.int32).contiguous()


def canonicalize(n_rows, n_cols, rows, cols, vals, ctx=None):
    """sparse.hpp:110-142 on the device -> canonical (rows, cols, vals)."""
    ctx = _ctx(ctx)
    dev = ctx.device
    rows, cols = _i32(rows, dev), _i32(cols, dev)
    vals = vals.to(dev).contiguous()
    if not (rows.numel() == cols.numel() == vals.numel()):
        raise ValueError("rows/cols/vals must have equal length")
    q = rows.numel()
    ro = torch.empty(q, dtype=torch.int32, device=dev)
    co = torch.empty(q, dtype=torch.int32, device=dev)
    vo = torch.empty(q, dtype=vals.dtype, device=dev)
    w = C.c_int64()
    check(lib.sgnn_coo_canonicalize(ctx.handle, n_rows, n_cols, q, _p(rows), _p(cols), _p(vals),
                                    _dt(vals), _p(ro), _p(co), _p(vo), C.byref(w)))
    return ro[:w.value], co[:w.value], vo[:w.value]


def add_self_loops(n, rows, cols, vals, ctx=None):
    ctx = _ctx(ctx)
    q = rows.numel()
    ro = torch.empty(q + n, dtype=torch.int32, device=ctx.device)
    co = torch.empty(q + n, dtype=torch.int32, device=ctx.device)
    vo = torch.empty(q + n, dtype=vals.dtype, device=ctx.device)
    w = C.c_int64()
    check(lib.sgnn_add_self_loops(ctx.handle, n, q, _p(rows), _p(cols), _p(vals), _dt(vals),
                                  _p(ro), _p(co), _p(vo), C.byref(w)))
    return ro[:w.value], co[:w.value], vo[:w.value]


def gcn_normalize(n, rows, cols, vals, ctx=None):
    """sparse.hpp:474-495 on a canonical COO (device tensors)."""
    ctx = _ctx(ctx)
    q = rows.numel()
    ro = torch.empty(q + n, dtype=torch.int32, device=ctx.device)
    co = torch.empty(q + n, dtype=torch.int32, device=ctx.device)
    vo = torch.empty(q + n, dtype=vals.dtype, device=ctx.device)
    w = C.c_int64()
    check(lib.sgnn_gcn_normalize(ctx.handle, n, q, _p(rows), _p(cols), _p(vals), _dt(vals),
                                 _p(ro), _p(co), _p(vo), C.byref(w)))
    return ro[:w.value], co[:w.value], vo[:w.value]


def csr_from_coo(n_rows, rows, ctx=None):
    ctx = _ctx(ctx)
    rp = torch.empty(n_rows + 1, dtype=torch.int32, device=ctx.device)
    check(lib.sgnn_csr_from_coo(ctx.handle, n_rows, rows.numel(), _p(rows), _p(rp)))
    return rp


def csc_from_coo(n_cols, rows, cols, vals, ctx=None):
    ctx = _ctx(ctx)
    q = rows.numel()
    dev = ctx.device
    cp = torch.empty(n_cols + 1, dtype=torch.int32, device=dev)
    cr = torch.empty(q, dtype=torch.int32, device=dev)
    cv = torch.empty(q, dtype=vals.dtype, device=dev)
    pm = torch.empty(q, dtype=torch.int32, device=dev)
    check(lib.sgnn_csc_from_coo(ctx.handle, n_cols, q, _p(rows), _p(cols), _p(vals), _dt(vals),
                                _p(cp), _p(cr), _p(cv), _p(pm)))
    return cp, cr, cv, pm


class Adjacency:
    """AdjacencyOp (kernels.hpp:191-211) from a canonical COO on the device."""

    def __init__(self, n_rows, n_cols, rows, cols, vals, format="csc", ctx=None):
        self.ctx = ctx = _ctx(ctx)
        if isinstance(format, str):
            if format not in _c.FORMATS:
                raise ValueError(f"unknown format '{format}'")
            format = _c.FORMATS[format]
        self.n_rows, self.n_cols, self.nnz = n_rows, n_cols, rows.numel()
        self.dtype = vals.dtype
        h = C.c_void_p()
        check(lib.sgnn_adj_create(ctx.handle, n_rows, n_cols, self.nnz, _p(rows), _p(cols),
                                  _p(vals), _dt(vals), int(format), C.byref(h)))
        self.handle = h

    @classmethod
    def from_coo(cls, n_rows, n_cols, rows, cols, vals, format="csc", ctx=None):
        r, c, v = canonicalize(n_rows, n_cols, rows, cols, vals, ctx)
        return cls(n_rows, n_cols, r, c, v, format, ctx)

    @classmethod
    def gcn_operator(cls, n, src, dst, dtype=torch.float32, format="csc", ctx=None):
        """adjacency(graph) -> gcn_normalize -> convert (bench.hpp:195-196)."""
        ctx = _ctx(ctx)
        ones = torch.ones(src.numel(), dtype=dtype, device=ctx.device)
        r, c, v = canonicalize(n, n, src, dst, ones, ctx)
        r, c, v = gcn_normalize(n, r, c, v, ctx)
        return cls(n, n, r, c, v, format, ctx)

    def spmm(self, B, transposed=False, bias=None, out=None):
        n_out = self.n_cols if transposed else self.n_rows
        n_in = self.n_rows if transposed else self.n_cols
        if B.dim() != 2 or B.shape[0] != n_in:
            raise ValueError("spmm: dimension mismatch")
        B = B.contiguous()
        if out is None:
            out = torch.empty((n_out, B.shape[1]), dtype=B.dtype, device=B.device)
        check(lib.sgnn_spmm(self.ctx.handle, self.handle, int(transposed), _p(B), B.shape[1],
                            _p(out), _p(bias)))
        return out

    multiply = spmm

    def multiply_transposed(self, B):
        return self.spmm(B, transposed=True)

    def __del__(self, _destroy=lib.sgnn_adj_destroy):
        if getattr(self, "handle", None):
            _destroy(self.handle)
            self.handle = None


class Pattern:
    """SparsePattern (pattern.hpp:17-95) from a device CSR."""

    def __init__(self, n, rowptr, cols, ctx=None):
        self.ctx = ctx = _ctx(ctx)
        self.n, self.nnz = n, cols.numel()
        h = C.c_void_p()
        check(lib.sgnn_pattern_create(ctx.handle, n, self.nnz, _p(rowptr), _p(cols),
                                      C.byref(h)))
        self.handle = h
        a = C.c_int()
        check(lib.sgnn_pattern_info(h, None, None, C.byref(a)))
        self.all_self_loops = bool(a.value)

    @classmethod
    def gat_pattern(cls, n, src, dst, ctx=None):
        """adjacency -> add_self_loops -> CSR -> SparsePattern (bench.hpp:208-209)."""
        ctx = _ctx(ctx)
        ones = torch.ones(src.numel(), dtype=torch.float32, device=ctx.device)
        r, c, v = canonicalize(n, n, src, dst, ones, ctx)
        r, c, v = add_self_loops(n, r, c, v, ctx)
        return cls(n, csr_from_coo(n, r, ctx), c, ctx)

    def arrays(self):
        ptrs = [C.c_void_p() for _ in range(6)]
        check(lib.sgnn_pattern_arrays(self.handle, *[C.byref(p) for p in ptrs]))
        dev = self.ctx.device
        sizes = [self.n + 1, self.nnz, self.n + 1, self.nnz, self.nnz, self.n]
        names = ["rowptr", "cols", "colptr", "rows", "perm", "diag"]
        return {nm: _view(p.value, sz, torch.int32, dev) for nm, p, sz in zip(names, ptrs, sizes)}

    def __del__(self, _destroy=lib.sgnn_pattern_destroy):
        if getattr(self, "handle", None):
            _destroy(self.handle)
            self.handle = None


# ---- kernels -----------------------------------------------------------------
def gemm(A, B, trans_a=False, trans_b=False, ctx=None, bias=None, out=None, colsum_b=None):
    """C = op(A) op(B) (+ bias fused); colsum_b (for A^T B): also 1^T B from
    the same read of B.  `out` may be a preallocated (e.g. strided-row) view."""
    ctx = _ctx(ctx)
    A, B = A.contiguous(), B.contiguous()
    m = A.shape[1] if trans_a else A.shape[0]
    n = B.shape[0] if trans_b else B.shape[1]
    if out is None:
        out = torch.empty((m, n), dtype=A.dtype, device=A.device)
    if bias is None and colsum_b is None:
        check(lib.sgnn_gemm(ctx.handle, _dt(A), _p(A), A.shape[0], A.shape[1], _p(B),
                            B.shape[0], B.shape[1], int(trans_a), int(trans_b), _p(out)))
    else:
        check(lib.sgnn_gemm_ex(ctx.handle, _dt(A), _p(A), A.shape[0], A.shape[1], _p(B),
                               B.shape[0], B.shape[1], int(trans_a), int(trans_b), _p(out),
                               _p(bias), _p(colsum_b)))
    return out


_GEMM_ACT = {"relu": 0, "relu_backward": 1, "elu_backward": 2}


def gemm_act(A, B, act, mask, trans_a=False, trans_b=False, bias=None, saved=None, out=None,
             ctx=None):
    """C = op(A) op(B) (+ bias) followed by an activation, fused into the
    tcgen05 epilogue where the shape allows it: act "relu" (writes `mask`),
    "relu_backward" / "elu_backward" (reads `mask`, and `saved` = the ELU
    output)."""
    ctx = _ctx(ctx)
    A, B = A.contiguous(), B.contiguous()
    m = A.shape[1] if trans_a else A.shape[0]
    n = B.shape[0] if trans_b else B.shape[1]
    if out is None:
        out = torch.empty((m, n), dtype=A.dtype, device=A.device)
    check(lib.sgnn_gemm_act(ctx.handle, _dt(A), _p(A), A.shape[0], A.shape[1], _p(B), B.shape[0],
                            B.shape[1], int(trans_a), int(trans_b), _p(out), _p(bias),
                            _GEMM_ACT[act], _p(mask), _p(saved)))
    return out


def column_sums(X, ctx=None):
    ctx = _ctx(ctx)
    X = X.contiguous()
    out = torch.empty(X.shape[1], dtype=X.dtype, device=X.device)
    check(lib.sgnn_column_sums(ctx.handle, _dt(X), _p(X), X.shape[0], X.shape[1], _p(out)))
    return out


def sddmm(pattern: Pattern, B, Cm):
    B, Cm = B.contiguous(), Cm.contiguous()
    if B.shape[1] != Cm.shape[0]:
        raise ValueError("sddmm: inner dimension mismatch")
    if B.shape[0] != pattern.n or Cm.shape[1] != pattern.n:
        raise ValueError("sddmm: outer dimension mismatch")
    out = torch.empty(pattern.nnz, dtype=B.dtype, device=B.device)
    check(lib.sgnn_sddmm(pattern.ctx.handle, pattern.handle, _p(B), B.shape[1], _p(Cm),
                         Cm.shape[1], _dt(B), _p(out)))
    return out


def edge_softmax(pattern: Pattern, w):
    """w: edge-major (q, heads) or (q,) -> alpha of the same shape."""
    w = w.contiguous()
    heads = 1 if w.dim() == 1 else w.shape[1]
    out = torch.empty_like(w)
    check(lib.sgnn_edge_softmax(pattern.ctx.handle, pattern.handle, heads, _p(w), _dt(w),
                                _p(out)))
    return out


# ---- GCN layer (gcn.hpp:91-193) ------------------------------------------------
class GcnCache:
    def __init__(self, handle, X, scheme):
        self.handle, self._X, self.scheme = handle, X, scheme  # X kept alive (borrowed)

    def retained_bytes(self):
        v = C.c_int64()
        check(lib.sgnn_gcn_cache_retained_bytes(self.handle, C.byref(v)))
        return v.value

    def __del__(self, _destroy=lib.sgnn_gcn_cache_destroy):
        if getattr(self, "handle", None):
            _destroy(self.handle)
            self.handle = None


def gcn_forward(adj: Adjacency, X, theta, bias, scheme, out=None):
    X, theta, bias = X.contiguous(), theta.contiguous(), bias.contiguous()
    if adj.n_rows != adj.n_cols or adj.n_cols != X.shape[0]:
        raise ValueError("gcn_forward: adjacency/input shape mismatch")
    if X.shape[1] != theta.shape[0]:
        raise ValueError("gcn_forward: input width does not match theta")
    if bias.numel() != theta.shape[1]:
        raise ValueError("bias_add_rows: bias length does not match columns")
    if X.dtype != adj.dtype or theta.dtype != adj.dtype:
        raise ValueError("gcn_forward: dtype mismatch")
    n, m, k = X.shape[0], X.shape[1], theta.shape[1]
    if out is None:
        out = torch.empty((n, k), dtype=X.dtype, device=X.device)
    h = C.c_void_p()
    check(lib.sgnn_gcn_forward(adj.ctx.handle, adj.handle, _p(X), m, _p(theta), _p(bias), k,
                               C.byref(scheme), _p(out), C.byref(h)))
    return out, GcnCache(h, X, scheme)


def gcn_backward(adj: Adjacency, d_out, theta, cache: GcnCache, needs_feature_grad,
                 d_theta=None, d_bias=None, d_input=None):
    d_out, theta = d_out.contiguous(), theta.contiguous()
    m, k = theta.shape
    dev, dt = d_out.device, d_out.dtype
    if d_out.shape != (adj.n_rows, k):
        lib.sgnn_gcn_backward(adj.ctx.handle, adj.handle, None, None, -1, -1, cache.handle, 0,
                              None, None, None)  # marks the cache consumed, like gcn.hpp:137
        raise ValueError("gcn_backward: gradient shape mismatch")
    d_theta = torch.empty((m, k), dtype=dt, device=dev) if d_theta is None else d_theta
    d_bias = torch.empty(k, dtype=dt, device=dev) if d_bias is None else d_bias
    if needs_feature_grad and d_input is None:
        d_input = torch.empty((adj.n_rows, m), dtype=dt, device=dev)
    check(lib.sgnn_gcn_backward(adj.ctx.handle, adj.handle, _p(d_out), _p(theta), m, k,
                                cache.handle, int(bool(needs_feature_grad)), _p(d_theta),
                                _p(d_bias), _p(d_input) if needs_feature_grad else None))
    return d_theta, d_bias, (d_input if needs_feature_grad else None)


def _host(t, name):
    if t.device.type != "cpu" or not t.is_contiguous():
        raise ValueError(f"{name}: contiguous host tensor expected")
    return t


def gcn_step_host(adj: Adjacency, hX, theta, bias, scheme, hG, needs_feature_grad,
                  h_out, h_d_theta, h_d_bias, h_d_input=None):
    """One GCN forward+backward step from HOST buffers (pinned for async
    copies): X and dX' in, out / dTheta / db / dX out; parameters on the
    device.  Copies overlap compute and each other (pipeline.cu).  Stream-
    ordered: synchronize the context before reading the host outputs."""
    m, k = theta.shape
    for t, nm in ((hX, "X"), (hG, "d_out"), (h_out, "out"), (h_d_theta, "d_theta"),
                  (h_d_bias, "d_bias")):
        _host(t, nm)
    if hX.shape != (adj.n_rows, m) or hG.shape != (adj.n_rows, k):
        raise ValueError("gcn_step_host: shape mismatch")
    if needs_feature_grad:
        _host(h_d_input, "d_input")
    check(lib.sgnn_gcn_step_host(adj.ctx.handle, adj.handle, _p(hX), m, _p(theta.contiguous()),
                                 _p(bias.contiguous()), k, C.byref(scheme), _p(hG),
                                 int(bool(needs_feature_grad)), _p(h_out), _p(h_d_theta),
                                 _p(h_d_bias), _p(h_d_input) if needs_feature_grad else None))


def gat_step_host(pattern: Pattern, hX, theta, a_src, a_dst, bias, heads, beta, level, hG,
                  needs_feature_grad, h_out, h_d_theta, h_d_a_src, h_d_a_dst, h_d_bias,
                  h_d_input=None):
    """GAT counterpart of gcn_step_host (gat.hpp:89-219 from host buffers)."""
    if isinstance(level, str):
        level = _c.LEVELS[level]
    m, hk = theta.shape
    k = hk // heads
    for t, nm in ((hX, "X"), (hG, "d_out"), (h_out, "out"), (h_d_theta, "d_theta")):
        _host(t, nm)
    if hX.shape != (pattern.n, m) or hG.shape != (pattern.n, hk):
        raise ValueError("gat_step_host: shape mismatch")
    check(lib.sgnn_gat_step_host(pattern.ctx.handle, pattern.handle, _p(hX), m,
                                 _p(theta.contiguous()), _p(a_src.contiguous()),
                                 _p(a_dst.contiguous()), _p(bias.contiguous()), heads, k,
                                 float(beta), int(level), _dt(theta), _p(hG),
                                 int(bool(needs_feature_grad)), _p(h_out), _p(h_d_theta),
                                 _p(h_d_a_src), _p(h_d_a_dst), _p(h_d_bias),
                                 _p(h_d_input) if needs_feature_grad else None))


# ---- GAT layer (gat.hpp:89-219) ------------------------------------------------
class GatCache:
    def __init__(self, handle, X, level, heads, k):
        self.handle, self._X, self.level, self.heads, self.k = handle, X, level, heads, k

    def extra_bytes(self):
        v = C.c_int64()
        check(lib.sgnn_gat_cache_extra_bytes(self.handle, C.byref(v)))
        return v.value

    @property
    def reordered(self):
        """True when the forward ran operator-reordered (gat_forward reorder=True)."""
        v = C.c_int()
        check(lib.sgnn_gat_cache_reordered(self.handle, C.byref(v)))
        return bool(v.value)

    def edge_values(self, pattern: Pattern, theta, a_src, a_dst):
        """alpha (h x q) and mask (h x q uint8), head-major like the reference."""
        dev = pattern.ctx.device
        alpha = torch.empty((self.heads, pattern.nnz), dtype=theta.dtype, device=dev)
        mask = torch.empty((self.heads, pattern.nnz), dtype=torch.uint8, device=dev)
        check(lib.sgnn_gat_cache_edge_values(pattern.ctx.handle, pattern.handle, self.handle,
                                             _p(theta), _p(a_src), _p(a_dst), _p(alpha),
                                             _p(mask)))
        return alpha, mask

    def __del__(self, _destroy=lib.sgnn_gat_cache_destroy):
        if getattr(self, "handle", None):
            _destroy(self.handle)
            self.handle = None


def gat_forward(pattern: Pattern, X, theta, a_src, a_dst, bias, heads, beta=0.2,
                level="none", out=None, reorder=False):
    """One GAT layer forward (gat.hpp:89-147).  reorder=True lets the device
    run it operator-reordered when the heads are wider than the input (k > m,
    float32; sgnn_gat_forward_ex): same outputs and gradients within float32
    rounding, the cache keeps Z = sum_j alpha X_j in place of M."""
    X, theta = X.contiguous(), theta.contiguous()
    a_src, a_dst, bias = a_src.contiguous(), a_dst.contiguous(), bias.contiguous()
    if isinstance(level, str):
        if level not in _c.LEVELS:
            raise ValueError(f"unknown caching level '{level}'")
        level = _c.LEVELS[level]
    if theta.shape[1] % heads != 0:
        raise ValueError("theta width must be heads*k")
    if pattern.n != X.shape[0]:
        raise ValueError("gat_forward: node count mismatch")
    if X.shape[1] != theta.shape[0]:
        raise ValueError("gat_forward: input width does not match theta")
    n, m, hk = X.shape[0], X.shape[1], theta.shape[1]
    k = hk // heads
    if out is None:
        out = torch.empty((n, hk), dtype=X.dtype, device=X.device)
    h = C.c_void_p()
    check(lib.sgnn_gat_forward_ex(pattern.ctx.handle, pattern.handle, _p(X), m, _p(theta),
                                  _p(a_src), _p(a_dst), _p(bias), heads, k, float(beta),
                                  int(level), _dt(X), _p(out), C.byref(h),
                                  _c.GAT_REORDER if reorder else 0))
    return out, GatCache(h, X, level, heads, k)


def gat_backward(pattern: Pattern, d_out, theta, a_src, a_dst, cache: GatCache,
                 needs_feature_grad, beta=0.2):
    d_out = d_out.contiguous()
    m, hk = theta.shape
    h, k = cache.heads, cache.k
    dev, dt = d_out.device, d_out.dtype
    d_theta = torch.empty((m, hk), dtype=dt, device=dev)
    d_as = torch.empty((h, k), dtype=dt, device=dev)
    d_ad = torch.empty((h, k), dtype=dt, device=dev)
    d_b = torch.empty(hk, dtype=dt, device=dev)
    d_x = torch.empty((pattern.n, m), dtype=dt, device=dev) if needs_feature_grad else None
    if d_out.shape != (pattern.n, hk):
        raise ValueError("gat_backward: gradient shape mismatch")
    check(lib.sgnn_gat_backward(pattern.ctx.handle, pattern.handle, _p(d_out), _p(theta),
                                _p(a_src), _p(a_dst), m, h, k, float(beta), cache.handle,
                                int(bool(needs_feature_grad)), _p(d_theta), _p(d_as), _p(d_ad),
                                _p(d_b), _p(d_x)))
    return d_theta, d_as, d_ad, d_b, d_x


# ---- activations / loss (dense.hpp:197-268, model.hpp loss_mse) ---------------
_ACT = {"relu": 0, "elu": 2}


def activation(X, kind, out=None, ctx=None):
    """(out, mask): relu or elu(1); out may be X itself (in place)."""
    ctx = _ctx(ctx)
    X = X.contiguous()
    out = torch.empty_like(X) if out is None else out
    mask = torch.empty(X.shape, dtype=torch.uint8, device=X.device)
    check(lib.sgnn_activation(ctx.handle, _ACT[kind], _dt(X), _p(X), X.numel(), _p(out),
                              _p(mask)))
    return out, mask


def activation_backward(grad_out, mask, kind, saved=None, out=None, ctx=None):
    ctx = _ctx(ctx)
    grad_out = grad_out.contiguous()
    out = torch.empty_like(grad_out) if out is None else out
    check(lib.sgnn_activation_backward(ctx.handle, _ACT[kind], _dt(grad_out), _p(grad_out),
                                       _p(mask), _p(saved), grad_out.numel(), _p(out)))
    return out


def loss_mse(out, target, total=None, ctx=None):
    """(loss device float64 scalar, grad); total = size of the whole
    prediction when `out` is a row block of it."""
    ctx = _ctx(ctx)
    out, target = out.contiguous(), target.contiguous()
    if out.shape != target.shape:
        raise ValueError("loss_mse: target shape mismatch")
    grad = torch.empty_like(out)
    loss = torch.zeros((), dtype=torch.float64, device=out.device)
    check(lib.sgnn_loss_mse(ctx.handle, _dt(out), _p(out), _p(target), out.numel(),
                            out.numel() if total is None else int(total), _p(grad), _p(loss)))
    return loss, grad


# ---- two-layer models (model.hpp:16-245) -----------------------------------------
class Model:
    """Gcn2Model / Gat2Model (model.hpp:40-245) over sgnn_model: GCN -> ReLU ->
    GCN or GAT -> ELU(1) -> GAT.  Parameters live on the device, initialised
    like the reference constructors (layer 2 from seed+101 / seed+201);
    `params` are zero-copy views in param_tensors() order (valid while the
    model lives).  `train_step` is the benchmark step (bench.hpp:193-219):
    forward, loss_mse against `target`, backward."""

    KINDS = {"gcn2": 0, "gat2": 1}

    def __init__(self, kind, in_features, hidden, out_features, heads=1, scheme="adaptive",
                 caching=False, gat_level="none", leaky_slope=0.2, input_grad=False, seed=0,
                 dtype=torch.float32, ctx=None):
        self.ctx = _ctx(ctx)
        if kind not in self.KINDS:
            raise ValueError(f"unknown model kind '{kind}'")
        if isinstance(scheme, str):
            if scheme not in _c.POLICIES:
                raise ValueError("unknown scheme")
            scheme = _c.POLICIES[scheme]
        if isinstance(gat_level, str):
            if gat_level not in _c.LEVELS:
                raise ValueError(f"unknown caching level '{gat_level}'")
            gat_level = _c.LEVELS[gat_level]
        self.kind, self.dtype = kind, dtype
        self.cfg = _c.ModelConfig(self.KINDS[kind], in_features, hidden, out_features, heads,
                                  scheme, int(bool(caching)), gat_level, float(leaky_slope),
                                  int(bool(input_grad)))
        h = C.c_void_p()
        check(lib.sgnn_model_create(self.ctx.handle, C.byref(self.cfg), int(seed),
                                    _DT[dtype], C.byref(h)))
        self.handle = h
        m, hid, o = in_features, hidden, out_features
        shapes = ([(m, hid), (hid,), (hid, o), (o,)] if kind == "gcn2" else
                  [(m, heads * hid), (heads, hid), (heads, hid), (heads * hid,),
                   (heads * hid, heads * o), (heads, o), (heads, o), (heads * o,)])
        cnt = C.c_int32()
        check(lib.sgnn_model_num_params(h, C.byref(cnt)))
        ts = {torch.float32: "<f4", torch.float64: "<f8"}[dtype]
        self.params = []
        for i in range(cnt.value):
            ptr, size, name = C.c_void_p(), C.c_int64(), C.c_char_p()
            check(lib.sgnn_model_param(h, i, C.byref(ptr), C.byref(size), C.byref(name)))
            t = torch.as_tensor(_CudaArray(ptr.value, size.value, ts), device=self.ctx.device)
            self.params.append((name.value.decode(), t.view(shapes[i])))
        self.out_width = o if kind == "gcn2" else heads * o

    def param_tensors(self):
        return self.params

    def train_step(self, graph, X, target, out=None):
        """graph: Adjacency (gcn2) or Pattern (gat2).  Returns (loss, out,
        grads, d_input): loss a device float64 scalar, grads in params order."""
        X, target = X.contiguous(), target.contiguous()
        n = X.shape[0]
        if target.shape != (n, self.out_width):
            raise ValueError("loss_mse: target shape mismatch")
        dev = self.ctx.device
        if out is None:
            out = torch.empty((n, self.out_width), dtype=self.dtype, device=dev)
        grads = [torch.empty_like(p) for _, p in self.params]
        gp = (C.c_void_p * len(grads))(*[g.data_ptr() for g in grads])
        d_in = torch.empty_like(X) if self.cfg.input_grad else None
        loss = torch.zeros((), dtype=torch.float64, device=dev)
        adj = graph.handle if self.kind == "gcn2" else None
        pat = graph.handle if self.kind == "gat2" else None
        check(lib.sgnn_model_train_step(self.ctx.handle, self.handle, adj, pat, _p(X), _p(target),
                                        _p(out), gp, _p(d_in), _p(loss)))
        return loss, out, grads, d_in

    def __del__(self, _destroy=lib.sgnn_model_destroy):
        if getattr(self, "handle", None):
            _destroy(self.handle)
            self.handle = None
