"""numpy/ctypes front of the C oracle -- TEST INFRASTRUCTURE ONLY.

Wraps ``liboracle.so`` (oracle/sgnn_oracle.c, a single-threaded C
restatement of the reference's GCN/GAT hot path; every C function cites the
reference file:line it follows).  Only tests/, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` leg may import this module, and only as the
checker.  The product package never imports it.

Parity pin: tests/test_oracle_golden.py checks these functions bit-for-bit
against tests/golden/*.npz, which oracle/gen_golden.py produced by running the
reference itself (oracle/_ref/libsgnn_ref.so, compiled from the unmodified
reference headers).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")


def _load():
    if not os.path.exists(_LIB_PATH):
        subprocess.check_call(["make", "-s", "liboracle.so"], cwd=_HERE)
    lib = C.CDLL(_LIB_PATH)
    I32, I64, U64, D, INT = C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_int
    sig = {
        "orc_random_uniform": (None, [I64, I64, U64, D, D, f64p]),
        "orc_random_uniform_f32": (None, [I64, I64, U64, D, D, f32p]),
        "orc_rng_u64": (None, [U64, I64, u64p]),
        "orc_rng_below": (None, [U64, U64, I64, u64p]),
        "orc_synthetic_graph_edges": (I64, [I32, D]),
        "orc_synthetic_graph": (INT, [I32, D, U64, i32p, i32p]),
        "orc_coo_canonicalize": (I64, [I32, I32, I64, i32p, i32p, f64p, i32p, i32p, f64p]),
        "orc_coo_to_csr": (None, [I32, I64, i32p, i32p]),
        "orc_coo_to_csc": (None, [I32, I64, i32p, i32p, f64p, i32p, i32p, f64p, i32p]),
        "orc_add_self_loops": (I64, [I32, I64, i32p, i32p, f64p, i32p, i32p, f64p]),
        "orc_gcn_normalize": (I64, [I32, I64, i32p, i32p, f64p, i32p, i32p, f64p]),
        "orc_gcn_normalize_f32": (I64, [I32, I64, i32p, i32p, f32p, i32p, i32p, f32p]),
        "orc_pattern_build": (INT, [I32, i32p, i32p, i32p, i32p, i32p, i32p]),
        "orc_spmm_csr": (None, [I32, i32p, i32p, f64p, f64p, I32, f64p]),
        "orc_spmm_csr_f32": (None, [I32, i32p, i32p, f32p, f32p, I32, f32p]),
        "orc_sddmm": (None, [I32, i32p, i32p, f64p, I32, f64p, I32, f64p]),
        "orc_edge_softmax": (INT, [I32, i32p, I64, I32, f64p, f64p]),
        "orc_spmm_semibatched": (None, [I32, i32p, i32p, I64, I32, I32, f64p, f64p, f64p]),
        "orc_gemm": (INT, [f64p, I32, I32, f64p, I32, I32, INT, INT, f64p]),
        "orc_column_sums": (None, [f64p, I32, I32, f64p]),
        "orc_max_rel_diff": (D, [f64p, f64p, I64]),
        "orc_max_rel_diff_f32": (D, [f32p, f64p, I64]),
        "orc_activation": (None, [f64p, I64, INT, D, f64p, u8p]),
        "orc_activation_backward": (None, [f64p, u8p, I64, INT, D, C.c_void_p, f64p]),
        "orc_loss_mse": (D, [f64p, f64p, I64, f64p]),
        "orc_spmm_cost": (INT, [INT, I64, I64, I64, I64, I64, I64, C.POINTER(I64),
                                C.POINTER(I64), C.POINTER(D)]),
        "orc_sddmm_cost": (INT, [INT, I64, I64, I64, I64, I64, I64, C.POINTER(I64),
                                 C.POINTER(I64), C.POINTER(D)]),
        "orc_gcn_select_scheme": (INT, [I64, I64, INT, INT, C.POINTER(INT), C.POINTER(INT),
                                        C.POINTER(INT)]),
        "orc_resolve_scheme": (INT, [INT, I64, I64, INT, INT, C.POINTER(INT), C.POINTER(INT),
                                     C.POINTER(INT)]),
        "orc_gcn_forward_flops": (I64, [INT, I64, I64, I64, I64]),
        "orc_gcn_backward_flops": (I64, [INT, I64, I64, I64, I64, INT]),
        "orc_gcn_forward_transients": (I64, [INT, I64, I64, I64]),
        "orc_gcn_backward_transients": (I64, [INT, I64, I64, I64, INT]),
        "orc_gat_cache_footprint": (I64, [INT, I64, I64, I64, I64, I64]),
        "orc_gcn_params_init": (None, [I32, I32, U64, f64p, f64p]),
        "orc_gcn_forward": (INT, [I32, i32p, i32p, f64p, f64p, I32, f64p, f64p, I32, INT,
                                  f64p, C.c_void_p]),
        "orc_gcn_backward": (INT, [I32, i32p, i32p, f64p, i32p, i32p, f64p, f64p, f64p, I32,
                                   f64p, I32, INT, INT, f64p, f64p, C.c_void_p]),
        "orc_gat_params_init": (None, [I32, I32, I32, U64, f64p, f64p, f64p, f64p]),
        "orc_gat_forward": (INT, [I32, i32p, i32p, f64p, I32, f64p, f64p, f64p, f64p, I32,
                                  I32, D, f64p, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_void_p]),
        "orc_gat_backward": (INT, [I32, i32p, i32p, i32p, i32p, i32p, f64p, f64p, I32, f64p,
                                   f64p, f64p, I32, I32, D, INT, f64p, f64p, f64p, f64p,
                                   C.c_void_p]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = _load()

FORMATS = {"coo": 0, "csr": 1, "csc": 2, "ellpack": 3, "hybrid": 4}
FWD_NAMES = ["transform_first", "propagate_first", "propagate_first_cached"]
BWD_NAMES = ["fused_propagate", "split_propagate", "split_propagate_cached"]
LEVELS = {"none": 0, "features": 1, "node-attn": 2, "full": 3}


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ---- rng / graph ---------------------------------------------------------
def random_uniform(rows, cols, seed, lo=-1.0, hi=1.0, dtype=np.float64):
    out = np.empty((rows, cols), dtype=dtype)
    if dtype == np.float32:
        _lib.orc_random_uniform_f32(rows, cols, seed, lo, hi, out)
    else:
        _lib.orc_random_uniform(rows, cols, seed, lo, hi, out)
    return out


def synthetic_graph(n, avg_degree, seed):
    ne = _lib.orc_synthetic_graph_edges(n, avg_degree)
    src = np.empty(ne, np.int32)
    dst = np.empty(ne, np.int32)
    if _lib.orc_synthetic_graph(n, avg_degree, seed, src, dst) != 0:
        raise ValueError("synthetic_graph: invalid arguments")
    return n, src, dst


# ---- sparse --------------------------------------------------------------
def coo_canonicalize(n_rows, n_cols, rows, cols, vals):
    rows, cols, vals = _i32(rows), _i32(cols), _f64(vals)
    q = len(rows)
    ro, co, vo = np.empty(q, np.int32), np.empty(q, np.int32), np.empty(q, np.float64)
    w = _lib.orc_coo_canonicalize(n_rows, n_cols, q, rows, cols, vals, ro, co, vo)
    if w < 0:
        raise ValueError("coo_from_triplets: index out of range")
    return ro[:w].copy(), co[:w].copy(), vo[:w].copy()


def coo_to_csr(n_rows, rows):
    rp = np.empty(n_rows + 1, np.int32)
    _lib.orc_coo_to_csr(n_rows, len(rows), _i32(rows), rp)
    return rp


def coo_to_csc(n_cols, rows, cols, vals):
    q = len(rows)
    cp = np.empty(n_cols + 1, np.int32)
    r, v, p = np.empty(q, np.int32), np.empty(q, np.float64), np.empty(q, np.int32)
    _lib.orc_coo_to_csc(n_cols, q, _i32(rows), _i32(cols), _f64(vals), cp, r, v, p)
    return cp, r, v, p


def add_self_loops(n, rows, cols, vals):
    q = len(rows)
    ro, co, vo = np.empty(q + n, np.int32), np.empty(q + n, np.int32), np.empty(q + n)
    w = _lib.orc_add_self_loops(n, q, _i32(rows), _i32(cols), _f64(vals), ro, co, vo)
    return ro[:w].copy(), co[:w].copy(), vo[:w].copy()


def gcn_normalize(n, rows, cols, vals, dtype=np.float64):
    """canonical COO in -> normalized canonical COO (sparse.hpp:474-495)."""
    q = len(rows)
    ro, co = np.empty(q + n, np.int32), np.empty(q + n, np.int32)
    if dtype == np.float32:
        vo = np.empty(q + n, np.float32)
        w = _lib.orc_gcn_normalize_f32(n, q, _i32(rows), _i32(cols),
                                       np.ascontiguousarray(vals, np.float32), ro, co, vo)
    else:
        vo = np.empty(q + n, np.float64)
        w = _lib.orc_gcn_normalize(n, q, _i32(rows), _i32(cols), _f64(vals), ro, co, vo)
    if w < 0:
        raise ValueError("gcn_normalize: negative edge weight")
    return ro[:w].copy(), co[:w].copy(), vo[:w].copy()


def pattern_build(n, rowptr, cols):
    q = int(rowptr[n])
    cp, r, p, d = (np.empty(n + 1, np.int32), np.empty(q, np.int32), np.empty(q, np.int32),
                   np.empty(n, np.int32))
    all_loops = _lib.orc_pattern_build(n, _i32(rowptr), _i32(cols), cp, r, p, d)
    return cp, r, p, d, bool(all_loops)


class Operator:
    """Canonical COO + CSR + CSC of one square sparse operator (AdjacencyOp,
    kernels.hpp:191-211)."""

    def __init__(self, n, rows, cols, vals):
        self.n = n
        self.rows, self.cols, self.vals = _i32(rows), _i32(cols), _f64(vals)
        self.rowptr = coo_to_csr(n, self.rows)
        self.colptr, self.crows, self.cvals, self.perm = coo_to_csc(n, self.rows, self.cols,
                                                                    self.vals)

    @property
    def nnz(self):
        return len(self.rows)


def gcn_operator(n, src, dst):
    """adjacency(graph) -> gcn_normalize (bench.hpp:195-196)."""
    r, c, v = coo_canonicalize(n, n, src, dst, np.ones(len(src)))
    return Operator(n, *gcn_normalize(n, r, c, v))


def gat_pattern(n, src, dst):
    """adjacency -> add_self_loops -> CSR -> SparsePattern (bench.hpp:208-209)."""
    r, c, v = coo_canonicalize(n, n, src, dst, np.ones(len(src)))
    return Operator(n, *add_self_loops(n, r, c, v))


# ---- kernels -------------------------------------------------------------
def spmm_csr(rowptr, cols, vals, B):
    B = np.ascontiguousarray(B)
    n_rows = len(rowptr) - 1
    f = B.shape[1]
    if B.dtype == np.float32:
        C_ = np.empty((n_rows, f), np.float32)
        _lib.orc_spmm_csr_f32(n_rows, _i32(rowptr), _i32(cols),
                              np.ascontiguousarray(vals, np.float32), B, f, C_)
    else:
        C_ = np.empty((n_rows, f), np.float64)
        _lib.orc_spmm_csr(n_rows, _i32(rowptr), _i32(cols), _f64(vals), _f64(B), f, C_)
    return C_


def sddmm(rowptr, cols, B, Cm):
    B, Cm = _f64(B), _f64(Cm)
    n = len(rowptr) - 1
    out = np.empty(int(rowptr[n]), np.float64)
    _lib.orc_sddmm(n, _i32(rowptr), _i32(cols), B, B.shape[1], Cm, Cm.shape[1], out)
    return out


def edge_softmax(rowptr, w):
    """w: head-major (h, q)."""
    w = _f64(np.atleast_2d(w))
    n = len(rowptr) - 1
    out = np.empty_like(w)
    if _lib.orc_edge_softmax(n, _i32(rowptr), w.shape[1], w.shape[0], w, out) != 0:
        raise ValueError("edge_softmax: pattern must contain all self loops")
    return out


def gemm(A, B, trans_a=False, trans_b=False):
    A, B = _f64(A), _f64(B)
    m = A.shape[1] if trans_a else A.shape[0]
    n = B.shape[0] if trans_b else B.shape[1]
    Cm = np.empty((m, n), np.float64)
    if _lib.orc_gemm(A, A.shape[0], A.shape[1], B, B.shape[0], B.shape[1], int(trans_a),
                     int(trans_b), Cm) != 0:
        raise ValueError("gemm: inner dimensions do not match")
    return Cm


def column_sums(X):
    X = _f64(X)
    out = np.empty(X.shape[1])
    _lib.orc_column_sums(X, X.shape[0], X.shape[1], out)
    return out


def max_rel_diff(a, b):
    """dense.hpp:303-316 on the flattened arrays (b promoted to float64)."""
    b = _f64(b).ravel()
    if np.asarray(a).dtype == np.float32:
        a = np.ascontiguousarray(a, np.float32).ravel()
        assert a.size == b.size
        return _lib.orc_max_rel_diff_f32(a, b, a.size)
    a = _f64(a).ravel()
    assert a.size == b.size
    return _lib.orc_max_rel_diff(a, b, a.size)


def activation(X, kind, param=0.0):
    X = _f64(X)
    out, mask = np.empty_like(X), np.empty(X.shape, np.uint8)
    _lib.orc_activation(X, X.size, {"relu": 0, "leaky_relu": 1, "elu": 2}[kind], param, out,
                        mask)
    return out, mask


def activation_backward(g, mask, kind, param=0.0, saved=None):
    g = _f64(g)
    out = np.empty_like(g)
    saved = None if saved is None else _f64(saved)
    _lib.orc_activation_backward(g, np.ascontiguousarray(mask, np.uint8), g.size,
                                 {"relu": 0, "leaky_relu": 1, "elu": 2}[kind], param,
                                 _ptr(saved), out)
    return out


def loss_mse(out, target):
    out, target = _f64(out), _f64(target)
    grad = np.empty_like(out)
    v = _lib.orc_loss_mse(out, target, out.size, grad)
    return v, grad


# ---- cost / selector -----------------------------------------------------
def _cost(fn, fmt, n, q, p, f, sb, ib):
    fl, by, oi = C.c_int64(), C.c_int64(), C.c_double()
    if fn(FORMATS[fmt], n, q, p, f, sb, ib, C.byref(fl), C.byref(by), C.byref(oi)) != 0:
        raise ValueError("cost: invalid format/arguments")
    return {"flops": fl.value, "bytes": by.value, "operational_intensity": oi.value}


def spmm_cost(fmt, n, q, p=0, f=64, scalar_bytes=4, index_bytes=4):
    return _cost(_lib.orc_spmm_cost, fmt, n, q, p, f, scalar_bytes, index_bytes)


def sddmm_cost(fmt, n, q, p=0, f=64, scalar_bytes=4, index_bytes=4):
    return _cost(_lib.orc_sddmm_cost, fmt, n, q, p, f, scalar_bytes, index_bytes)


def resolve_scheme(policy, m, k, fg=False, caching=False):
    """policy: 0 adaptive, 1 force transform-first, 2 force propagate-first.
    Returns (fwd, bwd, caching) ints."""
    a, b, c = C.c_int(), C.c_int(), C.c_int()
    if _lib.orc_resolve_scheme(policy, m, k, int(fg), int(caching), C.byref(a), C.byref(b),
                               C.byref(c)) != 0:
        raise ValueError("gcn_select_scheme: m and k must be >= 1")
    return a.value, b.value, c.value


def gcn_select_scheme(m, k, needs_feature_grad=False, caching=False):
    f, b, c = resolve_scheme(0, m, k, needs_feature_grad, caching)
    return {"forward": FWD_NAMES[f], "backward": BWD_NAMES[b], "caching": bool(c)}


gcn_forward_flops = lambda s, n, m, k, q: _lib.orc_gcn_forward_flops(s, n, m, k, q)  # noqa
gcn_backward_flops = lambda s, n, m, k, q, fg: _lib.orc_gcn_backward_flops(s, n, m, k, q, int(fg))  # noqa
gcn_forward_transients = lambda s, n, m, k: _lib.orc_gcn_forward_transients(s, n, m, k)  # noqa
gcn_backward_transients = lambda s, n, m, k, fg: _lib.orc_gcn_backward_transients(s, n, m, k, int(fg))  # noqa


def gat_cache_footprint(level, n, h, k, q, scalar_bytes=4):
    return _lib.orc_gat_cache_footprint(LEVELS[level], n, h, k, q, scalar_bytes)


# ---- layers --------------------------------------------------------------
def gcn_params(m, k, seed):
    th, b = np.empty((m, k)), np.empty(k)
    _lib.orc_gcn_params_init(m, k, seed, th, b)
    return th, b


def gat_params(m, h, k, seed):
    th, a_s, a_d, b = np.empty((m, h * k)), np.empty((h, k)), np.empty((h, k)), np.empty(h * k)
    _lib.orc_gat_params_init(m, h, k, seed, th, a_s, a_d, b)
    return th, a_s, a_d, b


def gcn_forward(op: Operator, X, theta, bias, fwd_scheme):
    X, theta, bias = _f64(X), _f64(theta), _f64(bias)
    n, m = X.shape
    k = theta.shape[1]
    out = np.empty((n, k))
    P = np.empty((n, m)) if fwd_scheme != 0 else None
    _lib.orc_gcn_forward(n, op.rowptr, op.cols, op.vals, X, m, theta, bias, k, fwd_scheme,
                         out, _ptr(P))
    return out, P


def gcn_backward(op: Operator, d_out, saved, theta, bwd_scheme, fg):
    d_out, saved, theta = _f64(d_out), _f64(saved), _f64(theta)
    n, k = d_out.shape
    m = theta.shape[0]
    dth, db = np.empty((m, k)), np.empty(k)
    dx = np.empty((n, m)) if fg else None
    _lib.orc_gcn_backward(n, op.rowptr, op.cols, op.vals, op.colptr, op.crows, op.cvals,
                          d_out, saved, m, theta, k, bwd_scheme, int(fg), dth, db, _ptr(dx))
    return dth, db, dx


def gcn_layer(op: Operator, X, theta, bias, scheme, G=None, fg=False):
    """forward (+ backward when G is given) for a resolved (fwd, bwd, caching)."""
    fwd, bwd, _ = scheme
    out, P = gcn_forward(op, X, theta, bias, fwd)
    if G is None:
        return out
    saved = P if bwd == 2 else X
    return (out,) + gcn_backward(op, G, saved, theta, bwd, fg)


def gat_forward(pat: Operator, X, theta, a_src, a_dst, bias, heads, beta=0.2, want=False):
    X, theta = _f64(X), _f64(theta)
    n, m = X.shape
    hk = theta.shape[1]
    k = hk // heads
    q = pat.nnz
    out = np.empty((n, hk))
    M, s, d = np.empty((n, hk)), np.empty((n, heads)), np.empty((n, heads))
    alpha, mask = np.empty((heads, q)), np.empty((heads, q), np.uint8)
    rc = _lib.orc_gat_forward(n, pat.rowptr, pat.cols, X, m, theta, _f64(a_src), _f64(a_dst),
                              _f64(bias), heads, k, beta, out, _ptr(M), _ptr(s), _ptr(d),
                              _ptr(alpha), _ptr(mask))
    if rc != 0:
        raise ValueError("gat_forward: pattern must contain all self loops / beta > 0")
    if want:
        return out, {"M": M, "s": s, "d": d, "alpha": alpha, "mask": mask}
    return out


def gat_backward(pat: Operator, G, X, theta, a_src, a_dst, heads, beta=0.2, fg=False):
    G, X, theta = _f64(G), _f64(X), _f64(theta)
    n, m = X.shape
    hk = theta.shape[1]
    k = hk // heads
    dth, das, dad, db = np.empty((m, hk)), np.empty((heads, k)), np.empty((heads, k)), \
        np.empty(hk)
    dx = np.empty((n, m)) if fg else None
    _lib.orc_gat_backward(n, pat.rowptr, pat.cols, pat.colptr, pat.crows, pat.perm, G, X, m,
                          theta, _f64(a_src), _f64(a_dst), heads, k, beta, int(fg), dth, das,
                          dad, db, _ptr(dx))
    return dth, das, dad, db, dx


# ---- two-layer models (model.hpp:40-245) -----------------------------------
def gcn2_params(m, hidden, out, seed):
    """Gcn2Model(cfg, seed): layer 2 from seed+101 (model.hpp:46-49)."""
    return gcn_params(m, hidden, seed) + gcn_params(hidden, out, seed + 101)


def gat2_params(m, heads, hidden, out, seed):
    """Gat2Model(cfg, seed): layer 2 input heads*hidden, seed+201 (model.hpp:126-130)."""
    return gat_params(m, heads, hidden, seed) + gat_params(heads * hidden, heads, out, seed + 201)


def gcn2_step(op: Operator, X, params, target, policy=0, caching=False, input_grad=False):
    """Gcn2Model forward (model.hpp:52-69), loss_mse, backward (model.hpp:71-81).
    Returns (loss, out, [dth1, db1, dth2, db2], dX-or-None)."""
    th1, b1, th2, b2 = params
    m, hid = th1.shape
    k = th2.shape[1]
    s1 = resolve_scheme(policy, m, hid, input_grad, caching)
    s2 = resolve_scheme(policy, hid, k, True, caching)  # model.hpp:61-62
    o1, P1 = gcn_forward(op, X, th1, b1, s1[0])
    h, mask = activation(o1, "relu")
    out, P2 = gcn_forward(op, h, th2, b2, s2[0])
    loss, g = loss_mse(out, target)
    dth2, db2, dh = gcn_backward(op, g, P2 if s2[1] == 2 else h, th2, s2[1], True)
    dh = activation_backward(dh, mask, "relu")
    dth1, db1, dx = gcn_backward(op, dh, P1 if s1[1] == 2 else X, th1, s1[1], input_grad)
    return loss, out, [dth1, db1, dth2, db2], dx


def gat2_step(pat: Operator, X, params, heads, target, beta=0.2, input_grad=False):
    """Gat2Model forward (model.hpp:133-150), loss_mse, backward (model.hpp:152-163);
    the cache level does not change the values (gat.hpp:150-170)."""
    th1, as1, ad1, b1, th2, as2, ad2, b2 = params
    o1 = gat_forward(pat, X, th1, as1, ad1, b1, heads, beta)
    h, mask = activation(o1, "elu", 1.0)
    out = gat_forward(pat, h, th2, as2, ad2, b2, heads, beta)
    loss, g = loss_mse(out, target)
    g2 = gat_backward(pat, g, h, th2, as2, ad2, heads, beta, True)
    dh = activation_backward(g2[4], mask, "elu", 1.0, h)
    g1 = gat_backward(pat, dh, X, th1, as1, ad1, heads, beta, input_grad)
    return loss, out, list(g1[:4]) + list(g2[:4]), g1[4]
