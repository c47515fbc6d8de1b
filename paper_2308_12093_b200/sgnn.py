"""Drop-in for the reference Python module ``sgnn`` (python/sgnn/__init__.py,
python/bindings.cpp:81-289): the same 14 functions with the same names,
argument meaning, numpy float64 / int32 I/O and error behaviour
(std::invalid_argument -> ValueError), computed on the B200 through
libsgnn_cuda.so.  ``import paper_2308_12093_b200.sgnn as sgnn``.

Extensions beyond the reference bindings (which bind no backward pass):
``gcn_layer`` and ``gat_layer`` return the forward output and all gradients.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _capi as _c
from . import device as _d
from ._capi import check, lib

__all__ = [
    "edge_softmax", "gat_cache_footprint", "gat_forward", "gcn_forward", "gcn_normalize",
    "gcn_select_scheme", "load_graph", "num_threads", "sddmm", "sddmm_cost", "set_num_threads",
    "spmm", "spmm_cost", "synthetic_graph", "gcn_layer", "gat_layer",
]

_threads = [None]


def _dev():
    return _d.Context.default().device


def _f64(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return torch.from_numpy(a).to(_dev())


def _mat(a):
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError("expected a 2-d array")
    return _f64(a)


def _i32(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(_dev())


def _np(t):
    return t.detach().cpu().numpy()


def _coo(n_rows, n_cols, rows, cols, vals):
    """bindings.cpp:44-52 to_coo_matrix: length check, canonicalize on entry."""
    rows = np.asarray(rows)
    cols = np.asarray(cols)
    vals = np.asarray(vals, dtype=np.float64)
    if rows.size != cols.size or rows.size != vals.size:
        raise ValueError("rows/cols/vals must have equal length")
    return _d.canonicalize(n_rows, n_cols, _i32(rows.ravel()), _i32(cols.ravel()),
                           _f64(vals.ravel()))


def _format(name):
    if name not in _c.FORMATS:
        raise ValueError(f"unknown format '{name}'")
    return name


def synthetic_graph(n, avg_degree, seed):
    """Seeded undirected simple graph; returns (n, src, dst)."""
    src, dst = _d.synthetic_graph(int(n), float(avg_degree), int(seed))
    return int(n), src.numpy(), dst.numpy()


def load_graph(path, format="edge-list"):
    """graph.hpp:62-147 loaders (host file parsing; dedup keeps the last weight)."""
    from ._graph_io import load_graph as _lg

    return _lg(path, format)


def gcn_normalize(n, rows, cols, vals):
    """Symmetric degree normalization of A + I; returns COO triplets."""
    r, c, v = _coo(n, n, rows, cols, vals)
    r, c, v = _d.gcn_normalize(n, r, c, v)
    return _np(r), _np(c), _np(v)


def spmm(n_rows, n_cols, rows, cols, vals, B, format="csr"):
    """Sparse times dense through the chosen storage format."""
    _format(format)
    Bt = _mat(B)
    r, c, v = _coo(n_rows, n_cols, rows, cols, vals)
    if Bt.shape[0] != n_cols:
        raise ValueError("spmm: dimension mismatch")
    adj = _d.Adjacency(n_rows, n_cols, r, c, v, format)
    return _np(adj.spmm(Bt))


def _pattern(n, rows, cols):
    r, c, _ = _coo(n, n, rows, cols, np.ones(np.asarray(rows).size))
    return _d.Pattern(n, _d.csr_from_coo(n, r), c), r, c


def sddmm(n, rows, cols, B, C):
    """Dense product sampled at the pattern positions; returns COO triplets."""
    Bt, Ct = _mat(B), _mat(C)
    pat, r, c = _pattern(n, rows, cols)
    out = _d.sddmm(pat, Bt, Ct)
    return _np(r), _np(c), _np(out)


def edge_softmax(n, rows, cols, scores):
    """Row-group softmax over a self-loop pattern given canonical-order scores."""
    pat, _, _ = _pattern(n, rows, cols)
    s = np.asarray(scores, dtype=np.float64).ravel()
    if s.size != pat.nnz:
        raise ValueError("scores length must equal the deduplicated nnz")
    return _np(_d.edge_softmax(pat, _f64(s)))


def _cost(fn, format, n, q, p, f, scalar_bytes, index_bytes):
    _format(format)
    fl, by, oi = _c.C.c_int64(), _c.C.c_int64(), _c.C.c_double()
    check(fn(_c.FORMATS[format], n, q, p, f, scalar_bytes, index_bytes, _c.C.byref(fl),
             _c.C.byref(by), _c.C.byref(oi)))
    return {"flops": fl.value, "bytes": by.value, "operational_intensity": oi.value}


def spmm_cost(format, n, q, p=0, f=64, scalar_bytes=4, index_bytes=4):
    return _cost(lib.sgnn_spmm_cost, format, n, q, p, f, scalar_bytes, index_bytes)


def sddmm_cost(format, n, q, p=0, f=64, scalar_bytes=4, index_bytes=4):
    return _cost(lib.sgnn_sddmm_cost, format, n, q, p, f, scalar_bytes, index_bytes)


def gcn_select_scheme(m, k, needs_feature_grad=False, caching=False):
    return _d.resolve_scheme("adaptive", m, k, needs_feature_grad, caching).as_dict()


def gat_cache_footprint(level, n, h, k, q, scalar_bytes=4):
    if level not in _c.LEVELS:
        raise ValueError(f"unknown caching level '{level}'")
    return lib.sgnn_gat_cache_footprint(_c.LEVELS[level], n, h, k, q, scalar_bytes)


def gcn_forward(n, rows, cols, vals, X, theta, bias, format="csc", scheme="adaptive"):
    """Single GCN layer forward over an already-normalized adjacency."""
    _format(format)
    Xt, th = _mat(X), _mat(theta)
    b = _f64(np.asarray(bias, dtype=np.float64).ravel())
    r, c, v = _coo(n, n, rows, cols, vals)
    adj = _d.Adjacency(n, n, r, c, v, format)
    choice = _d.resolve_scheme(scheme, th.shape[0], th.shape[1], False, False)
    out, _ = _d.gcn_forward(adj, Xt, th, b, choice)
    return _np(out)


def gat_forward(n, rows, cols, X, theta, a_src, a_dst, bias, heads=1, beta=0.2):
    """Single multi-head GAT layer forward; self loops are added to the pattern."""
    Xt, th, a_s, a_d = _mat(X), _mat(theta), _mat(a_src), _mat(a_dst)
    b = _f64(np.asarray(bias, dtype=np.float64).ravel())
    r, c, v = _coo(n, n, rows, cols, np.ones(np.asarray(rows).size))
    r, c, v = _d.add_self_loops(n, r, c, v)
    pat = _d.Pattern(n, _d.csr_from_coo(n, r), c)
    out, _ = _d.gat_forward(pat, Xt, th, a_s, a_d, b, heads, beta, "none")
    return _np(out)


def gcn_layer(n, rows, cols, vals, X, theta, bias, d_out, format="csc", scheme="adaptive",
              caching=False, needs_feature_grad=True):
    """Extension: forward + backward of one GCN layer (gcn.hpp:91-193)."""
    _format(format)
    Xt, th, G = _mat(X), _mat(theta), _mat(d_out)
    b = _f64(np.asarray(bias, dtype=np.float64).ravel())
    r, c, v = _coo(n, n, rows, cols, vals)
    adj = _d.Adjacency(n, n, r, c, v, format)
    choice = _d.resolve_scheme(scheme, th.shape[0], th.shape[1], needs_feature_grad, caching)
    out, cache = _d.gcn_forward(adj, Xt, th, b, choice)
    dth, db, dx = _d.gcn_backward(adj, G, th, cache, needs_feature_grad)
    return {"output": _np(out), "d_theta": _np(dth), "d_bias": _np(db),
            "d_input": None if dx is None else _np(dx), "scheme": choice.as_dict()}


def gat_layer(n, rows, cols, X, theta, a_src, a_dst, bias, d_out, heads=1, beta=0.2,
              level="none", needs_feature_grad=True):
    """Extension: forward + backward of one GAT layer (gat.hpp:89-219)."""
    Xt, th, a_s, a_d, G = _mat(X), _mat(theta), _mat(a_src), _mat(a_dst), _mat(d_out)
    b = _f64(np.asarray(bias, dtype=np.float64).ravel())
    r, c, v = _coo(n, n, rows, cols, np.ones(np.asarray(rows).size))
    r, c, v = _d.add_self_loops(n, r, c, v)
    pat = _d.Pattern(n, _d.csr_from_coo(n, r), c)
    out, cache = _d.gat_forward(pat, Xt, th, a_s, a_d, b, heads, beta, level)
    dth, das, dad, db, dx = _d.gat_backward(pat, G, th, a_s, a_d, cache, needs_feature_grad,
                                            beta)
    return {"output": _np(out), "d_theta": _np(dth), "d_a_src": _np(das), "d_a_dst": _np(dad),
            "d_bias": _np(db), "d_input": None if dx is None else _np(dx)}


def num_threads():
    """Host threads the reference would use; the device path uses every SM."""
    if _threads[0] is None:
        return torch.cuda.get_device_properties(_dev()).multi_processor_count
    return _threads[0]


def set_num_threads(n):
    _threads[0] = 1 if n < 1 else int(n)
