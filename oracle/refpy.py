"""ctypes front of oracle/_ref/libsgnn_ref.so -- TEST INFRASTRUCTURE ONLY.

The library is the UNMODIFIED reference (headers under
/root/reference/proj/include) compiled in place by oracle/Makefile through
oracle/ref_shim.cpp.  Used by oracle/gen_golden.py (fixtures) and by bench.py's
reference arm / cpu_baseline (timing the reference's own OpenMP CPU path).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libsgnn_ref.so")

i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
VP = C.c_void_p
LL, D, INT, ULL = C.c_longlong, C.c_double, C.c_int, C.c_ulonglong


def available():
    return os.path.exists(LIB_PATH)


def load():
    lib = C.CDLL(LIB_PATH)
    sig = {
        "ref_last_error": (C.c_char_p, []),
        "ref_num_threads": (INT, []),
        "ref_set_num_threads": (None, [INT]),
        "ref_synthetic_graph": (LL, [INT, D, ULL, VP, VP]),
        "ref_random_uniform": (None, [INT, INT, ULL, D, D, f64p]),
        "ref_load_graph": (LL, [C.c_char_p, INT, C.POINTER(INT), VP, VP, VP]),
        "ref_bench_report_json": (LL, [C.c_char_p, INT, INT, INT, INT, INT, INT, INT, INT, INT,
                                       INT, INT, ULL, C.c_char_p, LL]),
        "ref_coo_canonicalize": (LL, [INT, INT, LL, i32p, i32p, f64p, i32p, i32p, f64p]),
        "ref_gcn_normalize": (LL, [INT, LL, i32p, i32p, f64p, i32p, i32p, f64p]),
        "ref_gcn_normalize_f32": (LL, [INT, LL, i32p, i32p, f32p, i32p, i32p, f32p]),
        "ref_csr_csc": (None, [INT, INT, LL, i32p, i32p, f64p, i32p, i32p, i32p, f64p]),
        "ref_pattern": (INT, [INT, i32p, i32p, i32p, i32p, i32p, i32p]),
        "ref_spmm": (INT, [INT, INT, INT, LL, i32p, i32p, f64p, f64p, INT, f64p]),
        "ref_spmm_f32": (INT, [INT, INT, INT, LL, i32p, i32p, f32p, f32p, INT, f32p]),
        "ref_sddmm": (LL, [INT, LL, i32p, i32p, f64p, INT, f64p, f64p]),
        "ref_edge_softmax": (INT, [INT, LL, i32p, i32p, f64p, f64p]),
        "ref_select_scheme": (INT, [INT, LL, LL, INT, INT, C.POINTER(INT), C.POINTER(INT),
                                    C.POINTER(INT)]),
        "ref_spmm_cost": (INT, [INT, LL, LL, LL, LL, LL, LL, C.POINTER(LL), C.POINTER(LL),
                                C.POINTER(D)]),
        "ref_sddmm_cost": (INT, [INT, LL, LL, LL, LL, LL, LL, C.POINTER(LL), C.POINTER(LL),
                                 C.POINTER(D)]),
        "ref_gcn_params": (None, [INT, INT, ULL, f64p, f64p]),
        "ref_gat_params": (None, [INT, INT, INT, ULL, f64p, f64p, f64p, f64p]),
        "ref_gcn_layer": (INT, [INT, LL, i32p, i32p, f64p, INT, f64p, INT, f64p, f64p, INT,
                                INT, INT, INT, VP, INT, f64p, VP, VP, VP]),
        "ref_gat_layer": (INT, [INT, i32p, i32p, f64p, INT, f64p, f64p, f64p, f64p, INT, INT,
                                D, INT, VP, INT, f64p, VP, VP, VP, VP, VP, VP, VP]),
        "ref_model_step": (INT, [INT, INT, D, ULL, INT, INT, INT, INT, INT, INT, INT, INT,
                                 C.POINTER(D), f64p, f64p]),
        "ref_bench_create": (VP, [INT, INT, D, ULL, INT, INT, INT, INT, INT, INT, INT, INT]),
        "ref_bench_nnz": (LL, [VP]),
        "ref_bench_step": (D, [VP]),
        "ref_bench_destroy": (None, [VP]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


# ---------------------------------------------------------------------------
# float64 layer / model runs of the reference at full size (parity checker of
# tests/test_gpu_fullsize.py and of bench.py's `parity` field).  Inputs are
# float32-representable arrays widened exactly (SURVEY 8(c) golden policy).
# ---------------------------------------------------------------------------
_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        if not available():
            raise RuntimeError(f"{LIB_PATH} missing: build() compiles it in the dev container")
        _LIB = load()
    return _LIB


def _f64c(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def gcn_normalize(n, src, dst):
    """adjacency(graph) -> gcn_normalize (sparse.hpp:474-495), float64 COO."""
    L = lib()
    src, dst = np.ascontiguousarray(src, np.int32), np.ascontiguousarray(dst, np.int32)
    q = src.size
    ro = np.empty(q + n, np.int32)
    co = np.empty(q + n, np.int32)
    vo = np.empty(q + n, np.float64)
    w = L.ref_gcn_normalize(n, q, src, dst, np.ones(q), ro, co, vo)
    if w < 0:
        raise RuntimeError(L.ref_last_error().decode())
    return ro[:w], co[:w], vo[:w]


def gcn_layer(n, coo, fmt, X, theta, bias, scheme, G, fg):
    """gcn_forward + gcn_backward (gcn.hpp:91-193) in float64 over the
    canonical normalized COO `coo` stored in format `fmt` (0 coo .. 4 hybrid).
    Returns (out, d_theta, d_bias, d_input or None)."""
    L = lib()
    r, c, v = coo
    X, theta, bias, G = (_f64c(a) for a in (X, theta, bias, G))
    m, k = theta.shape
    out = np.empty((n, k))
    dth = np.empty((m, k))
    db = np.empty(k)
    dx = np.empty((n, m)) if fg else None
    fw, bw, ca = scheme
    rc = L.ref_gcn_layer(n, r.size, r, c, _f64c(v), fmt, X, m, theta, bias, k, int(fw), int(bw),
                         int(ca), G.ctypes.data, int(bool(fg)), out, dth.ctypes.data, db.ctypes.data,
                         dx.ctypes.data if fg else None)
    if rc != 0:
        raise RuntimeError(L.ref_last_error().decode())
    return out, dth, db, dx


def gat_layer(n, rowptr, cols, X, theta, a_src, a_dst, bias, heads, level, G, fg, beta=0.2):
    """gat_forward + gat_backward (gat.hpp:89-219) in float64 on the CSR pattern.
    Returns (out, d_theta, d_a_src, d_a_dst, d_bias, d_input or None)."""
    L = lib()
    rowptr, cols = np.ascontiguousarray(rowptr, np.int32), np.ascontiguousarray(cols, np.int32)
    X, theta, a_src, a_dst, bias, G = (_f64c(a) for a in (X, theta, a_src, a_dst, bias, G))
    m, hk = theta.shape
    k = hk // heads
    out = np.empty((n, hk))
    dth = np.empty((m, hk))
    das = np.empty((heads, k))
    dad = np.empty((heads, k))
    db = np.empty(hk)
    dx = np.empty((n, m)) if fg else None
    rc = L.ref_gat_layer(n, rowptr, cols, X, m, theta, a_src, a_dst, bias, heads, k, beta,
                         int(level), G.ctypes.data, int(bool(fg)), out, None, None, dth.ctypes.data,
                         das.ctypes.data, dad.ctypes.data, db.ctypes.data,
                         dx.ctypes.data if fg else None)
    if rc != 0:
        raise RuntimeError(L.ref_last_error().decode())
    return out, dth, das, dad, db, dx


def model_step(kind, n, deg, seed, m, hidden, out_f, heads=1, policy=0, caching=False,
               level=0, input_grad=False):
    """One Gcn2Model (kind 0) / Gat2Model (kind 1) training step in float64 on
    the run_benchmark_typed workload (bench.hpp:160-219).  Returns (loss,
    prediction, flat gradients in param_tensors() order)."""
    L = lib()
    ow = out_f if kind == 0 else heads * out_f
    if kind == 0:
        npar = m * hidden + hidden + hidden * out_f + out_f
    else:
        hh = heads * hidden
        npar = (m * hh + 2 * hh + hh) + (hh * heads * out_f + 2 * heads * out_f + heads * out_f)
    loss = C.c_double()
    pred = np.empty((n, ow))
    grads = np.empty(npar)
    rc = L.ref_model_step(kind, n, deg, seed, m, hidden, out_f, heads, policy, int(caching),
                          level, int(input_grad), C.byref(loss), pred, grads)
    if rc != 0:
        raise RuntimeError(L.ref_last_error().decode())
    return loss.value, pred, grads
