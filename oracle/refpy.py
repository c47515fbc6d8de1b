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
