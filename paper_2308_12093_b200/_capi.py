"""ctypes binding of the C-ABI in include/sgnn_cuda.h (libsgnn_cuda.so).

This is the binding a maintainer adds on the reference side (the reference
binds its C++ API with pybind11 in python/bindings.cpp).
The library is REQUIRED: there is no CPU fallback -- a missing or unloadable
library raises ImportError at import time.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SGNN_CUDA_LIB", os.path.join(_HERE, "libsgnn_cuda.so"))

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"libsgnn_cuda.so not found at {LIB_PATH}: build it with "
        "`python -c 'import __graft_entry__ as g; g.build()'` (make -C "
        "paper_2308_12093_b200/csrc). There is no CPU fallback.")

lib = C.CDLL(LIB_PATH)

SGNN_OK, SGNN_EINVAL, SGNN_ERUNTIME, SGNN_ECUDA, SGNN_ENCCL = 0, 1, 2, 3, 4
F32, F64 = 0, 1
FORMATS = {"coo": 0, "csr": 1, "csc": 2, "ellpack": 3, "hybrid": 4}
FWD_NAMES = ["transform_first", "propagate_first", "propagate_first_cached"]
BWD_NAMES = ["fused_propagate", "split_propagate", "split_propagate_cached"]
POLICIES = {"adaptive": 0, "transform-first": 1, "propagate-first": 2}
LEVELS = {"none": 0, "features": 1, "node-attn": 2, "full": 3}
GAT_REORDER = 1  # sgnn_gat_forward_ex flags (SGNN_GAT_REORDER)


class ModelConfig(C.Structure):
    """sgnn_model_config (model.hpp:18-29 ModelConfig)."""
    _fields_ = [("kind", C.c_int32), ("in_features", C.c_int32), ("hidden", C.c_int32),
                ("out_features", C.c_int32), ("heads", C.c_int32), ("scheme_policy", C.c_int32),
                ("caching", C.c_int32), ("gat_level", C.c_int32), ("leaky_slope", C.c_double),
                ("input_grad", C.c_int32)]


class Scheme(C.Structure):
    _fields_ = [("forward", C.c_int32), ("backward", C.c_int32), ("caching", C.c_int32)]

    def as_dict(self):
        return {"forward": FWD_NAMES[self.forward], "backward": BWD_NAMES[self.backward],
                "caching": bool(self.caching)}

    def __repr__(self):
        return f"Scheme({FWD_NAMES[self.forward]}, {BWD_NAMES[self.backward]}, {bool(self.caching)})"


VP, I32, I64, U64, D, INT = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double, C.c_int
PI64, PI32, PINT, PVP, PD = (C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_int),
                             C.POINTER(C.c_void_p), C.POINTER(C.c_double))

_SIGS = {
    "sgnn_last_error": (C.c_char_p, []),
    "sgnn_version": (C.c_char_p, []),
    "sgnn_ctx_create": (INT, [INT, VP, PVP]),
    "sgnn_ctx_destroy": (INT, [VP]),
    "sgnn_ctx_set_stream": (INT, [VP, VP]),
    "sgnn_ctx_synchronize": (INT, [VP]),
    "sgnn_ctx_launch_count": (INT, [VP, PI64]),
    "sgnn_gcn_select_scheme": (INT, [I64, I64, INT, INT, C.POINTER(Scheme)]),
    "sgnn_resolve_scheme": (INT, [INT, I64, I64, INT, INT, C.POINTER(Scheme)]),
    "sgnn_gcn_forward_flops": (I64, [INT, I64, I64, I64, I64]),
    "sgnn_gcn_backward_flops": (I64, [INT, I64, I64, I64, I64, INT]),
    "sgnn_gcn_forward_transients": (I64, [INT, I64, I64, I64]),
    "sgnn_gcn_backward_transients": (I64, [INT, I64, I64, I64, INT]),
    "sgnn_spmm_cost": (INT, [INT, I64, I64, I64, I64, I64, I64, PI64, PI64, PD]),
    "sgnn_sddmm_cost": (INT, [INT, I64, I64, I64, I64, I64, I64, PI64, PI64, PD]),
    "sgnn_gat_cache_footprint": (I64, [INT, I64, I64, I64, I64, I64]),
    "sgnn_synthetic_graph_edges": (I64, [I32, D]),
    "sgnn_synthetic_graph": (INT, [I32, D, U64, VP, VP]),
    "sgnn_random_uniform": (INT, [VP, I64, I64, U64, D, D, INT, VP]),
    "sgnn_gcn_params_init": (INT, [VP, I32, I32, U64, INT, VP, VP]),
    "sgnn_gat_params_init": (INT, [VP, I32, I32, I32, U64, INT, VP, VP, VP, VP]),
    "sgnn_coo_canonicalize": (INT, [VP, I32, I32, I64, VP, VP, VP, INT, VP, VP, VP, PI64]),
    "sgnn_csr_from_coo": (INT, [VP, I32, I64, VP, VP]),
    "sgnn_csc_from_coo": (INT, [VP, I32, I64, VP, VP, VP, INT, VP, VP, VP, VP]),
    "sgnn_add_self_loops": (INT, [VP, I32, I64, VP, VP, VP, INT, VP, VP, VP, PI64]),
    "sgnn_gcn_normalize": (INT, [VP, I32, I64, VP, VP, VP, INT, VP, VP, VP, PI64]),
    "sgnn_adj_create": (INT, [VP, I32, I32, I64, VP, VP, VP, INT, INT, PVP]),
    "sgnn_adj_destroy": (INT, [VP]),
    "sgnn_adj_info": (INT, [VP, PI32, PI32, PI64, PINT]),
    "sgnn_adj_arrays": (INT, [VP, PVP, PVP, PVP, PVP, PVP, PVP]),
    "sgnn_pattern_create": (INT, [VP, I32, I64, VP, VP, PVP]),
    "sgnn_pattern_destroy": (INT, [VP]),
    "sgnn_pattern_info": (INT, [VP, PI32, PI64, PINT]),
    "sgnn_pattern_arrays": (INT, [VP, PVP, PVP, PVP, PVP, PVP, PVP]),
    "sgnn_spmm": (INT, [VP, VP, INT, VP, I32, VP, VP]),
    "sgnn_sddmm": (INT, [VP, VP, VP, I32, VP, I32, INT, VP]),
    "sgnn_edge_softmax": (INT, [VP, VP, I32, VP, INT, VP]),
    "sgnn_gemm": (INT, [VP, INT, VP, I32, I32, VP, I32, I32, INT, INT, VP]),
    "sgnn_gemm_ex": (INT, [VP, INT, VP, I32, I32, VP, I32, I32, INT, INT, VP, VP, VP]),
    "sgnn_column_sums": (INT, [VP, INT, VP, I32, I32, VP]),
    "sgnn_gcn_forward": (INT, [VP, VP, VP, I32, VP, VP, I32, C.POINTER(Scheme), VP, PVP]),
    "sgnn_gcn_backward": (INT, [VP, VP, VP, VP, I32, I32, VP, INT, VP, VP, VP]),
    "sgnn_gcn_cache_destroy": (INT, [VP]),
    "sgnn_gcn_cache_retained_bytes": (INT, [VP, PI64]),
    "sgnn_gat_forward": (INT, [VP, VP, VP, I32, VP, VP, VP, VP, I32, I32, D, INT, INT, VP, PVP]),
    "sgnn_gat_backward": (INT, [VP, VP, VP, VP, VP, VP, I32, I32, I32, D, VP, INT, VP, VP, VP,
                                VP, VP]),
    "sgnn_gat_cache_destroy": (INT, [VP]),
    "sgnn_gat_cache_extra_bytes": (INT, [VP, PI64]),
    "sgnn_gat_cache_edge_values": (INT, [VP, VP, VP, VP, VP, VP, VP, VP]),
    "sgnn_gcn_step_host": (INT, [VP, VP, VP, I32, VP, VP, I32, C.POINTER(Scheme), VP, INT, VP, VP,
                                 VP, VP]),
    "sgnn_mem_stats": (INT, [INT, PI64, PI64, PI64]),
    "sgnn_gemm_act": (INT, [VP, INT, VP, I32, I32, VP, I32, I32, INT, INT, VP, VP, INT, VP, VP]),
    "sgnn_gcn_cache_arrays": (INT, [VP, PVP, PVP]),
    "sgnn_gat_cache_arrays": (INT, [VP, PVP, PVP, PVP, PVP, PVP]),
    "sgnn_gat_cache_reordered": (INT, [VP, C.POINTER(C.c_int)]),
    "sgnn_gat_forward_ex": (INT, [VP, VP, VP, I32, VP, VP, VP, VP, I32, I32, D, INT, INT, VP, PVP,
                                  INT]),
    "sgnn_mem_reset_peaks": (INT, []),
    "sgnn_gat_transform": (INT, [VP, VP, I32, I32, VP, I32, I32, VP, VP, VP, VP, VP]),
    "sgnn_rowplan_create": (INT, [VP, I32, VP, PVP]),
    "sgnn_rowplan_destroy": (INT, [VP]),
    "sgnn_gat_attention": (INT, [VP, I32, VP, VP, I32, VP, VP, D, VP, VP, VP]),
    "sgnn_gat_attention_ex": (INT, [VP, I32, VP, VP, I32, VP, VP, D, VP, VP, VP, VP]),
    "sgnn_gat_aggregate": (INT, [VP, I32, VP, VP, I32, I32, VP, VP, VP, VP, VP]),
    "sgnn_gat_sddmm": (INT, [VP, I32, VP, VP, I32, I32, VP, VP, VP, VP]),
    "sgnn_gat_softmax_backward": (INT, [VP, I32, VP, I32, VP, VP, VP, D, VP, VP, VP]),
    "sgnn_gat_softmax_backward_ex": (INT, [VP, I32, VP, I32, VP, VP, VP, D, VP, VP, VP, VP]),
    "sgnn_gat_column_stats_supported": (INT, [I32, I32]),
    "sgnn_gat_column_pass_stats": (INT, [VP, I32, VP, VP, I32, I32, VP, VP, VP, VP, D, VP, VP,
                                         VP, VP, VP, VP]),
    "sgnn_gat_column_pass": (INT, [VP, I32, VP, VP, VP, I32, I32, VP, VP, VP, VP, VP, VP, VP,
                                   VP, VP]),
    "sgnn_gat_param_grads": (INT, [VP, I32, I32, I32, VP, VP, VP, VP, VP, VP, VP]),
    "sgnn_powerlaw_graph_capacity": (I64, [I32, D]),
    "sgnn_powerlaw_graph": (INT, [VP, I32, D, D, U64, VP, VP, PI64]),
    "sgnn_activation": (INT, [VP, INT, INT, VP, I64, VP, VP]),
    "sgnn_activation_backward": (INT, [VP, INT, INT, VP, VP, VP, I64, VP]),
    "sgnn_loss_mse": (INT, [VP, INT, VP, VP, I64, I64, VP, VP]),
    "sgnn_model_create": (INT, [VP, C.POINTER(ModelConfig), U64, INT, PVP]),
    "sgnn_model_destroy": (INT, [VP]),
    "sgnn_model_num_params": (INT, [VP, PI32]),
    "sgnn_model_param": (INT, [VP, I32, PVP, PI64, C.POINTER(C.c_char_p)]),
    "sgnn_model_train_step": (INT, [VP, VP, VP, VP, VP, VP, VP, PVP, VP, VP]),
    "sgnn_gat_step_host": (INT, [VP, VP, VP, I32, VP, VP, VP, VP, I32, I32, D, INT, INT, VP, INT,
                                 VP, VP, VP, VP, VP, VP]),
}

for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args

SYMBOLS = tuple(_SIGS)


class SgnnError(RuntimeError):
    pass


def check(rc):
    """Map C-ABI status to the exceptions the reference's pybind11 module
    raises: std::invalid_argument -> ValueError, everything else RuntimeError."""
    if rc == SGNN_OK:
        return
    msg = (lib.sgnn_last_error() or b"").decode(errors="replace")
    if rc == SGNN_EINVAL:
        raise ValueError(msg)
    raise SgnnError(f"sgnn error {rc}: {msg}")


def version():
    return lib.sgnn_version().decode()
