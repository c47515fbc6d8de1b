"""sgnn-b200: B200-native (sm_100a) cached operator-reordering GCN and GAT
layers (arXiv 2308.12093), a drop-in for the reference `sgnn` layer API.

  paper_2308_12093_b200.sgnn    -- the reference Python module's API (numpy, float64)
  paper_2308_12093_b200.device  -- device-resident API (torch tensors) mirroring
                                   the reference C++ layer API
  include/sgnn_cuda.h           -- the C-ABI (libsgnn_cuda.so)

All computation runs in libsgnn_cuda.so; importing fails loudly when it is
missing (no CPU fallback).
"""
from . import _capi  # noqa: F401  (loads libsgnn_cuda.so or raises ImportError)

__version__ = "0.1.0"
