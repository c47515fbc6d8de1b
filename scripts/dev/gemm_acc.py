"""Dev: accuracy of the long-K tcgen05 GEMM (dTheta = P^T G, K = n = 169,343)
against float64, as a function of the split-K chunk (SGNN_GEMM_KCHUNK)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2308_12093_b200 import device as d  # noqa: E402

n = int(os.environ.get("N", "169343"))
P = d.random_uniform(n, 128, 21) * 0.3
G = d.random_uniform(n, 256, 12)
C = d.gemm(P, G, True, False)
ref = P.double().t() @ G.double()
c64 = C.double()
den = torch.maximum(torch.ones_like(ref), torch.maximum(ref.abs(), c64.abs()))
err = ((c64 - ref).abs() / den).max().item()
bias = ((c64 - ref) * ref.sign()).mean().item()
f32 = (P.t() @ G).double()  # cuBLAS fp32 (TF32 off by default)
e32 = ((f32 - ref).abs() / den).max().item()
print(f"kchunk={os.environ.get('SGNN_GEMM_KCHUNK', 'default')} max_rel_diff={err:.3e} "
      f"signed-bias={bias:.3e} |ref|max={ref.abs().max().item():.1f} cublas_fp32={e32:.3e}")
