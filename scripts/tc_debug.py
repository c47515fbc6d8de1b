"""Dev probe for the tcgen05 GEMM: small structured inputs, prints diffs per layout."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2308_12093_b200 import device as d

torch.manual_seed(0)

BNS = ["default"]
for bn in BNS:

  print('BN', bn)
  for (M, K, N) in [(128, 64, 128)]:
    for ta, tb in [(False, False)]:
        A = torch.randn(M, K, device="cuda") if not ta else torch.randn(K, M, device="cuda")
        B = torch.randn(N, K, device="cuda") if tb else torch.randn(K, N, device="cuda")
        ref = (A.T if ta else A).double() @ (B.T if tb else B).double()
        got = d.gemm(A, B, ta, tb)
        torch.cuda.synchronize()
        err = (got.double() - ref).abs().max().item()
        nz = (got != 0).float().mean().item()
        print(f"M={M} K={K} N={N} ta={ta} tb={tb}: maxerr={err:.3e} nonzero_frac={nz:.3f} "
              f"got00={got[0,0].item():.4f} ref00={ref[0,0].item():.4f} got[1,0]={got[1,0].item():.4f} ref10={ref[1,0].item():.4f}", flush=True)
