"""Dev: the GAT primitives bench.py times standalone (the reference's
sddmm_semibatched and column pass through the C-ABI, h=8, k=32, Arxiv
pattern), three launches each -- for the ncu capture of their DRAM traffic
(scripts/profile.sh -> profiles/traffic.json)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2308_12093_b200 import _capi as capi  # noqa: E402
from paper_2308_12093_b200 import device as d  # noqa: E402

n, H, K = 169343, 8, 32
ctx = d.Context.default(0)
src, dst = d.synthetic_graph(n, 1166243 / n, 1)
P = d.Pattern.gat_pattern(n, src, dst)
pa = P.arrays()
dev = torch.device("cuda")
M = d.random_uniform(n, H * K, 21)
G = d.random_uniform(n, H * K, 22)
_, a_s, a_d, _ = d.gat_params(128, H, K, 6)
da = torch.empty((P.nnz, H), dtype=torch.float32, device=dev)
al = torch.rand((P.nnz, H), dtype=torch.float32, device=dev) * 0.2
dy = torch.randn((P.nnz, H), dtype=torch.float32, device=dev) * 0.1
dS = torch.randn((n, H), dtype=torch.float32, device=dev)
dD = torch.empty((n, H), dtype=torch.float32, device=dev)
dM = torch.empty((n, H * K), dtype=torch.float32, device=dev)
vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
for _ in range(3):
    capi.check(capi.lib.sgnn_gat_sddmm(ctx.handle, n, vp(pa["rowptr"]), vp(pa["cols"]), H, K,
                                       vp(M), vp(G), vp(da), None))
    capi.check(capi.lib.sgnn_gat_column_pass(
        ctx.handle, n, vp(pa["colptr"]), vp(pa["rows"]), vp(pa["perm"]), H, K, vp(G), vp(al),
        vp(dy), vp(dS), vp(a_s), vp(a_d), vp(dD), vp(dM), None))
torch.cuda.synchronize()
