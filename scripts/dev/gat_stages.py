"""Dev: per-stage float32 error of the GAT backward kernels, each stage fed the
device's own inputs and compared with float64 evaluated on those same inputs."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2308_12093_b200 import _capi as capi  # noqa: E402
from paper_2308_12093_b200 import device as d  # noqa: E402

n, deg, h, k, m = 89250, 899756 / 89250, 8, int(os.environ.get("K", "64")), 500
ctx = d.Context.default(0)
src, dst = d.synthetic_graph(n, deg, 1)
P = d.Pattern.gat_pattern(n, src, dst)
pa = P.arrays()
q = P.nnz
X = d.random_uniform(n, m, 12)
G = d.random_uniform(n, h * k, 13)
th, a_s, a_d, b = d.gat_params(m, h, k, 14)
dev = X.device
f = lambda *s: torch.empty(s, dtype=torch.float32, device=dev)  # noqa: E731
p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
h64 = lambda t: t.double().cpu().numpy()  # noqa: E731
L = capi.lib
M, s, dd = f(n, h * k), f(n, h), f(n, h)
capi.check(L.sgnn_gat_transform(ctx.handle, p(X), n, m, p(th), h, k, p(a_s), p(a_d), p(M), p(s), p(dd)))
alpha = f(q, h)
mask = torch.empty((q, h), dtype=torch.uint8, device=dev)
capi.check(L.sgnn_gat_attention(ctx.handle, n, p(pa["rowptr"]), p(pa["cols"]), h, p(s), p(dd),
                                C.c_double(0.2), p(alpha), p(mask), None))
da = f(q, h)
capi.check(L.sgnn_gat_sddmm(ctx.handle, n, p(pa["rowptr"]), p(pa["cols"]), h, k, p(M), p(G), p(da), None))
dy, dS = f(q, h), f(n, h)
capi.check(L.sgnn_gat_softmax_backward(ctx.handle, n, p(pa["rowptr"]), h, p(alpha), p(mask), p(da),
                                       C.c_double(0.2), p(dy), p(dS), None))
dD, dM = f(n, h), f(n, h * k)
capi.check(L.sgnn_gat_column_pass(ctx.handle, n, p(pa["colptr"]), p(pa["rows"]), p(pa["perm"]), h, k,
                                  p(G), p(alpha), p(dy), p(dS), p(a_s), p(a_d), p(dD), p(dM), None))
torch.cuda.synchronize()
rp, cl = pa["rowptr"].cpu().numpy().astype(np.int64), pa["cols"].cpu().numpy().astype(np.int64)
cp, cr, pm = (pa[x].cpu().numpy().astype(np.int64) for x in ("colptr", "rows", "perm"))
rows = np.repeat(np.arange(n), np.diff(rp))


def rep(name, got, want):
    g = h64(got).reshape(want.shape)
    err = np.abs(g - want)
    den = np.maximum(1.0, np.maximum(np.abs(g), np.abs(want)))
    print(f"{name:10s} max_rel_diff {(err / den).max():.3e}  max abs err {err.max():.3e}  "
          f"max|want| {np.abs(want).max():.3e}  rel-to-max {err.max() / np.abs(want).max():.3e}")


Md = h64(M)
M3 = Md.reshape(n, h, k)
rep("M", M, h64(X) @ h64(th))
rep("s", s, np.einsum("nhk,hk->nh", M3, h64(a_s)))
rep("d", dd, np.einsum("nhk,hk->nh", M3, h64(a_d)))
sd, ddd = h64(s), h64(dd)
y = sd[rows] + ddd[cl]
mk = h64(mask).astype(bool)
print("mask flips vs f64 of device scores:", int((mk != (y > 0)).sum()))
w = np.where(mk, y, 0.2 * y)
wmax = np.maximum.reduceat(w, rp[:-1], axis=0)
ex = np.exp(w - wmax[rows])
al = ex / np.add.reduceat(ex, rp[:-1], axis=0)[rows]
rep("alpha", alpha, al)
G3 = h64(G).reshape(n, h, k)
da64 = np.concatenate([np.einsum("qhk,qhk->qh", G3[rows[i:i + 200000]], M3[cl[i:i + 200000]])
                       for i in range(0, q, 200000)])
rep("d_alpha", da, da64)
A, DA = h64(alpha), h64(da)
dot = np.add.reduceat(A * DA, rp[:-1], axis=0)
dw = A * (DA - dot[rows])
dy64 = np.where(mk, dw, 0.2 * dw)
rep("dy", dy, dy64)
rep("dS", dS, np.add.reduceat(h64(dy), rp[:-1], axis=0))
rep("dS(f64)", dS, np.add.reduceat(dy64, rp[:-1], axis=0))
DY = h64(dy)
dD64 = np.stack([np.bincount(cl, weights=DY[:, t], minlength=n) for t in range(h)], 1)
rep("dD", dD, dD64)
