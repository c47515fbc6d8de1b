"""Dev microbenchmark: time individual library kernels on Arxiv shapes (CUDA events,
L2 flushed between iterations)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2308_12093_b200 import device as d

n, m, k = 169343, 128, 256
dev = torch.device("cuda")
torch.manual_seed(0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
X = torch.randn(n, m, device=dev)
G = torch.randn(n, k, device=dev)
th = torch.randn(m, k, device=dev)
out = torch.empty(n, k, device=dev)
outm = torch.empty(n, m, device=dev)

FLUSH = os.environ.get("FLUSH", "write")
def do_flush():
    flush.fill_(1)
    if FLUSH == "readback":
        flush.view(torch.int64).sum()  # leave L2 holding clean lines

def t(fn, iters=20):
    for _ in range(3): fn()
    ms = []
    for _ in range(iters):
        do_flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
    return statistics.median(ms) * 1e3

which = sys.argv[1:] or ["nn", "tn", "nt", "colsum"]
if any(w.startswith("spmm") or w.startswith("gat") for w in which):
    src, dst = d.synthetic_graph(n, 1166243 / n, 1)
    A = d.Adjacency.gcn_operator(n, src, dst, torch.float32, "csc")
for w in which:
    if w == "nn":
        us = t(lambda: d.gemm(X, th)); byt = 4 * (n * m + n * k)
    elif w == "tn":
        us = t(lambda: d.gemm(X, G, True, False)); byt = 4 * (n * m + n * k)
    elif w == "nt":
        us = t(lambda: d.gemm(G, th, False, True)); byt = 4 * (n * m + n * k)
    elif w == "colsum":
        us = t(lambda: d.column_sums(G)); byt = 4 * n * k
    elif w == "spmm":
        us = t(lambda: A.spmm(X, out=outm)); byt = 4 * (n + 1) + 8 * A.nnz + 8 * n * m
    elif w == "spmmT":
        us = t(lambda: A.spmm(X, transposed=True, out=outm)); byt = 4 * (n + 1) + 8 * A.nnz + 8 * n * m
    elif w == "spmm256":
        us = t(lambda: A.spmm(G, out=out)); byt = 4 * (n + 1) + 8 * A.nnz + 8 * n * k
    elif w in ("gat", "gatfwd"):
        if "P" not in globals():
            P = d.Pattern.gat_pattern(n, src, dst)
            thg, asg, adg, bg = d.gat_params(m, 8, 32, 14)
            Gg = torch.randn(n, 256, device=dev)
        def gstep(bwd=(w == "gat")):
            o, c = d.gat_forward(P, X, thg, asg, adg, bg, 8, 0.2, "full")
            if bwd:
                d.gat_backward(P, Gg, thg, asg, adg, c, True)
        us = t(gstep); byt = 0
    elif w == "hash":  # bitwise fingerprint of the SpMM outputs (compare across modes)
        A.spmm(X, out=outm); A.spmm(G, out=out); o3 = torch.empty_like(outm); A.spmm(X, transposed=True, out=o3)
        torch.cuda.synchronize()
        hs = [int(t.view(torch.int32).to(torch.int64).mul(torch.arange(t.numel(), device=dev).view(t.shape) % 1000003 + 1).sum()) for t in (outm, out, o3)]
        print("hash", hs, flush=True); continue
    elif w.startswith("xform"):  # M = X Theta with the node scores fused: xform32 / xform40
        from paper_2308_12093_b200 import _capi as capi
        kk = int(w[5:] or 32); mi = 128 if kk == 32 else 256
        Xi = torch.randn(n, mi, device=dev); thi = torch.randn(mi, 8 * kk, device=dev)
        a_s = torch.randn(8 * kk, device=dev); a_d = torch.randn(8 * kk, device=dev)
        Mo = torch.empty(n, 8 * kk, device=dev); so = torch.empty(n, 8, device=dev); do_ = torch.empty(n, 8, device=dev)
        ctx = d.Context.default()
        us = t(lambda: capi.check(capi.lib.sgnn_gat_transform(ctx.handle, Xi.data_ptr(), n, mi, thi.data_ptr(), 8, kk,
               a_s.data_ptr(), a_d.data_ptr(), Mo.data_ptr(), so.data_ptr(), do_.data_ptr())))
        byt = 4 * (n * mi + n * 8 * kk)
    elif w in ("l2nn", "l2tn", "l2nt"):  # Gat2 layer 2: n x 256 <-> n x 320
        H1 = torch.randn(n, 256, device=dev); Z = torch.randn(n, 320, device=dev); th2 = torch.randn(256, 320, device=dev)
        f = {"l2nn": lambda: d.gemm(H1, th2), "l2tn": lambda: d.gemm(H1, Z, True, False),
             "l2nt": lambda: d.gemm(Z, th2, False, True)}[w]
        us = t(f); byt = 4 * (n * 256 + n * 320)
    elif w == "copy":
        us = t(lambda: out.copy_(G)); byt = 8 * n * k
    print(f"{w}: {us:.1f} us  {byt / us / 1e3:.0f} GB/s", flush=True)
    if os.environ.get("ONE"):
        break
