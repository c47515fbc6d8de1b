"""Dev A/B timer: Arxiv GCN step (128->256, fg, adaptive + caching) and GAT
layer (h=8, k=32, level full, fg) forward / backward, eager, CUDA events, L2
flushed (256 MiB write) before each timed call; median of ITERS.  Run once per
variant (SGNN_CUDA_LIB / SGNN_* knobs) and compare:
  python scripts/dev/ab_step.py <tag>"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2308_12093_b200 import device as d  # noqa: E402

ITERS = int(os.environ.get("ITERS", "30"))
n = 169343
src, dst = d.synthetic_graph(n, 1166243 / n, 1)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn):
    for _ in range(3):
        fn()
    ms = []
    for _ in range(ITERS):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    return statistics.median(ms)


A = d.Adjacency.gcn_operator(n, src, dst, torch.float32, "csc")
X = d.random_uniform(n, 128, 12)
G = d.random_uniform(n, 256, 13)
th, b = d.gcn_params(128, 256, 14)
s = d.resolve_scheme("adaptive", 128, 256, True, True)


def gcn_step():
    out, c = d.gcn_forward(A, X, th, b, s)
    d.gcn_backward(A, G, th, c, True)


P = d.Pattern.gat_pattern(n, src, dst)
thg, a_s, a_d, bg = d.gat_params(128, 8, 32, 6)
Gg = d.random_uniform(n, 256, 7)
state = {}


def gat_fwd():
    state["o"], state["c"] = d.gat_forward(P, X, thg, a_s, a_d, bg, 8, 0.2, "full")


def gat_layer():  # a cache is consumed by its backward
    gat_fwd()
    d.gat_backward(P, Gg, thg, a_s, a_d, state["c"], True)


res = {"gcn_step": timed(gcn_step), "gat_fwd": timed(gat_fwd), "gat_layer": timed(gat_layer)}
res["gat_bwd"] = res["gat_layer"] - res["gat_fwd"]
print(sys.argv[1] if len(sys.argv) > 1 else "run", {k: round(v, 4) for k, v in res.items()})
