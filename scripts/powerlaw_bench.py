"""GCN / GAT layer fwd+bwd on Arxiv-sized graphs: the reference's uniform
generator vs the device power-law generator (hub rows)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2308_12093_b200 import device as d
n, deg = 169343, 1166243 / 169343
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def timed(fn, it=10):
    for _ in range(3): fn()
    ms = []
    for _ in range(it):
        flush.fill_(1); flush.view(torch.int64).sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ms.append(a.elapsed_time(b))
    return statistics.median(ms)
X = d.random_uniform(n, 128, 12); G = d.random_uniform(n, 256, 13)
th, b = d.gcn_params(128, 256, 14); tg, a_s, a_d, bg = d.gat_params(128, 8, 32, 15)
for name, gen in (("uniform", lambda: d.synthetic_graph(n, deg, 1)),
                  ("powerlaw g=3.0", lambda: d.powerlaw_graph(n, deg, 3.0, 1)),
                  ("powerlaw g=2.5", lambda: d.powerlaw_graph(n, deg, 2.5, 1)),
                  ("powerlaw g=2.2", lambda: d.powerlaw_graph(n, deg, 2.2, 1))):
    s, t = gen()
    A = d.Adjacency.gcn_operator(n, s, t, torch.float32, "csc")
    P = d.Pattern.gat_pattern(n, s, t)
    maxdeg = int(torch.bincount(s.cuda().long(), minlength=n).max())
    sch = d.resolve_scheme("adaptive", 128, 256, True, True)
    def gcn():
        o, c = d.gcn_forward(A, X, th, b, sch); d.gcn_backward(A, G, th, c, True)
    def gat():
        o, c = d.gat_forward(P, X, tg, a_s, a_d, bg, 8, 0.2, "full"); d.gat_backward(P, G, tg, a_s, a_d, c, True)
    print(f"{name:16s} nnz={A.nnz} maxdeg={maxdeg}: gcn {timed(gcn):.3f} ms  gat {timed(gat):.3f} ms", flush=True)
