"""Dev probe: the GCN layer step replayed from a CUDA graph vs eager launches."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2308_12093_b200 import device as d

n = 169343
ctx = d.Context.default(0)
src, dst = d.synthetic_graph(n, 1166243 / n, 1)
A = d.Adjacency.gcn_operator(n, src, dst, torch.float32, "csc", ctx)
X = d.random_uniform(n, 128, 12, ctx=ctx)
G = d.random_uniform(n, 256, 13, ctx=ctx)
th, b = d.gcn_params(128, 256, 14, ctx=ctx)
sch = d.resolve_scheme("adaptive", 128, 256, True, True)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

def step():
    out, c = d.gcn_forward(A, X, th, b, sch)
    return (out,) + d.gcn_backward(A, G, th, c, True)

def timed(fn, it=20):
    for _ in range(3): fn()
    ms = []
    for _ in range(it):
        flush.fill_(1); flush.view(torch.int64).sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ms.append(e0.elapsed_time(e1))
    return statistics.median(ms) * 1e3

eager = timed(step)
ref = step()
torch.cuda.synchronize()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
ctx.set_stream(s)
with torch.cuda.stream(s):
    step()  # warm on the capture stream
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        res = step()
ctx.set_stream(torch.cuda.current_stream())
torch.cuda.synchronize()
graph = timed(g.replay)
g.replay(); torch.cuda.synchronize()
same = all(torch.equal(a, b) for a, b in zip(res, ref))
print(f"eager {eager:.1f} us  graph {graph:.1f} us  identical={same}")
