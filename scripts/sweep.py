"""Configs 2 and 3 of BASELINE.json, measured on one B200 (device time, CUDA
events, L2 flushed + read back before each step, median of --steps):

  config 2: one GCN layer fwd+bwd on the Arxiv-shaped graph, 128 -> k for
            k in 8..1024, needs_feature_grad in {0, 1}, the adaptive scheme
            (with caching) against both forced schemes;
  config 3: one GAT layer fwd+bwd (8 heads, 500 -> 8 x k) on PubMed- and
            Flickr-shaped graphs for k in 8..128 and every cache level.

Prints one JSON object (kept under profiles/)."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2308_12093_b200 import device as d  # noqa: E402

STEPS = int(os.environ.get("STEPS", "10"))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn):
    for _ in range(3):
        fn()
    ms = []
    for _ in range(STEPS):
        flush.fill_(1)
        flush.view(torch.int64).sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    return round(statistics.median(ms), 4)


def config2():
    n, m = 169343, 128
    src, dst = d.synthetic_graph(n, 1166243 / n, 1)
    A = d.Adjacency.gcn_operator(n, src, dst, torch.float32, "csc")
    X = d.random_uniform(n, m, 12)
    rows = []
    for k in (8, 16, 32, 64, 128, 256, 512, 1024):
        th, b = d.gcn_params(m, k, 14)
        G = d.random_uniform(n, k, 13)
        for fg in (False, True):
            cell = {"k": k, "fg": fg}
            for name, pol, caching in (("adaptive", "adaptive", True),
                                       ("transform-first", "transform-first", False),
                                       ("propagate-first", "propagate-first", False)):
                sch = d.resolve_scheme(pol, m, k, fg, caching)

                def step():
                    out, c = d.gcn_forward(A, X, th, b, sch)
                    d.gcn_backward(A, G, th, c, fg)

                cell[name] = timed(step)
                if name == "adaptive":
                    cell["adaptive_choice"] = str(sch)
            rows.append(cell)
            print(json.dumps(cell), file=sys.stderr, flush=True)
    return {"graph": "arxiv-shaped (n=169343, nnz=1335587)", "m": m, "unit": "ms", "rows": rows}


def config3():
    out = {}
    for name, n, edges in (("pubmed", 19717, 88648), ("flickr", 89250, 899756)):
        src, dst = d.synthetic_graph(n, edges / n, 1)
        P = d.Pattern.gat_pattern(n, src, dst)
        X = d.random_uniform(n, 500, 12)
        rows = []
        for k in (8, 16, 32, 64, 128):
            th, a_s, a_d, b = d.gat_params(500, 8, k, 14)
            G = d.random_uniform(n, 8 * k, 13)
            cell = {"k": k}
            for level in ("none", "features", "node-attn", "full"):
                def step():
                    o, c = d.gat_forward(P, X, th, a_s, a_d, b, 8, 0.2, level)
                    d.gat_backward(P, G, th, a_s, a_d, c, True)

                cell[level] = timed(step)
            rows.append(cell)
            print(name, json.dumps(cell), file=sys.stderr, flush=True)
        out[name] = {"n": n, "nnz": P.nnz, "heads": 8, "m": 500, "rows": rows}
    return out


if __name__ == "__main__":
    res = {"config2_gcn_layer": config2(), "config3_gat_layer": config3(),
           "protocol": f"median of {STEPS} fwd+bwd steps, L2 flushed (256 MiB write + read-back)"}
    print(json.dumps(res))
