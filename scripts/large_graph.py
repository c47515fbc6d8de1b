"""Config 5 at one GPU: 2-layer GCN / GAT training steps on the large synthetic
graphs, 100 input features: the power-law graph of BASELINE config 5 (device
Chung-Lu generator, 2,449,029 nodes, 61,859,140 / 2,449,029 average degree,
exponent 2.5) and the reference generator's uniform ER proxy of SURVEY 8.
Prints one JSON line; results are kept under profiles/.

  python scripts/large_graph.py [--steps K] [--graph powerlaw|uniform|both]
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2308_12093_b200 import device as d  # noqa: E402

N, EDGES, SEED, M_IN = 2449029, 61859140, 1, 100


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--graph", default="both", choices=["powerlaw", "uniform", "both"])
    args = ap.parse_args()
    kinds = ["powerlaw", "uniform"] if args.graph == "both" else [args.graph]
    lines = [run(args, kind) for kind in kinds]
    print(json.dumps({"config5_one_gpu": lines}), flush=True)


def run(args, kind):
    ctx = d.Context.default(0)
    stream = torch.cuda.current_stream()
    t0 = time.perf_counter()
    if kind == "powerlaw":
        src, dst = d.powerlaw_graph(N, EDGES / N, 2.5, SEED, ctx)
        torch.cuda.synchronize()
    else:
        src, dst = d.synthetic_graph(N, EDGES / N, SEED)
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    A = d.Adjacency.gcn_operator(N, src, dst, torch.float32, "csc", ctx)
    P = d.Pattern.gat_pattern(N, src, dst, ctx)
    torch.cuda.synchronize()
    t_pre = time.perf_counter() - t0
    X = d.random_uniform(N, M_IN, SEED + 11, ctx=ctx)

    def timed(fn, iters, warm=2):
        for _ in range(warm):
            fn()
        ms = []
        for _ in range(iters):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        return statistics.median(ms)

    maxdeg = int(torch.bincount(src.to(ctx.device).long(), minlength=N).max())
    res = {"workload": "config 5 at 1 GPU: 2-layer train steps (MSE)",
           "graph": (f"powerlaw_graph(n={N}, deg={EDGES}/{N}, exponent=2.5, seed={SEED})"
                     if kind == "powerlaw" else
                     f"synthetic_graph(n={N}, deg={EDGES}/{N}, seed={SEED}) (ER proxy)"),
           "max_degree": maxdeg,
           "n": N, "nnz_gcn": A.nnz, "nnz_gat": P.nnz, "m": M_IN,
           "generate_s": round(t_gen, 2), "device_preprocess_s": round(t_pre, 2)}
    out = {}
    for name, model, graph, ow in (
            ("gcn2", d.Model("gcn2", M_IN, 256, 47, scheme="adaptive", caching=True,
                             seed=SEED + 13, ctx=ctx), A, 47),
            ("gat2", d.Model("gat2", M_IN, 32, 8, heads=8, gat_level="full", seed=SEED + 13,
                             ctx=ctx), P, 64)):
        tgt = d.random_uniform(N, ow, SEED + 12, ctx=ctx)
        ms = timed(lambda: model.train_step(graph, X, tgt), args.steps)
        out[name] = {"ms": round(ms, 3), "edges_per_s": round(graph.nnz / (ms * 1e-3), 1)}
        del model, tgt
        torch.cuda.empty_cache()
    out["gcn2"]["shape"] = f"{M_IN}-256-47 adaptive+caching"
    out["gat2"]["shape"] = f"{M_IN}-(8x32)-(8x8) level full"
    res["steps"] = out
    print(json.dumps(res), file=sys.stderr, flush=True)
    del A, P, X
    torch.cuda.empty_cache()
    return res


if __name__ == "__main__":
    main()
