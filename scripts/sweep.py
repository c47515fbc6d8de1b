"""Configs 2 and 3 of BASELINE.json on one B200, next to the reference's own
CPU path timed in the same run on this box's host cores:

  config 2: one GCN layer fwd+bwd on the Arxiv-shaped graph, 128 -> k for
            k in 8..1024, needs_feature_grad in {0, 1}, the adaptive scheme
            (with caching) against both forced schemes;
  config 3: one GAT layer fwd+bwd (8 heads, 500 -> 8 x k, input gradients)
            on PubMed- and Flickr-shaped graphs for k in 8..128 and every
            cache level.

Per cell: device ms (the step captured once into a CUDA graph and replayed --
device.StepGraph -- CUDA events, L2 flushed with a 256 MiB write + read-back
before every replay, median of STEPS), the step's algorithmic bytes (the
compulsory bytes of its kernels: SpMM 4(n+1)+8q'+8nf, GEMM
4(rows K + K N + rows N), GAT kernels as listed there) and their fraction of
the measured HBM copy bandwidth, edges/s, and the reference's CPU ms for the
same cell (oracle/_ref: the unmodified headers, -O3 -fopenmp, float32, CSC /
the GAT pattern, one step after a warm-up, every host core).  Prints one JSON
object (kept under profiles/<round>/).

  STEPS=10 REF=1 python scripts/sweep.py > profiles/r2/sweep_config2_config3.json
"""
import json
import os
import platform
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import torch  # noqa: E402

from paper_2308_12093_b200 import device as d  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from stepbytes import gat_step_bytes, gcn_step_bytes  # noqa: E402

STEPS = int(os.environ.get("STEPS", "10"))
REF = os.environ.get("REF", "1") == "1"
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
SEED = 1


def _peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except Exception:
        return 6650.0


HBM = _peak()


def timed(fn):
    g = d.StepGraph(fn)
    for _ in range(3):
        g.replay()
    ms = []
    for _ in range(STEPS):
        flush.fill_(1)
        flush.view(torch.int64).sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    return statistics.median(ms)


def ref_ms(kind, n, deg, m, k, heads, fg, policy, caching, level):
    """The reference's CPU step for the same cell (oracle/_ref, float32)."""
    if not REF:
        return None
    import refpy

    L = refpy.lib()
    h = L.ref_bench_create(kind, n, deg, SEED, m, k, heads, int(fg), policy, int(caching), level,
                           2)
    if not h:
        return f"unavailable: {L.ref_last_error().decode()}"
    L.ref_bench_step(h)  # warm-up
    t = L.ref_bench_step(h)
    L.ref_bench_destroy(h)
    return round(1e3 * t, 2)


def cell(ms, by, nnz, ref):
    gbs = by / (ms * 1e-3) / 1e9
    out = {"ms": round(ms, 4), "algorithmic_bytes": by, "gbs": round(gbs, 1),
           "frac_hbm": round(gbs / HBM, 3), "edges_per_s": round(nnz / (ms * 1e-3), 1)}
    if ref is not None:
        out["reference_cpu_ms"] = ref
        if isinstance(ref, float):
            out["speedup_vs_reference"] = round(ref / ms, 1)
    return out


def config2():
    n, m, edges = 169343, 128, 1166243
    src, dst = d.synthetic_graph(n, edges / n, SEED)
    A = d.Adjacency.gcn_operator(n, src, dst, torch.float32, "csc")
    X = d.random_uniform(n, m, SEED + 11)
    rows = []
    for k in (8, 16, 32, 64, 128, 256, 512, 1024):
        th, b = d.gcn_params(m, k, SEED + 13)
        G = d.random_uniform(n, k, SEED + 12)
        for fg in (False, True):
            row = {"k": k, "fg": fg}
            for name, pol, caching in (("adaptive", "adaptive", True),
                                       ("transform-first", "transform-first", False),
                                       ("propagate-first", "propagate-first", False)):
                sch = d.resolve_scheme(pol, m, k, fg, caching)

                def step(sch=sch, fg=fg):
                    out, c = d.gcn_forward(A, X, th, b, sch)
                    return (out,) + d.gcn_backward(A, G, th, c, fg)

                ms = timed(step)
                polid = {"adaptive": 0, "transform-first": 1, "propagate-first": 2}[pol]
                row[name] = cell(ms, gcn_step_bytes(sch, n, A.nnz, m, k, fg), A.nnz,
                                 ref_ms(0, n, edges / n, m, k, 1, fg, polid, caching, 0))
                row[name]["scheme"] = str(sch)
            rows.append(row)
            print(json.dumps(row), file=sys.stderr, flush=True)
    return {"graph": f"synthetic_graph(n={n}, deg={edges}/{n}, seed={SEED}) + gcn_normalize",
            "nnz": A.nnz, "m": m, "rows": rows}


def config3():
    out = {}
    for name, n, edges in (("pubmed", 19717, 88648), ("flickr", 89250, 899756)):
        src, dst = d.synthetic_graph(n, edges / n, SEED)
        P = d.Pattern.gat_pattern(n, src, dst)
        X = d.random_uniform(n, 500, SEED + 11)
        rows = []
        for k in (8, 16, 32, 64, 128):
            th, a_s, a_d, b = d.gat_params(500, 8, k, SEED + 13)
            G = d.random_uniform(n, 8 * k, SEED + 12)
            row = {"k": k}
            for li, level in enumerate(("none", "features", "node-attn", "full")):
                def step(level=level):
                    o, c = d.gat_forward(P, X, th, a_s, a_d, b, 8, 0.2, level)
                    return (o,) + d.gat_backward(P, G, th, a_s, a_d, c, True)

                ms = timed(step)
                row[level] = cell(ms, gat_step_bytes(level, n, P.nnz, 500, 8, k), P.nnz,
                                  ref_ms(1, n, edges / n, 500, k, 8, True, 0, False, li))
            rows.append(row)
            print(name, json.dumps(row), file=sys.stderr, flush=True)
        out[name] = {"graph": f"synthetic_graph(n={n}, deg={edges}/{n}, seed={SEED}) "
                              "+ add_self_loops", "n": n, "nnz": P.nnz, "heads": 8, "m": 500,
                     "rows": rows}
    return out


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or platform.machine()


if __name__ == "__main__":
    cores = None
    if REF:
        import refpy

        cores = refpy.lib().ref_num_threads()
    res = {"config2_gcn_layer": config2(), "config3_gat_layer": config3(),
           "protocol": f"CUDA-graph replay, median of {STEPS} fwd+bwd steps, L2 flushed "
                       "(256 MiB write + read-back) before each",
           "hbm_peak_gbs": HBM,
           "reference": {"kind": "oracle/_ref (unmodified headers, -O3 -fopenmp, float32)",
                         "cores": cores, "cpu": _cpu_model(),
                         "sample": "1 step after 1 warm-up step per cell"} if REF else None,
           "device": torch.cuda.get_device_name()}
    print(json.dumps(res))
