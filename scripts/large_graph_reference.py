"""Config 5 CPU baseline: the reference's own Gcn2Model / Gat2Model training
step (oracle/_ref: the unmodified headers, -O3 -fopenmp, float32, every host
core) at the large-graph shape -- n = 2,449,029, 61,859,140 / n average degree,
100 input features, Gcn2 100-256-47 (adaptive + caching), Gat2 100-(8x32)-(8x8)
(level full), MSE.  The reference has no power-law generator, so its graph is
its own uniform synthetic_graph at the same n and degree (the ER proxy of
SURVEY 8); bench.py's `large_graph` line times the device engine on the
power-law graph and profiles/r2/large_graph.json keeps both.  One step after
one warm-up (each takes tens of seconds on the CPU).

  python scripts/large_graph_reference.py > gpurun_out/large_graph_reference.json
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import refpy  # noqa: E402

N, EDGES, SEED, M = 2449029, 61859140, 1, 100


def main():
    L = refpy.lib()
    out = {"graph": f"synthetic_graph(n={N}, deg={EDGES}/{N}, seed={SEED}) (the reference's "
                    "uniform generator; ER proxy of the power-law graph)",
           "cores": L.ref_num_threads(), "precision": "f32",
           "kind": "oracle/_ref (unmodified reference headers, -O3 -fopenmp)"}
    for name, kind, hid, heads, caching, level in (("gcn2", 2, 256, 1, 1, 47 << 8),
                                                    ("gat2", 3, 32, 8, 0, 3 | (8 << 8))):
        t0 = time.perf_counter()
        h = L.ref_bench_create(kind, N, EDGES / N, SEED, M, hid, heads, 0, 0, caching, level, 2)
        if not h:
            out[name] = {"unavailable": L.ref_last_error().decode()}
            continue
        setup = time.perf_counter() - t0
        L.ref_bench_step(h)
        ms = 1e3 * L.ref_bench_step(h)
        out[name] = {"ms": round(ms, 1), "nnz": L.ref_bench_nnz(h), "setup_s": round(setup, 1),
                     "edges_per_s": round(2 * L.ref_bench_nnz(h) / (ms * 1e-3), 1)}
        L.ref_bench_destroy(h)
        print(name, json.dumps(out[name]), file=sys.stderr, flush=True)
    out["gcn2"]["shape"] = f"{M}-256-47 adaptive+caching, MSE"
    out["gat2"]["shape"] = f"{M}-(8x32)-(8x8) level full, MSE"
    print(json.dumps(out))


if __name__ == "__main__":
    main()
