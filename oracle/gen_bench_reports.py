"""Golden BenchReports -- TEST INFRASTRUCTURE ONLY.

Runs the reference's own run_benchmark (bench.hpp:228-288, through oracle/_ref
ref_bench_report_json) over a grid of 2-layer model configurations on a small
synthetic graph and keeps the deterministic fields of each report (n, q, the
operation counters and cache_mem).  tests/test_report.py pins the analytic
counter restatement of paper_2308_12093_b200/report.py to them.
Run in the dev container:  python oracle/gen_bench_reports.py
"""
import ctypes as C
import itertools
import json
import os

import refpy

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "..", "tests", "golden", "bench_reports.json")
DATASET = "synth:n=240,deg=5,seed=3"
KEEP = ("n", "q", "flops", "bytes", "gemm_flops", "spmm_flops", "sddmm_flops", "edge_flops",
        "elementwise_flops", "cache_mem", "scheme", "caching", "pass", "precision", "format",
        "model", "hidden", "heads")
FORMATS = ["coo", "csr", "csc", "ellpack", "hybrid"]


def main():
    lib = refpy.lib()
    buf = C.create_string_buffer(1 << 16)
    cells = []
    grid = []
    for fmt, pol, cach, fb, fg, f32 in itertools.product(range(5), range(3), range(2), (0, 1),
                                                        (0, 1), (0, 1)):
        grid.append(dict(gat2=0, fmt=fmt, hidden=6, heads=1, policy=pol, level=cach,
                         fwdbwd=fb, fg=fg, f32=f32, in_features=9, classes=4))
    for fmt, lv, fb, fg, f32 in itertools.product(range(5), range(4), (0, 1), (0, 1), (0, 1)):
        grid.append(dict(gat2=1, fmt=fmt, hidden=3, heads=2, policy=0, level=lv, fwdbwd=fb,
                         fg=fg, f32=f32, in_features=5, classes=2))
    for g in grid:
        n = lib.ref_bench_report_json(DATASET.encode(), g["gat2"], g["fmt"], g["hidden"],
                                      g["heads"], g["policy"], g["level"], g["fwdbwd"], g["fg"],
                                      g["f32"], g["in_features"], g["classes"], 0, buf, 1 << 16)
        if n < 0:
            raise RuntimeError(lib.ref_last_error().decode())
        rep = json.loads(buf.value.decode())
        assert rep["schema_version"] == 1 and "error" not in rep, rep
        cells.append({"config": g, "report": {k: rep[k] for k in KEEP}})
    with open(OUT, "w") as fh:
        json.dump({"dataset": DATASET, "seed": 0, "cells": cells}, fh, indent=0, sort_keys=True)
    print(f"{len(cells)} reports -> {OUT}")


if __name__ == "__main__":
    main()
