"""Benchmark reports (bench.hpp:52-71, 292-437): the BenchReport record with
schema_version 1, its CSV row / JSON object emission, and the analytic
operation counters of a 2-layer model step.

The reference's counters (counters.hpp) are analytic: every kernel entry point
charges its model cost once per call (flops per class and model_bytes).
`step_counters` restates those charges for the work a Gcn2Model / Gat2Model
step performs -- dense.hpp:108-111 (gemm), 163 (bias), 204 / 242
(activation), 274 (column_sums); kernels.hpp:150-162 (spmm: cost.hpp
spmm_cost / spmm_cost_hybrid bytes), 224-227 / 264-267 (semibatched SpMM),
348-351 (SDDMM), 392-394 (node scores), 432-434 (edge scores), 463 / 486
(LeakyReLU), 504-506 / 542-544 (softmax), 573 / 642 (row / column sums), 598
(attention_param_grad), 621 (add_scaled_rows); model.hpp loss_mse -- in the
order gcn.hpp:91-193, gat.hpp:89-219 and model.hpp:52-163 call them.  They
are pinned to the reference's own BenchReport counters over a grid of
configurations (tests/test_report.py, tests/golden/bench_reports.json).
Host-pure: no device work here.
"""
from __future__ import annotations

import json
import math

import numpy as np

SCHEMA_VERSION = 1
FORMATS = ("coo", "csr", "csc", "ellpack", "hybrid")
LEVELS = ("none", "features", "node-attn", "full")

# cost.hpp:259-272 (the cost CLI's recorded dataset statistics)
DATASET_STATS = {
    "cora": dict(nodes=2708, edges=10556, features=1433, classes=7, avg_degree=7.8,
                 max_degree=168),
    "citeseer": dict(nodes=3327, edges=9104, features=3703, classes=6, avg_degree=5.47,
                     max_degree=0),
    "pubmed": dict(nodes=19717, edges=88648, features=500, classes=3, avg_degree=8.99,
                   max_degree=0),
    "flickr": dict(nodes=89250, edges=899756, features=500, classes=7, avg_degree=5.47,
                   max_degree=0),
    "ogb-arxiv": dict(nodes=169343, edges=1166243, features=128, classes=40, avg_degree=13.77,
                      max_degree=436),
}


# ---------------------------------------------------------------------------
# cost model (cost.hpp:42-114)
# ---------------------------------------------------------------------------
def _sparse_bytes(fmt, n, q, p, sb, ib=4):
    if fmt in ("csr", "csc"):
        return ib * (q + n + 1) + sb * q
    if fmt == "coo":
        return ib * 2 * q + sb * q
    if fmt == "ellpack":
        if p <= 0:
            raise ValueError("cost: ELLPACK width p is required")
        return (ib + sb) * n * p
    raise ValueError("cost: hybrid needs the per-part split, use the *_hybrid overload")


def spmm_cost(fmt, n, q, p, f, sb=4, ib=4):
    flops = 2 * q * f
    by = _sparse_bytes(fmt, n, q, p, sb, ib) + 3 * sb * n * f
    return flops, by, (flops / by if by else 0.0)


def spmm_cost_hybrid(n, q_csr, q_coo, f, sb=4, ib=4):
    q = q_csr + q_coo
    by = _sparse_bytes("csr", n, q_csr, 0, sb, ib) + _sparse_bytes("coo", n, q_coo, 0, sb, ib) \
        + 3 * sb * n * f
    return 2 * q * f, by, (2 * q * f / by if by else 0.0)


# ---------------------------------------------------------------------------
# the operator a layer multiplies with, as the cost model sees it
# ---------------------------------------------------------------------------
class OperatorShape:
    """n, q and the per-row / per-column nonzero counts of the stored matrix
    in `fmt` -- enough for every spmm_cost the forward (stored matrix) and
    backward (its transpose, transpose_any: sparse.hpp:423-451) charge."""

    def __init__(self, fmt, n, row_counts, col_counts):
        if fmt not in FORMATS:
            raise ValueError(f"unknown format '{fmt}'")
        self.fmt, self.n = fmt, int(n)
        self.rows = np.asarray(row_counts, np.int64)
        self.cols = np.asarray(col_counts, np.int64)
        self.q = int(self.rows.sum())
        # sparse.hpp:294-299 default_hybrid_t (the transpose keeps the same t)
        self.t = max(1, math.ceil(self.q / self.n)) if self.n else 1

    def spmm_bytes(self, f, sb, transposed=False):
        counts = self.cols if transposed else self.rows
        if self.fmt == "hybrid":
            q_csr = int(np.minimum(counts, self.t).sum())
            return spmm_cost_hybrid(self.n, q_csr, self.q - q_csr, f, sb)[1]
        fmt = self.fmt
        if transposed and fmt in ("csr", "csc"):
            fmt = "csc" if fmt == "csr" else "csr"
        p = int(counts.max()) if (fmt == "ellpack" and len(counts)) else 0
        return spmm_cost(fmt, self.n, self.q, p, f, sb)[1]


class Counters:
    """counters.hpp OpCounters."""

    FIELDS = ("gemm_flops", "spmm_flops", "sddmm_flops", "edge_flops", "elementwise_flops",
              "model_bytes")

    def __init__(self):
        for f in self.FIELDS:
            setattr(self, f, 0)

    def total_flops(self):
        return (self.gemm_flops + self.spmm_flops + self.sddmm_flops + self.edge_flops
                + self.elementwise_flops)

    # kernel charge sites
    def gemm(self, m, n, kk, sb):  # dense.hpp:108-111, C (m x n) = op(A) (m x kk) op(B)
        self.gemm_flops += 2 * m * n * kk
        self.model_bytes += sb * (m * kk + kk * n + m * n)

    def spmm(self, op: OperatorShape, f, sb, transposed=False):  # kernels.hpp:150-162
        self.spmm_flops += 2 * op.q * f
        self.model_bytes += op.spmm_bytes(f, sb, transposed)

    def elementwise(self, count):
        self.elementwise_flops += count


# ---------------------------------------------------------------------------
# GCN / GAT layer and model steps
# ---------------------------------------------------------------------------
def _gcn_forward(c, op, n, m, k, fwd, sb):
    if fwd == 0:  # transform-first: M = X Theta, A'M
        c.gemm(n, k, m, sb)
        c.spmm(op, k, sb)
    else:  # propagate-first (+cached): P = A'X, P Theta
        c.spmm(op, m, sb)
        c.gemm(n, k, m, sb)
    c.elementwise(n * k)  # bias


def _gcn_backward(c, op, n, m, k, bwd, fg, sb):
    c.elementwise(n * k)  # column_sums(d_out)
    if bwd == 0:  # fused
        c.spmm(op, k, sb, transposed=True)
        c.gemm(m, k, n, sb)
        if fg:
            c.gemm(n, m, k, sb)
    elif bwd == 1:  # split
        c.spmm(op, m, sb)
        if fg:
            c.gemm(n, m, k, sb)
        c.gemm(m, k, n, sb)
        if fg:
            c.spmm(op, m, sb, transposed=True)
    else:  # split cached
        c.gemm(m, k, n, sb)
        if fg:
            c.gemm(n, m, k, sb)
            c.spmm(op, m, sb, transposed=True)


def _gat_scores_softmax(c, n, h, k, q, sb):
    c.gemm_flops += 4 * n * h * k  # node_scores (kernels.hpp:392-394)
    c.model_bytes += sb * (n * h * k + 2 * n * h)
    c.edge_flops += q * h  # edge_scores (:432-434)
    c.model_bytes += sb * (q * h + 2 * n * h)
    c.edge_flops += h * q  # leaky_relu_edges (:463)
    c.edge_flops += 5 * h * q  # edge_softmax (:504-506)
    c.model_bytes += 2 * sb * h * q


def _semibatched(c, n, h, k, q, sb):  # kernels.hpp:224-227 / 264-267
    c.spmm_flops += 2 * q * h * k
    c.model_bytes += sb * (h * q + 3 * n * h * k) + 4 * (q + n + 1)


def _gat_forward(c, n, m, h, k, q, sb):
    c.gemm(n, h * k, m, sb)
    _gat_scores_softmax(c, n, h, k, q, sb)
    _semibatched(c, n, h, k, q, sb)
    c.elementwise(n * h * k)  # bias


def _gat_backward(c, n, m, h, k, q, level, fg, sb):
    hk = h * k
    c.elementwise(n * hk)  # column_sums(d_out)
    lv = LEVELS.index(level)
    if lv < 1:
        c.gemm(n, hk, m, sb)  # gat_recompute: M = X Theta
    if lv < 3:
        if lv != 2:
            c.gemm_flops += 4 * n * h * k
            c.model_bytes += sb * (n * h * k + 2 * n * h)
        c.edge_flops += q * h
        c.model_bytes += sb * (q * h + 2 * n * h)
        c.edge_flops += 6 * h * q
        c.model_bytes += 2 * sb * h * q
    c.sddmm_flops += q * h * (2 * k + 1)  # kernels.hpp:348-351
    c.model_bytes += sb * (q * h * (k + 1)) + 4 * (q + n + 1)
    c.edge_flops += 4 * h * q  # edge_softmax_backward (:542-544)
    c.model_bytes += 3 * sb * h * q
    c.edge_flops += 3 * h * q  # leaky backward, row sums, column sums
    _semibatched(c, n, h, k, q, sb)  # spmm_semibatched_transposed
    c.elementwise(2 * 2 * n * hk)  # add_scaled_rows_inplace x 2
    c.gemm_flops += 2 * 2 * n * hk  # attention_param_grad x 2
    c.gemm(m, hk, n, sb)  # dTheta = X^T dM
    if fg:
        c.gemm(n, m, hk, sb)  # dX = dM Theta^T


def step_counters(model, op: OperatorShape, n, in_features, hidden, classes, heads=1,
                  scheme=(None, None), gat_level="none", fwdbwd=True, input_grad=False,
                  scalar_bytes=8) -> Counters:
    """Counters of one Gcn2Model / Gat2Model step (model.hpp:52-163 plus
    loss_mse when fwdbwd), i.e. the reference's instrumented bench pass
    (bench.hpp:228-257).  scheme: the two layers' (forward, backward) scheme
    ints for gcn2 (device.resolve_scheme / the reference's resolve_scheme)."""
    c, sb = Counters(), scalar_bytes
    if model == "gcn2":
        (f1, b1), (f2, b2) = scheme
        _gcn_forward(c, op, n, in_features, hidden, f1, sb)
        c.elementwise(n * hidden)  # relu
        _gcn_forward(c, op, n, hidden, classes, f2, sb)
        if fwdbwd:
            c.elementwise(3 * n * classes)  # loss_mse
            _gcn_backward(c, op, n, hidden, classes, b2, True, sb)
            c.elementwise(n * hidden)  # relu backward
            _gcn_backward(c, op, n, in_features, hidden, b1, input_grad, sb)
        return c
    q = op.q
    _gat_forward(c, n, in_features, heads, hidden, q, sb)
    c.elementwise(n * heads * hidden)  # elu
    _gat_forward(c, n, heads * hidden, heads, classes, q, sb)
    if fwdbwd:
        c.elementwise(3 * n * heads * classes)  # loss_mse
        _gat_backward(c, n, heads * hidden, heads, classes, q, gat_level, True, sb)
        c.elementwise(n * heads * hidden)  # elu backward
        _gat_backward(c, n, in_features, heads, hidden, q, gat_level, input_grad, sb)
    return c


# ---------------------------------------------------------------------------
# BenchReport and its emission (bench.hpp:52-71, 292-437)
# ---------------------------------------------------------------------------
REPORT_KEYS = ("schema_version", "dataset", "format", "model", "hidden", "heads", "scheme",
               "caching", "pass", "precision", "warmups", "blocks", "runs_per_block", "seed",
               "n", "q", "threads", "median_s", "std_s", "block_seconds", "flops", "bytes",
               "gemm_flops", "spmm_flops", "sddmm_flops", "edge_flops", "elementwise_flops",
               "peak_mem", "cache_mem")


def new_report(**kw):
    r = {k: 0 for k in REPORT_KEYS}
    r.update(schema_version=SCHEMA_VERSION, dataset="", format="", model="", scheme="",
             caching="", precision="", block_seconds=[])
    r["pass"] = ""
    r.update(kw)
    return r


def fill_counters(rep, c: Counters):
    """bench.hpp:152-161 fill_report_counters."""
    rep.update(flops=c.total_flops(), bytes=c.model_bytes, gemm_flops=c.gemm_flops,
               spmm_flops=c.spmm_flops, sddmm_flops=c.sddmm_flops, edge_flops=c.edge_flops,
               elementwise_flops=c.elementwise_flops)
    return rep


def timing_stats(block_seconds):
    """bench.hpp:82-108: median over blocks and the population std."""
    s = sorted(block_seconds)
    mid = len(s) // 2
    med = s[mid] if len(s) % 2 else 0.5 * (s[mid - 1] + s[mid])
    mean = sum(block_seconds) / len(block_seconds)
    std = math.sqrt(sum((x - mean) ** 2 for x in block_seconds) / len(block_seconds))
    return med, std


def csv_header():
    return ("dataset,format,model,hidden,heads,scheme,caching,pass,median_s,std_s,flops,bytes,"
            "peak_mem,cache_mem")


def _csv_quote(s):
    s = str(s)
    if not any(ch in s for ch in ',"\n'):
        return s
    return '"' + s.replace('"', '""') + '"'


def to_csv_row(r):
    cells = [r["dataset"], r["format"], r["model"], str(r["hidden"]), str(r["heads"]),
             r["scheme"], r["caching"], r["pass"]]
    if not r.get("error"):
        cells += ["%.9e" % r["median_s"], "%.9e" % r["std_s"], str(r["flops"]), str(r["bytes"]),
                  str(r["peak_mem"]), str(r["cache_mem"])]
    else:
        cells += [""] * 6
    return ",".join(_csv_quote(c) for c in cells)


def reports_to_csv(reports):
    return csv_header() + "\n" + "".join(to_csv_row(r) + "\n" for r in reports)


def report_to_json(r):
    j = {k: r[k] for k in REPORT_KEYS}
    if r.get("error"):
        j["error"] = r["error"]
    return j


def reports_to_json(reports):
    return {"schema_version": SCHEMA_VERSION, "reports": [report_to_json(r) for r in reports]}


def report_from_json(j):
    """bench.hpp:380-414: every key is required."""
    r = {k: j[k] for k in REPORT_KEYS}
    if "error" in j:
        r["error"] = j["error"]
    return r


def emit(reports, emit_format, path):
    text = reports_to_csv(reports) if emit_format == "csv" else \
        json.dumps(reports_to_json(reports), indent=2) + "\n"
    if path == "-":
        return text
    try:
        with open(path, "w") as fh:
            fh.write(text)
    except OSError:
        raise RuntimeError(f"cannot open {path} for writing") from None
    return None
