"""sgnn-bench on B200 (tools/sgnn_bench.cpp:1-392): benchmark and inspection CLI.

  bench      time one 2-layer model configuration and emit a BenchReport
  sweep      run a grid (comma lists for --hidden/--format/--caching/--scheme)
  cost       print the analytic SpMM / SDDMM FLOP / byte / intensity model as CSV
  gradcheck  central finite-difference check of the model gradients (sum loss)
  gen        write a synthetic edge-list graph

Same subcommands, flags, SGNN_* environment variables, protocol defaults
(bench.hpp:43-49: forward 10 warmups + 10 blocks x 10 runs, forward+backward
10 warmups + 5 blocks x 4 runs) and report schema (schema_version 1,
bench.hpp:292-437) as the reference CLI.  The model steps run on the device
(libsgnn_cuda.so); block times are CUDA-event times on the context stream.
Report fields: counters are the reference's analytic charges
(report.step_counters, pinned to the reference's reports); peak_mem /
cache_mem are the device engine's tracked bytes (sgnn_mem_stats: logical
intermediates, caches); threads = the SM count the kernels run on.

  python -m paper_2308_12093_b200.bench_cli bench --dataset synth:n=2000,deg=8 ...
"""
from __future__ import annotations

import argparse
import math
import os
import sys

import numpy as np

from . import report as R

FORMATS = R.FORMATS
SCHEMES = ("adaptive", "transform-first", "propagate-first")
LEVELS = R.LEVELS


class UsageError(Exception):
    pass


def _env(name, default):
    return os.environ.get("SGNN_" + name, default)


def _add_common(p, gradcheck=False):
    e = _env
    if gradcheck:
        p.add_argument("--dataset", default=e("DATASET", ""))
    else:
        p.add_argument("--dataset", default=e("DATASET", None),
                       required=e("DATASET", None) is None,
                       help="graph file (.mtx or edge list) or synth:n=N,deg=D[,seed=S]")
        p.add_argument("--format", default=e("FORMAT", "csc"))
        p.add_argument("--pass", dest="pass_", default=e("PASS", "fwd"))
        p.add_argument("--feature-grad", default=e("FEATURE_GRAD", "off"))
        p.add_argument("--warmups", type=int, default=int(e("WARMUPS", -1)))
        p.add_argument("--blocks", type=int, default=int(e("BLOCKS", -1)))
        p.add_argument("--runs", type=int, default=int(e("RUNS", -1)))
        p.add_argument("--threads", type=int, default=int(e("THREADS", 0)))
        p.add_argument("--out", default=e("OUT", "-"))
        p.add_argument("--emit", default=e("EMIT", "csv"))
    p.add_argument("--model", default=e("MODEL", "gcn2"))
    p.add_argument("--hidden", default=e("HIDDEN", "5" if gradcheck else "64"))
    p.add_argument("--heads", type=int, default=int(e("HEADS", 2 if gradcheck else 8)))
    p.add_argument("--scheme", default=e("SCHEME", "adaptive"))
    p.add_argument("--caching", default=e("CACHING", "none"))
    p.add_argument("--precision", default=e("PRECISION", "f64"))
    p.add_argument("--in-features", type=int, default=int(e("IN_FEATURES", 4 if gradcheck else 128)))
    p.add_argument("--classes", type=int, default=int(e("CLASSES", 3 if gradcheck else 32)))
    p.add_argument("--seed", type=int, default=int(e("SEED", 0)))


# ---------------------------------------------------------------------------
# graphs (bench.hpp:115-140 resolve_dataset)
# ---------------------------------------------------------------------------
def resolve_dataset(spec, default_seed):
    """(n, src, dst, weight or None) -- host arrays for files, device for synth."""
    from . import _graph_io
    from . import device as d

    if spec.startswith("synth:"):
        n, deg, seed = 0, 0.0, default_seed
        for kv in filter(None, spec[6:].split(",")):
            if "=" not in kv:
                raise ValueError(f"synthetic spec: expected key=value, got '{kv}'")
            key, val = kv.split("=", 1)
            if key == "n":
                n = int(val)
            elif key == "deg":
                deg = float(val)
            elif key == "seed":
                seed = int(val)
            else:
                raise ValueError(f"synthetic spec: unknown key '{key}'")
        src, dst = d.synthetic_graph(n, deg, seed)
        return n, src, dst, None
    g = _graph_io.load_graph(spec, "matrix-market" if spec.endswith(".mtx") else "edge-list")
    return g["n"], g["src"], g["dst"], g["weight"]


def _device_graph(model, n, src, dst, w, fmt, dtype, ctx):
    """adjacency(graph) -> gcn_normalize -> convert (gcn2) or add_self_loops ->
    CSR -> SparsePattern (gat2), bench.hpp:193-211; with the OperatorShape the
    cost model charges."""
    import torch

    from . import device as d

    dev = ctx.device
    t = lambda a, dt: (a if isinstance(a, torch.Tensor) else torch.from_numpy(  # noqa: E731
        np.ascontiguousarray(a))).to(dev, dt)
    src, dst = t(src, torch.int32), t(dst, torch.int32)
    vals = torch.ones(src.numel(), dtype=dtype, device=dev) if w is None else t(w, dtype)
    r, c, v = d.canonicalize(n, n, src, dst, vals, ctx)
    if model == "gcn2":
        r, c, v = d.gcn_normalize(n, r, c, v, ctx)
        graph = d.Adjacency(n, n, r, c, v, fmt, ctx)
    else:
        r, c, v = d.add_self_loops(n, r, c, v, ctx)
        graph = d.Pattern(n, d.csr_from_coo(n, r, ctx), c, ctx)
    rc = torch.bincount(r.long(), minlength=n).cpu().numpy()
    cc = torch.bincount(c.long(), minlength=n).cpu().numpy()
    return graph, R.OperatorShape(fmt, n, rc, cc)


# ---------------------------------------------------------------------------
# bench / sweep (bench.hpp:163-288)
# ---------------------------------------------------------------------------
def _config_checks(o, hidden, fmt, caching, scheme):
    if fmt not in FORMATS:
        raise UsageError(f"--format: unknown format '{fmt}'")
    if scheme not in SCHEMES:
        raise UsageError(f"--scheme: unknown scheme '{scheme}'")
    if caching not in LEVELS:
        raise UsageError(f"--caching: unknown caching level '{caching}'")
    if o.pass_ not in ("fwd", "fwdbwd"):
        raise UsageError("--pass: expected fwd or fwdbwd")
    if o.precision not in ("f32", "f64"):
        raise UsageError("--precision: expected f32 or f64")
    if o.model not in ("gcn2", "gat2"):
        raise UsageError("--model: expected gcn2 or gat2")
    if o.feature_grad not in ("on", "off"):
        raise UsageError("--feature-grad: expected on or off")
    if o.model == "gcn2" and caching not in ("none", "features"):
        raise UsageError("--caching: gcn2 supports none or features")
    return int(hidden)


def run_benchmark(o, hidden, fmt, caching, scheme):
    """One BenchReport; failures are recorded in `error` (bench.hpp:264-280)."""
    rep = R.new_report(dataset=o.dataset, format=fmt, model=o.model, scheme=scheme,
                       hidden=hidden, heads=o.heads if o.model == "gat2" else 0,
                       caching=("features" if caching == "features" else "none")
                       if o.model == "gcn2" else caching)
    rep["pass"] = o.pass_
    try:
        return _run_benchmark(o, hidden, fmt, caching, scheme, rep)
    except Exception as ex:  # noqa: BLE001 -- a failed cell carries its error
        rep["error"] = str(ex)
        return rep


def _run_benchmark(o, hidden, fmt, caching, scheme, rep):
    import torch

    from . import device as d

    ctx = d.Context.default()
    dtype = torch.float32 if o.precision == "f32" else torch.float64
    fwdbwd = o.pass_ == "fwdbwd"
    warm = o.warmups if o.warmups >= 0 else 10
    blocks = o.blocks if o.blocks >= 0 else (5 if fwdbwd else 10)
    runs = o.runs if o.runs >= 0 else (4 if fwdbwd else 10)
    if blocks < 1 or runs < 1:
        raise ValueError("run_timed: blocks*runs must be positive")
    rep.update(precision=o.precision, warmups=warm, blocks=blocks, runs_per_block=runs,
               seed=o.seed, threads=ctx_sms(ctx))
    n, src, dst, w = resolve_dataset(o.dataset, o.seed)
    graph, shape = _device_graph(o.model, n, src, dst, w, fmt, dtype, ctx)
    rep.update(n=n, q=shape.q)
    fg = o.feature_grad == "on"
    gcn = o.model == "gcn2"
    model = d.Model(o.model, o.in_features, hidden, o.classes, heads=o.heads, scheme=scheme,
                    caching=caching == "features", gat_level=caching, input_grad=fg,
                    seed=o.seed + 13, dtype=dtype, ctx=ctx)
    X = d.random_uniform(n, o.in_features, o.seed + 11, dtype=dtype, ctx=ctx)
    target = d.random_uniform(n, model.out_width, o.seed + 12, dtype=dtype, ctx=ctx)
    params = [p for _, p in model.param_tensors()]
    s1 = d.resolve_scheme(scheme, o.in_features, hidden, fg, caching == "features")
    s2 = d.resolve_scheme(scheme, hidden, o.classes, True, caching == "features")

    def forward():  # model.hpp:52-69 / 133-150 through the layer API
        if gcn:
            o1, c1 = d.gcn_forward(graph, X, params[0], params[1], s1)
            h, _ = d.activation(o1, "relu", ctx=ctx)
            return d.gcn_forward(graph, h, params[2], params[3], s2), c1
        o1, c1 = d.gat_forward(graph, X, *params[:4], o.heads, 0.2, caching)
        h, _ = d.activation(o1, "elu", ctx=ctx)
        return d.gat_forward(graph, h, *params[4:], o.heads, 0.2, caching), c1

    def step():
        if fwdbwd:
            model.train_step(graph, X, target)
        else:
            forward()

    # instrumented pass (bench.hpp:228-257): counters, device peak / cache bytes
    torch.cuda.synchronize()
    live0 = d.memory_stats("all")[0]
    cache0 = d.memory_stats("cache")[0]
    d.reset_memory_peaks()
    (out2, c2), c1 = forward()
    torch.cuda.synchronize()
    rep["cache_mem"] = d.memory_stats("cache")[0] - cache0
    del out2, c2, c1
    step()
    torch.cuda.synchronize()
    rep["peak_mem"] = d.memory_stats("all")[1] - live0
    sc = ((s1.forward, s1.backward), (s2.forward, s2.backward))
    R.fill_counters(rep, R.step_counters(o.model, shape, n, o.in_features, hidden, o.classes,
                                         heads=o.heads, scheme=sc, gat_level=caching,
                                         fwdbwd=fwdbwd, input_grad=fg,
                                         scalar_bytes=4 if dtype == torch.float32 else 8))
    # timed protocol (bench.hpp:82-108), device time per block / runs
    for _ in range(warm):
        step()
    stream = torch.cuda.current_stream()
    secs = []
    for _ in range(blocks):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(runs):
            step()
        e1.record(stream)
        e1.synchronize()
        secs.append(e0.elapsed_time(e1) * 1e-3 / runs)
    rep["block_seconds"] = secs
    rep["median_s"], rep["std_s"] = R.timing_stats(secs)
    return rep


def ctx_sms(ctx):
    import torch

    return torch.cuda.get_device_properties(ctx.device).multi_processor_count


def _split(s):
    return [x for x in s.split(",") if x]


def cmd_bench(o, grid):
    cells = []
    for h in (_split(o.hidden) if grid else [o.hidden]):
        for f in (_split(o.format) if grid else [o.format]):
            for c in (_split(o.caching) if grid else [o.caching]):
                for s in (_split(o.scheme) if grid else [o.scheme]):
                    cells.append((_config_checks(o, h, f, c, s), f, c, s))
    if o.emit not in ("csv", "json"):
        raise UsageError("--emit: expected csv or json")
    reports = [run_benchmark(o, *cell) for cell in cells]
    text = R.emit(reports, o.emit, o.out)
    if text is not None:
        sys.stdout.write(text)
    else:
        print(f"wrote {len(reports)} report(s) to {o.out}", file=sys.stderr)
    fails = [r for r in reports if r.get("error")]
    for r in fails:
        print(f"cell failed: {r['dataset']} hidden={r['hidden']}: {r['error']}", file=sys.stderr)
    return 0 if not fails else 1


# ---------------------------------------------------------------------------
# cost (sgnn_bench.cpp:188-218)
# ---------------------------------------------------------------------------
def cmd_cost(o):
    from . import sgnn

    n, q, p, f = o.n, o.q, o.max_degree, o.f
    if o.dataset_stats:
        st = R.DATASET_STATS.get(o.dataset_stats)
        if st is None:
            raise UsageError(f"--dataset-stats: unknown dataset '{o.dataset_stats}'")
        n, q, p = st["nodes"], st["edges"], st["max_degree"]
    lines = ["op,format,n,q,p,f,flops,bytes,oi"]
    for fmt in ("csr", "csc", "coo", "ellpack"):
        pp = p if fmt == "ellpack" else 0
        if fmt == "ellpack" and p <= 0:
            continue
        for op, fn in (("spmm", sgnn.spmm_cost), ("sddmm", sgnn.sddmm_cost)):
            if o.op in (op, "both"):
                c = fn(fmt, n, q, p=pp, f=f)
                lines.append(f"{op},{fmt},{n},{q},{pp},{f},{c['flops']},{c['bytes']},"
                             f"{c['operational_intensity']:.6f}")
    text = "\n".join(lines) + "\n"
    if o.out == "-":
        sys.stdout.write(text)
    else:
        with open(o.out, "w") as fh:
            fh.write(text)
    return 0


# ---------------------------------------------------------------------------
# gradcheck (sgnn_bench.cpp:220-289, model.hpp:326-363)
# ---------------------------------------------------------------------------
def cmd_gradcheck(o):
    import torch

    from . import device as d

    gat = o.model == "gat2"
    eps = o.eps if o.eps > 0 else (1e-5 if gat else 1e-6)
    tol = o.tol if o.tol > 0 else (1e-5 if gat else 1e-6)
    dtype = torch.float32 if o.precision == "f32" else torch.float64
    ctx = d.Context.default()
    if o.dataset:
        n, src, dst, w = resolve_dataset(o.dataset, o.seed + 1)
    else:
        src, dst = d.synthetic_graph(o.n, o.avg_degree, o.seed + 1)
        n, w = o.n, None
    graph, _ = _device_graph(o.model, n, src, dst, w, "csc", dtype, ctx)
    hidden = int(o.hidden)
    X = d.random_uniform(n, o.in_features, o.seed + 2, dtype=dtype, ctx=ctx)
    model = d.Model(o.model, o.in_features, hidden, o.classes, heads=o.heads, scheme=o.scheme,
                    caching=o.caching != "none", gat_level=o.caching, input_grad=True,
                    seed=o.seed + 3, dtype=dtype, ctx=ctx)
    named = model.param_tensors()
    P = [p for _, p in named]
    level = o.caching
    s1 = d.resolve_scheme(o.scheme, o.in_features, hidden, True, o.caching != "none")
    s2 = d.resolve_scheme(o.scheme, hidden, o.classes, True, o.caching != "none")

    def forward():
        if gat:
            o1, c1 = d.gat_forward(graph, X, *P[:4], o.heads, 0.2, level)
            h, mask = d.activation(o1, "elu", ctx=ctx)
            o2, c2 = d.gat_forward(graph, h, *P[4:], o.heads, 0.2, level)
        else:
            o1, c1 = d.gcn_forward(graph, X, P[0], P[1], s1)
            h, mask = d.activation(o1, "relu", ctx=ctx)
            o2, c2 = d.gcn_forward(graph, h, P[2], P[3], s2)
        return o2, (c1, c2, h, mask)

    out, (c1, c2, h, mask) = forward()  # loss_sum: dL/dout = 1
    ones = torch.ones_like(out)
    if gat:
        g2 = d.gat_backward(graph, ones, *P[4:7], c2, True)
        dh = d.activation_backward(g2[4], mask, "elu", saved=h, ctx=ctx)
        g1 = d.gat_backward(graph, dh, *P[:3], c1, True)
        grads = list(g1[:4]) + list(g2[:4])
    else:
        g2 = d.gcn_backward(graph, ones, P[2], c2, True)
        dh = d.activation_backward(g2[2], mask, "relu", ctx=ctx)
        g1 = d.gcn_backward(graph, dh, P[0], c1, True)
        grads = [g1[0], g1[1], g2[0], g2[1]]

    def loss():
        return float(forward()[0].double().sum())

    rng = np.random.default_rng(o.seed + 4)
    worst, worst_name, coords = 0.0, "", 0
    for (name, p), g in zip(named, grads):
        flat, gflat = p.view(-1), g.reshape(-1).double().cpu().numpy()
        idx = range(flat.numel()) if flat.numel() <= 200 else rng.integers(0, flat.numel(), 200)
        for i in idx:
            saved = float(flat[i])
            flat[i] = saved + eps
            up = loss()
            flat[i] = saved - eps
            down = loss()
            flat[i] = saved
            if not (math.isfinite(up) and math.isfinite(down)):
                raise RuntimeError("gradient_check: non-finite loss")
            fd = (up - down) / (2 * eps)
            err = abs(gflat[i] - fd) / max(1.0, abs(gflat[i]), abs(fd))
            if err > worst:
                worst, worst_name = err, name
            coords += 1
    print(f"model={o.model} coords={coords} max_rel_err={worst:g} worst={worst_name} "
          f"tol={tol:g} -> {'PASS' if worst < tol else 'FAIL'}")
    return 0 if worst < tol else 1


# ---------------------------------------------------------------------------
# gen (graph.hpp:149-158 save_edge_list)
# ---------------------------------------------------------------------------
def cmd_gen(o):
    from . import device as d

    src, dst = d.synthetic_graph(o.n, o.avg_degree, o.seed)
    s, t = src.cpu().numpy(), dst.cpu().numpy()
    try:
        fh = open(o.out, "w")
    except OSError:
        raise RuntimeError(f"cannot open {o.out} for writing") from None
    with fh:
        fh.write(f"# nodes {o.n} edges {len(s)}\n")
        fh.write("".join(f"{a} {b}\n" for a, b in zip(s.tolist(), t.tolist())))
    print(f"wrote {o.out}", file=sys.stderr)
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser(prog="sgnn-bench",
                                 description="sparse GNN training kernels on B200: benchmarks, "
                                             "cost model, checks")
    sub = ap.add_subparsers(dest="cmd", required=True)
    _add_common(sub.add_parser("bench", help="time one configuration"))
    _add_common(sub.add_parser("sweep", help="run a configuration grid"))
    c = sub.add_parser("cost", help="print the analytic cost model")
    c.add_argument("--n", type=int, default=int(_env("N", 0)))
    c.add_argument("--q", type=int, default=int(_env("Q", 0)))
    c.add_argument("--max-degree", type=int, default=int(_env("MAX_DEGREE", 0)))
    c.add_argument("--f", type=int, default=int(_env("F", 64)))
    c.add_argument("--op", default=_env("OP", "both"))
    c.add_argument("--dataset-stats", default=_env("DATASET_STATS", ""))
    c.add_argument("--out", default=_env("OUT", "-"))
    g = sub.add_parser("gradcheck", help="finite-difference gradient check")
    _add_common(g, gradcheck=True)
    g.add_argument("--n", type=int, default=int(_env("N", 12)))
    g.add_argument("--avg-degree", type=float, default=float(_env("AVG_DEGREE", 3.0)))
    g.add_argument("--eps", type=float, default=float(_env("EPS", 0.0)))
    g.add_argument("--tol", type=float, default=float(_env("TOL", 0.0)))
    n = sub.add_parser("gen", help="write a synthetic edge-list graph")
    n.add_argument("--n", type=int, required=_env("N", None) is None, default=_env("N", None))
    n.add_argument("--avg-degree", type=float, required=_env("AVG_DEGREE", None) is None,
                   default=_env("AVG_DEGREE", None))
    n.add_argument("--seed", type=int, default=int(_env("SEED", 0)))
    n.add_argument("--out", required=_env("OUT", None) is None, default=_env("OUT", None))
    o = ap.parse_args(argv)
    try:
        if o.cmd in ("bench", "sweep"):
            return cmd_bench(o, o.cmd == "sweep")
        if o.cmd == "cost":
            return cmd_cost(o)
        if o.cmd == "gradcheck":
            return cmd_gradcheck(o)
        if o.cmd == "gen":
            o.n, o.avg_degree = int(o.n), float(o.avg_degree)
            return cmd_gen(o)
    except UsageError as ex:
        print(f"error: {ex}", file=sys.stderr)
        return 2
    except Exception as ex:  # noqa: BLE001 -- sgnn_bench.cpp:383-388
        print(f"error: {ex}", file=sys.stderr)
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
