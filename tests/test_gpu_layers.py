"""GPU parity of the GCN scheme engine and the GAT engine against the oracle
(and through it the reference golden vectors).  Bars: float64 <= 1e-10 (the
reference's own cross-scheme bar, test_gcn.cpp:94-99), float32 <= 1e-4
(north star) under max_rel_diff (dense.hpp:303-316)."""
import itertools

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

SCHEMES = [(0, 0, 0), (0, 1, 0), (1, 0, 0), (1, 1, 0), (2, 2, 1)]


@pytest.fixture(scope="module")
def d():
    from paper_2308_12093_b200 import device

    return device


def cu(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    return (t.to(dtype) if dtype is not None else t).cuda()


def np_(t):
    return t.cpu().numpy()


def _adj(d, op, dtype, fmt="csc"):
    return d.Adjacency(op.n, op.n, cu(op.rows), cu(op.cols), cu(op.vals.astype(dtype)), fmt)


@pytest.mark.parametrize("mk", [(7, 5), (5, 9)])
def test_gcn_golden_every_scheme(d, golden, orc, mk):
    """Device GCN vs the reference's own outputs (tests/golden/gcn.npz)."""
    g = golden("gcn")
    m, k = mk
    op = orc.Operator(int(g["n"]), g["rows"], g["cols"], g["vals"])
    X, th, bi, G = (g[f"{nm}_{m}_{k}"] for nm in ("X", "theta", "bias", "G"))
    for (fw, bw, ca), fmt, fg in itertools.product(SCHEMES, ("csr", "csc"), (0, 1)):
        tag = f"{m}_{k}_{fw}{bw}_{1 if fmt == 'csr' else 2}_{fg}"
        A = _adj(d, op, np.float64, fmt)
        out, cache = d.gcn_forward(A, cu(X), cu(th), cu(bi), d.make_scheme(fw, bw, ca))
        dth, db, dx = d.gcn_backward(A, cu(G), cu(th), cache, bool(fg))
        assert orc.max_rel_diff(np_(out), g["out_" + tag]) < 1e-13, tag
        assert orc.max_rel_diff(np_(dth), g["dtheta_" + tag]) < 1e-12, tag
        assert orc.max_rel_diff(np_(db), g["dbias_" + tag]) < 1e-13, tag
        if fg:
            assert orc.max_rel_diff(np_(dx), g["dinput_" + tag]) < 1e-12, tag
        else:
            assert dx is None


@pytest.mark.parametrize("n,deg,m,k", [(2000, 7.0, 16, 8), (3000, 12.0, 40, 33),
                                       (1500, 5.0, 64, 128), (2708, 3.9, 1433, 16)])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_gcn_schemes_vs_oracle(d, orc, n, deg, m, k, dtype):
    _, s, t = orc.synthetic_graph(n, deg, n + m)
    op = orc.gcn_operator(n, s, t)
    X = orc.random_uniform(n, m, 11)
    th, bi = orc.gcn_params(m, k, 13)
    G = orc.random_uniform(n, k, 12)
    tol = 1e-10 if dtype == np.float64 else 1e-4
    ref = orc.gcn_layer(op, X, th, bi, (0, 0, 0), G, True)
    A = _adj(d, op, dtype)
    for sch in SCHEMES:
        out, cache = d.gcn_forward(A, cu(X.astype(dtype)), cu(th.astype(dtype)),
                                   cu(bi.astype(dtype)), d.make_scheme(*sch))
        dth, db, dx = d.gcn_backward(A, cu(G.astype(dtype)), cu(th.astype(dtype)), cache, True)
        for got, want in zip((out, dth, db, dx), ref):
            assert orc.max_rel_diff(np_(got).astype(np.float64), want) < tol, sch


def test_gcn_cache_semantics(d, orc):
    n, m, k = 50, 6, 4
    _, s, t = orc.synthetic_graph(n, 4.0, 3)
    op = orc.gcn_operator(n, s, t)
    A = _adj(d, op, np.float64)
    X, G = cu(orc.random_uniform(n, m, 1)), cu(orc.random_uniform(n, k, 3))
    th, bi = (cu(a) for a in orc.gcn_params(m, k, 2))
    _, cache = d.gcn_forward(A, X, th, bi, d.make_scheme(0, 0, 0))
    d.gcn_backward(A, G, th, cache, False)
    with pytest.raises(ValueError, match="cache already consumed"):
        d.gcn_backward(A, G, th, cache, False)
    # a failed backward still consumes the cache (gcn.hpp:137-138)
    _, cache = d.gcn_forward(A, X, th, bi, d.make_scheme(1, 1, 0))
    with pytest.raises(ValueError):
        d.gcn_backward(A, cu(orc.random_uniform(n, k + 1, 3)), th, cache, False)
    with pytest.raises(ValueError, match="cache already consumed"):
        d.gcn_backward(A, G, th, cache, False)
    # cached pair retains P (n x m), uncached retains X: same footprint
    _, c1 = d.gcn_forward(A, X, th, bi, d.make_scheme(2, 2, 1))
    _, c2 = d.gcn_forward(A, X, th, bi, d.make_scheme(1, 1, 0))
    assert c1.retained_bytes() == c2.retained_bytes() == 8 * n * m
    with pytest.raises(ValueError, match="input width"):
        d.gcn_forward(A, cu(orc.random_uniform(n, m + 1, 1)), th, bi, d.make_scheme(0, 0, 0))


def _pattern(d, pat):
    return d.Pattern(pat.n, cu(pat.rowptr), cu(pat.cols))


def test_gat_golden_every_level(d, golden, orc):
    g = golden("gat")
    n, h, k, beta = int(g["n"]), int(g["heads"]), int(g["k"]), float(g["beta"])
    p = d.Pattern(n, cu(g["rowptr"]), cu(g["cols"]))
    X, th, a_s, a_d, bi, G = (cu(g[nm]) for nm in ("X", "theta", "a_src", "a_dst", "bias", "G"))
    for level in range(4):
        out, cache = d.gat_forward(p, X, th, a_s, a_d, bi, h, beta, level)
        alpha, mask = cache.edge_values(p, th, a_s, a_d)
        assert cache.extra_bytes() == orc.gat_cache_footprint(
            ["none", "features", "node-attn", "full"][level], n, h, k, p.nnz, 8)
        dth, das, dad, db, dx = d.gat_backward(p, G, th, a_s, a_d, cache, True, beta)
        assert orc.max_rel_diff(np_(out), g[f"out_{level}"]) < 1e-13
        assert orc.max_rel_diff(np_(alpha), g[f"alpha_{level}"]) < 1e-14
        assert np.array_equal(np_(mask), g[f"mask_{level}"])
        for nm, got in (("dtheta", dth), ("da_src", das), ("da_dst", dad), ("dbias", db),
                        ("dinput", dx)):
            assert orc.max_rel_diff(np_(got), g[f"{nm}_{level}"]) < 1e-12, (level, nm)


@pytest.mark.parametrize("n,deg,m,h,k", [(800, 6.0, 20, 8, 8), (1200, 9.0, 50, 8, 64),
                                         (500, 4.0, 12, 3, 5), (300, 5.0, 16, 1, 33),
                                         (400, 7.0, 24, 2, 128), (256, 6.0, 10, 40, 4),
                                         (600, 8.0, 20, 8, 40), (500, 6.0, 12, 4, 12),
                                         (300, 40.0, 16, 2, 20), (700, 5.0, 24, 8, 128),
                                         (400, 6.0, 16, 8, 256), (300, 9.0, 12, 4, 512),
                                         (300, 6.0, 12, 1, 256), (300, 6.0, 12, 2, 256),
                                         (250, 5.0, 12, 1, 512)])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_gat_vs_oracle(d, orc, n, deg, m, h, k, dtype):
    _, s, t = orc.synthetic_graph(n, deg, n + h)
    pat = orc.gat_pattern(n, s, t)
    X = orc.random_uniform(n, m, 21)
    th, a_s, a_d, bi = orc.gat_params(m, h, k, 23)
    G = orc.random_uniform(n, h * k, 22)
    ref_out = orc.gat_forward(pat, X, th, a_s, a_d, bi, h, 0.2)
    ref = orc.gat_backward(pat, G, X, th, a_s, a_d, h, 0.2, True)
    tol = 1e-10 if dtype == np.float64 else 1e-4
    p = _pattern(d, pat)
    c = lambda a: cu(a.astype(dtype))  # noqa: E731
    for level in ("none", "features", "node-attn", "full"):
        out, cache = d.gat_forward(p, c(X), c(th), c(a_s), c(a_d), c(bi), h, 0.2, level)
        assert orc.max_rel_diff(np_(out).astype(np.float64), ref_out) < tol, level
        got = d.gat_backward(p, c(G), c(th), c(a_s), c(a_d), cache, True, 0.2)
        for nm, gv, rv in zip(("dth", "das", "dad", "db", "dx"), got, ref):
            assert orc.max_rel_diff(np_(gv).astype(np.float64), rv) < tol, (level, nm)


def test_gat_errors(d, orc):
    r, c = np.array([0, 0], np.int32), np.array([0, 1], np.int32)
    p = d.Pattern(2, cu(orc.coo_to_csr(2, r)), cu(c))
    th, a_s, a_d, bi = (cu(x) for x in orc.gat_params(3, 1, 2, 142))
    X = cu(orc.random_uniform(2, 3, 141))
    with pytest.raises(ValueError, match="self loops"):
        d.gat_forward(p, X, th, a_s, a_d, bi, 1, 0.2)
    _, s, t = orc.synthetic_graph(4, 2.0, 1)
    pat = orc.gat_pattern(4, s, t)
    p = _pattern(d, pat)
    X4 = cu(orc.random_uniform(4, 3, 144))
    with pytest.raises(ValueError, match="beta must be positive"):
        d.gat_forward(p, X4, th, a_s, a_d, bi, 1, -0.5)
    _, cache = d.gat_forward(p, X4, th, a_s, a_d, bi, 1, 0.2)
    G = cu(orc.random_uniform(4, 2, 145))
    d.gat_backward(p, G, th, a_s, a_d, cache, False)
    with pytest.raises(ValueError, match="cache already consumed"):
        d.gat_backward(p, G, th, a_s, a_d, cache, False)


def test_gat_rows_sum_to_one_and_single_node(d, orc):
    _, s, t = orc.synthetic_graph(300, 8.0, 4)
    pat = orc.gat_pattern(300, s, t)
    p = _pattern(d, pat)
    th, a_s, a_d, bi = (cu(x) for x in orc.gat_params(5, 4, 2, 123))
    X = cu(orc.random_uniform(300, 5, 122))
    _, cache = d.gat_forward(p, X, th, a_s, a_d, bi, 4, 0.2, "full")
    alpha, _ = cache.edge_values(p, th, a_s, a_d)
    sums = np.add.reduceat(np_(alpha), pat.rowptr[:-1], axis=1)
    assert np.abs(sums - 1.0).max() <= 1e-12
    # one node with only a self loop: X' = X Theta + b (test_gat.cpp:32-41)
    p1 = d.Pattern(1, cu(np.array([0, 1], np.int32)), cu(np.array([0], np.int32)))
    X1 = orc.random_uniform(1, 4, 3)
    th1, as1, ad1, b1 = orc.gat_params(4, 2, 3, 4)
    out, _ = d.gat_forward(p1, cu(X1), cu(th1), cu(as1), cu(ad1), cu(b1), 2)
    assert orc.max_rel_diff(np_(out), X1 @ th1 + b1) < 1e-15


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("fg", [0, 1])
def test_step_host_matches_device_path(d, orc, dtype, fg):
    """gcn/gat_step_host (host buffers, overlapped copies) give exactly the
    device-path results: same kernels, only the transfers differ."""
    n, m, k, h, kk = 1800, 24, 40, 4, 8
    _, s, t = orc.synthetic_graph(n, 9.0, 3)
    src, dst = torch.from_numpy(s), torch.from_numpy(t)
    A = d.Adjacency.gcn_operator(n, src, dst, dtype, "csc")
    X = torch.rand(n, m, dtype=dtype) * 2 - 1
    G = torch.rand(n, k, dtype=dtype) * 2 - 1
    th, bi = d.gcn_params(m, k, 13, dtype=dtype)
    for policy in ("adaptive", "transform-first", "propagate-first"):
        sch = d.resolve_scheme(policy, m, k, bool(fg), True)
        out, cache = d.gcn_forward(A, X.cuda(), th, bi, sch)
        ref = (out,) + d.gcn_backward(A, G.cuda(), th, cache, bool(fg))
        pin = lambda *sh: torch.empty(sh, dtype=dtype).pin_memory()  # noqa: E731
        ho, hth, hb, hx = pin(n, k), pin(m, k), pin(k), pin(n, m)
        d.gcn_step_host(A, X.pin_memory(), th, bi, sch, G.pin_memory(), bool(fg), ho, hth, hb,
                        hx if fg else None)
        A.ctx.synchronize()
        got = (ho, hth, hb, hx if fg else None)
        for a, b in zip(got, ref):
            if b is None:
                continue
            assert torch.equal(a, b.cpu()), policy
    P = d.Pattern.gat_pattern(n, src, dst)
    th2, a_s, a_d, b2 = d.gat_params(m, h, kk, 23, dtype=dtype)
    G2 = torch.rand(n, h * kk, dtype=dtype) * 2 - 1
    for level in ("none", "full"):
        o, c = d.gat_forward(P, X.cuda(), th2, a_s, a_d, b2, h, 0.2, level)
        ref = (o,) + d.gat_backward(P, G2.cuda(), th2, a_s, a_d, c, bool(fg))
        pin = lambda *sh: torch.empty(sh, dtype=dtype).pin_memory()  # noqa: E731
        hs = (pin(n, h * kk), pin(m, h * kk), pin(h, kk), pin(h, kk), pin(h * kk), pin(n, m))
        d.gat_step_host(P, X.pin_memory(), th2, a_s, a_d, b2, h, 0.2, level, G2.pin_memory(),
                        bool(fg), *hs[:5], hs[5] if fg else None)
        P.ctx.synchronize()
        for a, b in zip(hs, ref):
            if b is None:
                continue
            assert torch.equal(a, b.cpu()), level


def test_step_graph_replay_is_bit_identical(d, orc):
    """A GCN + GAT fwd+bwd step captured into a CUDA graph (device.StepGraph)
    replays to exactly the eager results."""
    n, m, k = 3000, 32, 64
    _, s, t = orc.synthetic_graph(n, 9.0, 4)
    src, dst = torch.from_numpy(s), torch.from_numpy(t)
    A = d.Adjacency.gcn_operator(n, src, dst, torch.float32, "csc")
    P = d.Pattern.gat_pattern(n, src, dst)
    X = d.random_uniform(n, m, 1)
    G = d.random_uniform(n, k, 2)
    th, b = d.gcn_params(m, k, 3)
    tg, a_s, a_d, bg = d.gat_params(m, 8, 8, 4)
    sch = d.resolve_scheme("adaptive", m, k, True, True)

    def step():
        out, c = d.gcn_forward(A, X, th, b, sch)
        o2, c2 = d.gat_forward(P, X, tg, a_s, a_d, bg, 8, 0.2, "full")
        return (out,) + d.gcn_backward(A, G, th, c, True) + (o2,) + \
            d.gat_backward(P, G, tg, a_s, a_d, c2, True)

    ref = step()
    g = d.StepGraph(step)
    for _ in range(2):
        got = g.replay()
    torch.cuda.synchronize()
    for a, r in zip(got, ref):
        assert torch.equal(a, r)
