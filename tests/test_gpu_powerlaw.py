"""Device Chung-Lu power-law generator (sgnn_powerlaw_graph): the
synthetic_graph output contract (undirected, both directions, no self loops,
no duplicates, canonical order), determinism, agreement with a numpy
restatement of the same draws, and the layers on a hub-heavy graph against
the oracle."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

MASK = (1 << 64) - 1


def _mix(seed, i):
    z = (seed + (i + 2) * 0x9E3779B97F4A7C15) & MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return z ^ (z >> 31)


def _numpy_powerlaw(n, deg, gamma, seed):
    w = np.arange(1, n + 1, dtype=np.float64) ** (-1.0 / (gamma - 1.0))
    cdf = np.cumsum(w)
    pairs = int(round(deg * n / 2.0))
    edges = set()
    for p in range(pairs):
        u1 = (_mix(seed, 2 * p) >> 11) * 2.0 ** -53 * cdf[-1]
        u2 = (_mix(seed, 2 * p + 1) >> 11) * 2.0 ** -53 * cdf[-1]
        a, b = int(np.searchsorted(cdf, u1, side="right")), int(np.searchsorted(cdf, u2, side="right"))
        if a != b:
            edges.add((min(a, b), max(a, b)))
    return edges


def test_powerlaw_contract_and_numpy_restatement():
    from paper_2308_12093_b200 import device as d

    n, deg, gamma, seed = 3000, 8.0, 2.5, 7
    s, t = d.powerlaw_graph(n, deg, gamma, seed)
    s2, t2 = d.powerlaw_graph(n, deg, gamma, seed)
    assert torch.equal(s, s2) and torch.equal(t, t2)
    s, t = s.cpu().numpy().astype(np.int64), t.cpu().numpy().astype(np.int64)
    key = s * n + t
    assert np.all(np.diff(key) > 0)           # canonical order, no duplicates
    assert np.all(s != t)                      # no self loops
    assert set(zip(s.tolist(), t.tolist())) == set(zip(t.tolist(), s.tolist()))  # symmetric
    got = {(a, b) for a, b in zip(s.tolist(), t.tolist()) if a < b}
    want = _numpy_powerlaw(n, deg, gamma, seed)
    # the device prefix sum folds in a different order than np.cumsum: a draw
    # landing within an ulp of a bucket edge may differ
    assert len(got ^ want) <= max(2, len(want) // 1000)
    degs = np.bincount(s, minlength=n)
    assert degs.max() > 20 * np.median(degs)   # heavy tail


def test_layers_on_powerlaw_graph_vs_oracle(orc):
    from paper_2308_12093_b200 import device as d

    n, m, k = 4000, 24, 40
    s, t = d.powerlaw_graph(n, 12.0, 2.2, 3)
    sh, th = s.cpu().numpy(), t.cpu().numpy()
    assert np.bincount(sh, minlength=n).max() > 300  # rows longer than any fast-path batch
    op = orc.gcn_operator(n, sh, th)
    X = orc.random_uniform(n, m, 11)
    theta, bias = orc.gcn_params(m, k, 13)
    G = orc.random_uniform(n, k, 12)
    A = d.Adjacency.gcn_operator(n, s, t, torch.float32, "csc")
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()  # noqa: E731
    for pol in ("transform-first", "propagate-first"):
        sch = d.resolve_scheme(pol, m, k, True, pol == "propagate-first")
        out, c = d.gcn_forward(A, cu(X), cu(theta), cu(bias), sch)
        got = (out,) + d.gcn_backward(A, cu(G), cu(theta), c, True)
        ref = orc.gcn_layer(op, X, theta, bias, (sch.forward, sch.backward, sch.caching), G, True)
        for a, b in zip(got, ref):
            assert orc.max_rel_diff(a.cpu().numpy().astype(np.float64), b) < 1e-4, pol


# hub rows on every SDDMM reduction mode: power-of-two heads (8x8), heads of
# two whole 32-lane chunks (4x256), shared-memory fold (8x40)
@pytest.mark.parametrize("h,kk", [(8, 8), (4, 256), (8, 40)])
def test_gat_on_powerlaw_graph_vs_oracle(orc, h, kk):
    from paper_2308_12093_b200 import device as d

    n, m = 4000, 24
    s, t = d.powerlaw_graph(n, 12.0, 2.2, 3)
    sh, th = s.cpu().numpy(), t.cpu().numpy()
    X = orc.random_uniform(n, m, 11)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()  # noqa: E731
    pat = orc.gat_pattern(n, sh, th)
    P = d.Pattern.gat_pattern(n, s, t)
    tg, a_s, a_d, bg = orc.gat_params(m, h, kk, 21)
    G2 = orc.random_uniform(n, h * kk, 22)
    o, c = d.gat_forward(P, cu(X), cu(tg), cu(a_s), cu(a_d), cu(bg), h, 0.2, "full")
    g2 = d.gat_backward(P, cu(G2), cu(tg), cu(a_s), cu(a_d), c, True)
    ro = orc.gat_forward(pat, X, tg, a_s, a_d, bg, h, 0.2)
    rg = orc.gat_backward(pat, G2, X, tg, a_s, a_d, h, 0.2, True)
    for a, b in zip((o,) + tuple(g2), (ro,) + tuple(rg)):
        assert orc.max_rel_diff(a.cpu().numpy().astype(np.float64), b) < 1e-4


@pytest.mark.parametrize("f", [24, 47, 128, 300])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_spmm_hub_rows_vs_oracle(orc, f, dtype):
    """Rows longer than the hub threshold run as segments + in-order combine
    (lean, windowed and generic paths, both directions)."""
    from paper_2308_12093_b200 import device as d

    n = 3000
    s, t = d.powerlaw_graph(n, 10.0, 2.1, 5)
    sh, th = s.cpu().numpy(), t.cpu().numpy()
    assert np.bincount(sh, minlength=n).max() > 500  # several 128-edge segments
    op = orc.gcn_operator(n, sh, th)
    A = d.Adjacency.gcn_operator(n, s, t, dtype, "csc")
    B = orc.random_uniform(n, f, 9)
    Bt = torch.from_numpy(B).to("cuda", dtype)
    ref = orc.spmm_csr(op.rowptr, op.cols, op.vals, B)
    tol = 1e-5 if dtype == torch.float32 else 1e-13
    for tr in (False, True):
        got = A.spmm(Bt, transposed=tr).double().cpu().numpy()
        assert orc.max_rel_diff(got, ref) < tol, tr  # the operator is symmetric


@pytest.mark.parametrize("f", [47, 5, 130])
def test_unaligned_widths_bit_identical(orc, f):
    """float32 widths that are not a multiple of 4 (config 5's 47 classes)
    run the vector kernels on a 16-byte-aligned padded copy of B (products
    with >= 2^20 nonzeros): still bit-identical to the reference's in-order
    accumulation (the float32 oracle), both directions, bias added last."""
    from paper_2308_12093_b200 import device as d

    n = 140000  # uniform graph: every row below the hub threshold keeps the stored order
    s, t = d.synthetic_graph(n, 8.0, 5)
    sh, th = s.cpu().numpy(), t.cpu().numpy()
    op = orc.gcn_operator(n, sh, th)
    A = d.Adjacency.gcn_operator(n, s, t, torch.float32, "csr")
    assert A.nnz >= 1 << 20
    B = orc.random_uniform(n, f, 3).astype(np.float32)
    bias = orc.random_uniform(1, f, 4).astype(np.float32).reshape(-1)
    Bt, bt = torch.from_numpy(B).cuda(), torch.from_numpy(bias).cuda()
    ref = orc.spmm_csr(op.rowptr, op.cols, op.vals.astype(np.float32), B)
    assert np.array_equal(A.spmm(Bt, bias=bt).cpu().numpy(), ref + bias)
    assert np.array_equal(A.spmm(Bt, transposed=True).cpu().numpy(), ref)  # symmetric operator
