"""GPU parity: sparse-format layer and kernels vs the oracle / golden vectors.
Bar: bit-exact for indices, formats, normalized values and (unfused, stored
order) SpMM/SDDMM; documented tolerances for GEMM and softmax."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def d():
    from paper_2308_12093_b200 import device

    return device


def cu(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def np_(t):
    return t.cpu().numpy()


def test_canonicalize_csr_csc_bit_exact(d, golden):
    g = golden("sparse")
    nr, nc = int(g["n_rows"]), int(g["n_cols"])
    r, c, v = d.canonicalize(nr, nc, cu(g["in_rows"]), cu(g["in_cols"]), cu(g["in_vals"]))
    assert np.array_equal(np_(r), g["canon_rows"]) and np.array_equal(np_(c), g["canon_cols"])
    assert np.array_equal(np_(v), g["canon_vals"])  # keep-last duplicates
    assert np.array_equal(np_(d.csr_from_coo(nr, r)), g["rowptr"])
    cp, cr, cv, perm = d.csc_from_coo(nc, r, c, v)
    assert np.array_equal(np_(cp), g["colptr"]) and np.array_equal(np_(cr), g["csc_rows"])
    assert np.array_equal(np_(cv), g["csc_vals"])


def test_canonicalize_errors_and_empty(d):
    with pytest.raises(ValueError, match="index out of range"):
        d.canonicalize(3, 3, cu(np.array([0, 3], np.int32)), cu(np.array([0, 1], np.int32)),
                       cu(np.ones(2)))
    r, c, v = d.canonicalize(5, 5, cu(np.zeros(0, np.int32)), cu(np.zeros(0, np.int32)),
                             cu(np.zeros(0)))
    assert r.numel() == 0
    assert np.array_equal(np_(d.csr_from_coo(5, r)), np.zeros(6, np.int32))


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_gcn_normalize_bit_exact(d, golden, dtype):
    g = golden("sparse")
    n = int(g["norm_n"])
    r, c, v = d.canonicalize(n, n, cu(g["norm_in_rows"]), cu(g["norm_in_cols"]),
                             cu(g["norm_in_vals"].astype(dtype)))
    r, c, v = d.gcn_normalize(n, r, c, v)
    assert np.array_equal(np_(r), g["norm_rows"]) and np.array_equal(np_(c), g["norm_cols"])
    ref = g["norm_vals"] if dtype == np.float64 else g["norm_vals_f32"]
    assert np.array_equal(np_(v), ref)


def test_gcn_normalize_negative_weight(d):
    r, c, v = d.canonicalize(2, 2, cu(np.array([0, 1], np.int32)), cu(np.array([1, 0], np.int32)),
                             cu(np.array([1.0, -1.0])))
    with pytest.raises(ValueError, match="negative edge weight"):
        d.gcn_normalize(2, r, c, v)


def test_pattern_bit_exact(d, golden):
    g = golden("pattern")
    for s in ("0", "1"):
        p = d.Pattern(50, cu(g["rowptr" + s]), cu(g["cols" + s]))
        a = p.arrays()
        for nm in ("colptr", "rows", "perm", "diag"):
            assert np.array_equal(np_(a[nm]), g[nm + s]), (s, nm)
        assert p.all_self_loops == bool(g["all" + s])


@pytest.mark.parametrize("fmt", ["coo", "csr", "csc", "ellpack", "hybrid"])
def test_spmm_bit_exact_f64_every_format(d, golden, fmt):
    g = golden("kernels")
    nr, nc = int(g["n_rows"]), int(g["n_cols"])
    A = d.Adjacency.from_coo(nr, nc, cu(g["rows"]), cu(g["cols"]), cu(g["vals"]), fmt)
    assert np.array_equal(np_(A.spmm(cu(g["B"]))), g["C_" + fmt])


def test_spmm_bit_exact_f32(d, golden):
    g = golden("kernels")
    nr, nc = int(g["n_rows"]), int(g["n_cols"])
    A = d.Adjacency.from_coo(nr, nc, cu(g["rows"]), cu(g["cols"]),
                             cu(g["vals"].astype(np.float32)), "csr")
    assert np.array_equal(np_(A.spmm(cu(g["B32"]))), g["C32"])


@pytest.mark.parametrize("f", [1, 3, 4, 8, 16, 33, 64, 128, 200, 256, 1024, 1100])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_spmm_widths_and_transpose_vs_oracle(d, orc, f, dtype):
    n = 300
    _, s, t = orc.synthetic_graph(n, 9.0, f)
    op = orc.gcn_operator(n, s, t)
    B = orc.random_uniform(n, f, 7 + f).astype(dtype)
    bias = orc.random_uniform(1, f, 3).ravel().astype(dtype)
    A = d.Adjacency(n, n, cu(op.rows), cu(op.cols), cu(op.vals.astype(dtype)), "csc")
    got = np_(A.spmm(cu(B)))
    ref = orc.spmm_csr(op.rowptr, op.cols, op.vals.astype(dtype), B)
    assert np.array_equal(got, ref)  # stored-order, unfused: bit-exact in both precisions
    got_b = np_(A.spmm(cu(B), bias=cu(bias)))
    assert np.array_equal(got_b, (ref + bias).astype(dtype))
    got_t = np_(A.spmm(cu(B), transposed=True))
    ref_t = orc.spmm_csr(op.colptr, op.crows, op.cvals.astype(dtype), B)
    assert np.array_equal(got_t, ref_t)


def test_spmm_rectangular_and_empty_rows(d, orc):
    rng = np.random.default_rng(3)
    nr, nc, q = 97, 41, 300
    r = rng.integers(0, nr // 2, q).astype(np.int32)  # upper half of rows empty
    c = rng.integers(0, nc, q).astype(np.int32)
    v = rng.standard_normal(q)
    B = rng.standard_normal((nc, 12))
    rr, cc, vv = orc.coo_canonicalize(nr, nc, r, c, v)
    A = d.Adjacency.from_coo(nr, nc, cu(r), cu(c), cu(v), "csr")
    ref = orc.spmm_csr(orc.coo_to_csr(nr, rr), cc, vv, B)
    assert np.array_equal(np_(A.spmm(cu(B))), ref)
    with pytest.raises(ValueError):
        A.spmm(cu(rng.standard_normal((nc + 1, 3))))


def test_sddmm_and_edge_softmax(d, golden, orc):
    g = golden("kernels")
    n = int(g["sddmm_n"])
    r, c, _ = d.canonicalize(n, n, cu(g["sddmm_rows"]), cu(g["sddmm_cols"]),
                             cu(np.ones(len(g["sddmm_rows"]))))
    p = d.Pattern(n, d.csr_from_coo(n, r), c)
    out = np_(d.sddmm(p, cu(g["sddmm_B"]), cu(g["sddmm_C"])))
    assert np.array_equal(out, g["sddmm_vals"])
    r, c, _ = d.canonicalize(n, n, cu(g["softmax_rows"]), cu(g["softmax_cols"]),
                             cu(np.ones(len(g["softmax_rows"]))))
    p = d.Pattern(n, d.csr_from_coo(n, r), c)
    alpha = np_(d.edge_softmax(p, cu(g["softmax_scores"])))
    assert np.all(np.isfinite(alpha))
    assert orc.max_rel_diff(alpha, g["softmax_alpha"]) < 1e-14  # exp() within 1 ulp


def test_edge_softmax_requires_self_loops(d):
    r, c, _ = d.canonicalize(2, 2, cu(np.array([0, 1], np.int32)), cu(np.array([1, 1], np.int32)),
                             cu(np.ones(2)))
    p = d.Pattern(2, d.csr_from_coo(2, r), c)
    assert not p.all_self_loops
    with pytest.raises(ValueError, match="self loops"):
        d.edge_softmax(p, cu(np.zeros(2)))


# (20000, 256, 320): 160-wide tiles (two per row block), split-K dTheta shape;
# (5000, 96, 300): 160-wide tiles with a ragged last tile; stored widths that
# are not multiples of 4 (Cora's 1433 features) run on tcgen05 from padded
# staging copies: (2708, 1433, 16) pads K, (3000, 64, 1433) pads N (and K
# with tb), (1433, 2708, 16) with ta pads M (the dTheta shape); one tiny
# dimension (skinny.cu): (20000, 128, 8) narrow N, (128, 20000, 8) with ta the
# narrow dTheta, (20000, 8, 128) thin K, (8000, 1433, 16) Cora-wide K
@pytest.mark.parametrize("shape", [(1000, 7, 5), (300, 128, 256), (4096, 64, 40), (70000, 16, 8),
                                   (20000, 256, 320), (5000, 96, 300), (2708, 1433, 16),
                                   (3000, 64, 1433), (1433, 2708, 16), (20000, 128, 8),
                                   (128, 20000, 8), (20000, 8, 128), (8000, 1433, 16),
                                   (16, 9000, 4)])
@pytest.mark.parametrize("trans", [(False, False), (True, False), (False, True)])
def test_gemm_vs_oracle(d, orc, shape, trans):
    n, m, k = shape
    ta, tb = trans
    # build operands so that op(A) is n x m, op(B) is m x k
    A = orc.random_uniform(m, n, 1) if ta else orc.random_uniform(n, m, 1)
    B = orc.random_uniform(k, m, 2) if tb else orc.random_uniform(m, k, 2)
    ref = orc.gemm(A, B, ta, tb)
    got64 = np_(d.gemm(cu(A), cu(B), ta, tb))
    assert orc.max_rel_diff(got64, ref) < 1e-12
    got32 = np_(d.gemm(cu(A.astype(np.float32)), cu(B.astype(np.float32)), ta, tb))
    assert orc.max_rel_diff(got32, ref) < 1e-4  # north-star fp32 bar


def test_column_sums(d, orc):
    X = orc.random_uniform(169343, 37, 5)
    ref = orc.column_sums(X)
    assert orc.max_rel_diff(np_(d.column_sums(cu(X))), ref) < 1e-12
    assert orc.max_rel_diff(np_(d.column_sums(cu(X.astype(np.float32)))), ref) < 1e-5


def test_random_uniform_bit_exact(d, golden, orc):
    g = golden("rng")
    assert np.array_equal(np_(d.random_uniform(7, 5, 42, dtype=torch.float64)), g["u_7x5_s42"])
    assert np.array_equal(np_(d.random_uniform(3, 11, 0, -2, 2, dtype=torch.float64)),
                          g["u_3x11_s0_pm2"])
    assert np.array_equal(np_(d.random_uniform(123, 77, 9, dtype=torch.float32)),
                          orc.random_uniform(123, 77, 9, dtype=np.float32))
    th, b = d.gcn_params(33, 17, 13, dtype=torch.float64)
    oth, ob = orc.gcn_params(33, 17, 13)
    assert np.array_equal(np_(th), oth) and np.array_equal(np_(b), ob)
    th, a_s, a_d, b = d.gat_params(9, 3, 5, 23, dtype=torch.float64)
    for got, ref in zip((th, a_s, a_d, b), orc.gat_params(9, 3, 5, 23)):
        assert np.array_equal(np_(got), ref)


# fused (per-chunk heads): 8x32; fused (heads ending mid-chunk): 8x40, 8x20,
# 4x40, 8x16; separate score kernel (heads do not divide the tile): 8x12, 2x40,
# and heads wider than a tile (k = 128 LPW, 4 items per warp): 2x256, 8x256, 1x512
@pytest.mark.parametrize("hk", [(8, 32), (8, 40), (8, 20), (4, 40), (8, 16), (8, 12), (2, 40),
                                (2, 256), (8, 256), (1, 512)])
def test_gat_transform_scores(d, orc, hk):
    """sgnn_gat_transform: M = X Theta with the node scores (kernels.hpp:385-423)
    fused into the GEMM epilogue when whole heads fit a tile (k % 4 == 0), else
    the separate score kernel -- both against float64 numpy."""
    from paper_2308_12093_b200 import _capi as capi
    h, k = hk
    n, m = 9000, 96
    X = orc.random_uniform(n, m, 3).astype(np.float32)
    th = orc.random_uniform(m, h * k, 4).astype(np.float32)
    a_s = orc.random_uniform(h, k, 5).astype(np.float32)
    a_d = orc.random_uniform(h, k, 6).astype(np.float32)
    Xc, thc, asc, adc = cu(X), cu(th), cu(a_s), cu(a_d)
    M = torch.empty((n, h * k), dtype=torch.float32, device="cuda")
    s = torch.empty((n, h), dtype=torch.float32, device="cuda")
    dd = torch.empty((n, h), dtype=torch.float32, device="cuda")
    ctx = d.Context.default()
    capi.check(capi.lib.sgnn_gat_transform(ctx.handle, Xc.data_ptr(), n, m, thc.data_ptr(), h, k,
                                           asc.data_ptr(), adc.data_ptr(), M.data_ptr(),
                                           s.data_ptr(), dd.data_ptr()))
    Mr = X.astype(np.float64) @ th.astype(np.float64)
    sr = np.einsum("ntc,tc->nt", Mr.reshape(n, h, k), a_s.astype(np.float64))
    dr = np.einsum("ntc,tc->nt", Mr.reshape(n, h, k), a_d.astype(np.float64))
    assert orc.max_rel_diff(np_(M), Mr) < 1e-4
    assert orc.max_rel_diff(np_(s), sr) < 1e-4
    assert orc.max_rel_diff(np_(dd), dr) < 1e-4


def test_unaligned_widths_run_on_tensor_cores(d, orc):
    """Cora's X (2708 x 1433, fp32): the 5732-byte row pitch is staged into
    zero-padded copies for the TMA / tcgen05 GEMM (pad A, pad B, Theta hi/lo
    split, GEMM) instead of the one-launch SIMT fallback."""
    A = cu(orc.random_uniform(2708, 1433, 1).astype(np.float32))
    B = cu(orc.random_uniform(1433, 16, 2).astype(np.float32))
    ctx = d.Context.default()
    c0 = ctx.launch_count
    d.gemm(A, B)
    assert ctx.launch_count - c0 >= 3
