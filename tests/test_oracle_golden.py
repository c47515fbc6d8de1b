"""Pin the C oracle (oracle/sgnn_oracle.c) to golden vectors the REFERENCE
produced (oracle/gen_golden.py over oracle/_ref).  CPU only.

Bar: bit-exact (np.array_equal) for integers, indices, scheme choices and
every float64 value -- the oracle restates the reference loops in the same
order without FP contraction, so it is the reference, restated.
"""
import itertools

import numpy as np
import pytest


def test_rng_streams(golden, orc):
    g = golden("rng")
    assert np.array_equal(orc.random_uniform(7, 5, 42), g["u_7x5_s42"])
    assert np.array_equal(orc.random_uniform(3, 11, 0, -2, 2), g["u_3x11_s0_pm2"])
    assert np.array_equal(orc.random_uniform(1, 1000, 99, 0.0, 1.0), g["u_1x1000_s99"])


@pytest.mark.parametrize("n,deg,seed,tag", [(500, 6.0, 7, "500_6_7"),
                                            (2708, 10556 / 2708, 1, "cora_1"),
                                            (97, 3.3, 123, "97_3p3_123")])
def test_synthetic_graph(golden, orc, n, deg, seed, tag):
    g = golden("synthetic_graph")
    _, s, d = orc.synthetic_graph(n, deg, seed)
    assert np.array_equal(s, g["src_" + tag]) and np.array_equal(d, g["dst_" + tag])
    assert not np.any(s == d)


def test_canonicalize_keep_last_and_formats(golden, orc):
    g = golden("sparse")
    nr, nc = int(g["n_rows"]), int(g["n_cols"])
    r, c, v = orc.coo_canonicalize(nr, nc, g["in_rows"], g["in_cols"], g["in_vals"])
    assert np.array_equal(r, g["canon_rows"]) and np.array_equal(c, g["canon_cols"])
    assert np.array_equal(v, g["canon_vals"])
    assert np.array_equal(orc.coo_to_csr(nr, r), g["rowptr"])
    cp, cr, cv, perm = orc.coo_to_csc(nc, r, c, v)
    assert np.array_equal(cp, g["colptr"]) and np.array_equal(cr, g["csc_rows"])
    assert np.array_equal(cv, g["csc_vals"])
    assert np.array_equal(cv, v[perm])


def test_canonicalize_range_error(orc):
    with pytest.raises(ValueError):
        orc.coo_canonicalize(3, 3, [0, 3], [0, 1], [1.0, 1.0])


def test_gcn_normalize_bit_exact(golden, orc):
    g = golden("sparse")
    n = int(g["norm_n"])
    r, c, v = orc.coo_canonicalize(n, n, g["norm_in_rows"], g["norm_in_cols"],
                                   g["norm_in_vals"])
    nr_, nc_, nv_ = orc.gcn_normalize(n, r, c, v)
    assert np.array_equal(nr_, g["norm_rows"]) and np.array_equal(nc_, g["norm_cols"])
    assert np.array_equal(nv_, g["norm_vals"])
    _, _, nv32 = orc.gcn_normalize(n, r, c, v.astype(np.float32), dtype=np.float32)
    assert np.array_equal(nv32, g["norm_vals_f32"])


def test_gcn_normalize_known_answer(orc):
    # path 0-1-2: degrees with self loops [2,3,2]; (0,1) = 1/sqrt(6) (test_sparse.cpp:146-158)
    r, c, v = orc.gcn_normalize(3, [0, 1, 1, 2], [1, 0, 2, 1], np.ones(4))
    idx = int(np.nonzero((r == 0) & (c == 1))[0][0])
    assert v[idx] == 1.0 / np.sqrt(6.0)
    assert np.array_equal(orc.coo_to_csr(3, [0, 1, 1, 2]), [0, 1, 3, 4])


def test_pattern_build(golden, orc):
    g = golden("pattern")
    for s in ("0", "1"):
        cp, rows, perm, diag, flag = orc.pattern_build(50, g["rowptr" + s], g["cols" + s])
        assert np.array_equal(cp, g["colptr" + s]) and np.array_equal(rows, g["rows" + s])
        assert np.array_equal(perm, g["perm" + s]) and np.array_equal(diag, g["diag" + s])
        assert flag == bool(g["all" + s])


def test_spmm_all_formats_and_f32(golden, orc):
    g = golden("kernels")
    nr, nc = int(g["n_rows"]), int(g["n_cols"])
    r, c, v = orc.coo_canonicalize(nr, nc, g["rows"], g["cols"], g["vals"])
    rp = orc.coo_to_csr(nr, r)
    C = orc.spmm_csr(rp, c, v, g["B"])
    for fmt in ("coo", "csr", "csc", "ellpack", "hybrid"):
        assert np.array_equal(C, g["C_" + fmt]), fmt  # all formats: same per-row order
    C32 = orc.spmm_csr(rp, c, v.astype(np.float32), g["B32"])
    assert np.array_equal(C32, g["C32"])


def test_sddmm_and_softmax(golden, orc):
    g = golden("kernels")
    n = int(g["sddmm_n"])
    r, c, _ = orc.coo_canonicalize(n, n, g["sddmm_rows"], g["sddmm_cols"],
                                   np.ones(len(g["sddmm_rows"])))
    rp = orc.coo_to_csr(n, r)
    assert np.array_equal(orc.sddmm(rp, c, g["sddmm_B"], g["sddmm_C"]), g["sddmm_vals"])
    r, c, _ = orc.coo_canonicalize(n, n, g["softmax_rows"], g["softmax_cols"],
                                   np.ones(len(g["softmax_rows"])))
    rp = orc.coo_to_csr(n, r)
    alpha = orc.edge_softmax(rp, g["softmax_scores"][None, :])[0]
    assert np.array_equal(alpha, g["softmax_alpha"])
    assert np.all(np.isfinite(alpha))


def test_selector_full_grid(golden, orc):
    g = golden("cost")
    sel = g["select"]
    for pi, (mi, m) in itertools.product(range(3), enumerate(g["ms"])):
        for ki, k in enumerate(g["ks"]):
            for fg in (0, 1):
                for ca in (0, 1):
                    got = orc.resolve_scheme(pi, int(m), int(k), fg, ca)
                    assert tuple(sel[pi, mi, ki, fg, ca]) == got, (pi, m, k, fg, ca)
    with pytest.raises(ValueError):
        orc.resolve_scheme(0, 0, 4)


def test_cost_formulas(golden, orc):
    g = golden("cost")
    names = ["coo", "csr", "csc", "ellpack"]
    for row in g["costs"]:
        fn_i, n, q, p, fmt, f, sb, rc, fl, by, oi = row
        fn = orc.spmm_cost if fn_i == 0 else orc.sddmm_cost
        if rc != 0:
            with pytest.raises(ValueError):
                fn(names[int(fmt)], int(n), int(q), int(p), int(f), int(sb))
            continue
        got = fn(names[int(fmt)], int(n), int(q), int(p), int(f), int(sb))
        assert (got["flops"], got["bytes"]) == (int(fl), int(by))
        assert got["operational_intensity"] == oi
    # published intensities (PAPER Table 6, test_smoke.py:34-40)
    assert abs(orc.spmm_cost("csr", 2708, 10556, f=64)["operational_intensity"] - 0.621) <= .005
    assert orc.gat_cache_footprint("full", 3, 2, 4, 5) == 146


def _gcn_op(orc, g):
    return orc.Operator(int(g["n"]), g["rows"], g["cols"], g["vals"])


@pytest.mark.parametrize("mk", [(7, 5), (5, 9)])
def test_gcn_layer_all_schemes(golden, orc, mk):
    g = golden("gcn")
    m, k = mk
    op = _gcn_op(orc, g)
    X, th, bi, G = (g[f"{nm}_{m}_{k}"] for nm in ("X", "theta", "bias", "G"))
    for (fw, bw, ca) in [(0, 0, 0), (0, 1, 0), (1, 0, 0), (1, 1, 0), (2, 2, 1)]:
        for fmt in (1, 2):  # csr and csc store the same per-row order
            for fg in (0, 1):
                tag = f"{m}_{k}_{fw}{bw}_{fmt}_{fg}"
                out, dth, db, dx = orc.gcn_layer(op, X, th, bi, (fw, bw, ca), G, fg)
                assert np.array_equal(out, g["out_" + tag]), tag
                assert np.array_equal(dth, g["dtheta_" + tag]), tag
                assert np.array_equal(db, g["dbias_" + tag]), tag
                if fg:
                    assert np.array_equal(dx, g["dinput_" + tag]), tag


def test_gcn_cora_config1(golden, orc):
    g = golden("gcn_cora")
    sg = golden("synthetic_graph")
    op = orc.gcn_operator(2708, sg["src_cora_1"], sg["dst_cora_1"])
    assert op.nnz == int(g["nnz"]) == 13264
    assert np.array_equal(op.vals[::13], g["norm_vals_sample"])
    X = orc.random_uniform(2708, 1433, 11)
    th, bi = orc.gcn_params(1433, 16, 13)
    G = orc.random_uniform(2708, 16, 12)
    sch = orc.resolve_scheme(0, 1433, 16, True, True)
    assert tuple(g["scheme"]) == sch == (0, 0, 0)  # caching on still picks TF/fused
    out, dth, db, dx = orc.gcn_layer(op, X, th, bi, sch, G, True)
    assert np.array_equal(out, g["out"]) and np.array_equal(dth, g["dtheta"])
    assert np.array_equal(db, g["dbias"])
    assert np.array_equal(dx[::97], g["dinput_rows"])


def test_gat_layer_all_levels(golden, orc):
    g = golden("gat")
    n, h, k = int(g["n"]), int(g["heads"]), int(g["k"])
    pat = orc.Operator(n, np.repeat(np.arange(n, dtype=np.int32), np.diff(g["rowptr"])),
                       g["cols"], np.ones(len(g["cols"])))
    out, im = orc.gat_forward(pat, g["X"], g["theta"], g["a_src"], g["a_dst"], g["bias"], h,
                              float(g["beta"]), want=True)
    dth, das, dad, db, dx = orc.gat_backward(pat, g["G"], g["X"], g["theta"], g["a_src"],
                                             g["a_dst"], h, float(g["beta"]), True)
    for level in range(4):  # every level is bit-identical in the reference (test_gat.cpp:71-124)
        assert np.array_equal(out, g[f"out_{level}"])
        assert np.array_equal(im["alpha"], g[f"alpha_{level}"])
        assert np.array_equal(im["mask"], g[f"mask_{level}"])
        assert np.array_equal(dth, g[f"dtheta_{level}"])
        assert np.array_equal(das, g[f"da_src_{level}"])
        assert np.array_equal(dad, g[f"da_dst_{level}"])
        assert np.array_equal(db, g[f"dbias_{level}"])
        assert np.array_equal(dx, g[f"dinput_{level}"])


@pytest.mark.parametrize("tag", ["gcn2_adaptive_cached", "gcn2_adaptive_fg", "gcn2_tf",
                                 "gat2_h2", "gat2_h8"])
def test_oracle_model_step_matches_reference(golden, orc, tag):
    """oracle.gcn2_step / gat2_step (model.hpp restated over the oracle layers)
    against the reference's own Gcn2Model / Gat2Model step."""
    g = golden("models")
    kind, n, seed, m, hid, o, h, pol, ca, lv, ig = (int(x) for x in g[f"{tag}_cfg"])
    deg = float(g[f"{tag}_deg"][0])
    _, s, t = orc.synthetic_graph(n, deg, seed)
    X = orc.random_uniform(n, m, seed + 11)
    if kind == 0:
        op = orc.gcn_operator(n, s, t)
        target = orc.random_uniform(n, o, seed + 12)
        loss, out, grads, dx = orc.gcn2_step(op, X, orc.gcn2_params(m, hid, o, seed + 13), target,
                                             pol, bool(ca), bool(ig))
    else:
        pat = orc.gat_pattern(n, s, t)
        target = orc.random_uniform(n, h * o, seed + 12)
        loss, out, grads, dx = orc.gat2_step(pat, X, orc.gat2_params(m, h, hid, o, seed + 13), h,
                                             target, 0.2, bool(ig))
    flat = np.concatenate([np.asarray(x).ravel() for x in grads])
    assert orc.max_rel_diff(out, g[f"{tag}_pred"]) < 1e-12
    assert orc.max_rel_diff(flat, g[f"{tag}_grads"]) < 1e-12
    assert abs(loss - g[f"{tag}_loss"][0]) < 1e-12


def test_gat_f64_restatement_matches_reference_golden(golden):
    """oracle/gat_f64.py (vectorised float64 GAT, the full-size checker) against
    the reference's own outputs (tests/golden/gat.npz) at 1e-12, and its
    mask override is the identity when given the reference's own mask."""
    import gat_f64

    g = golden("gat")
    h, beta = int(g["heads"]), float(g["beta"])
    rp, cl = g["rowptr"], g["cols"]
    out, st = gat_f64.forward(rp, cl, g["X"], g["theta"], g["a_src"], g["a_dst"], g["bias"], h,
                              beta)
    assert np.abs(out - g["out_0"]).max() <= 1e-12 * max(1.0, np.abs(g["out_0"]).max())
    assert np.array_equal(st["mask"].T.astype(np.uint8), g["mask_0"])
    assert np.abs(st["alpha"].T - g["alpha_0"]).max() <= 1e-13
    for mask in (None, g["mask_0"].T.astype(bool)):
        got = gat_f64.backward(rp, cl, g["G"], g["X"], g["theta"], g["a_src"], g["a_dst"], h,
                               beta, True, mask=mask)
        for x, nm in zip(got, ("dtheta", "da_src", "da_dst", "dbias", "dinput")):
            want = g[f"{nm}_0"]
            assert np.abs(x - want).max() <= 1e-12 * max(1.0, np.abs(want).max()), nm
