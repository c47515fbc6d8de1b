"""Full-size parity: the CUDA path against the reference itself at the sizes
BASELINE.json quotes (configs 1-4), float64 reference vs float32 device under
max_rel_diff <= 1e-4 (the north-star bar; dense.hpp:303-316).

The checker is oracle/_ref -- the unmodified reference headers compiled with
-O3 -fopenmp by oracle/Makefile -- run in S=double on float32-representable
inputs widened exactly (SURVEY 8(c) golden policy: the float32 reference
drifts up to 7.3e-4 on the n=169k reductions, so it is not a golden).  The
device inputs are the reference harness's (bench.hpp:182-194): graph
synthetic_graph(n, q/n, seed=1), X from seed+11, dX' / target from seed+12,
parameters from seed+13, generated on the device bit-identically.

Reference call sites: gcn.hpp:91-193, gat.hpp:89-219, model.hpp:43-201."""
import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

SEED = 1
TOL = 1e-4
ARXIV = (169343, 1166243 / 169343)
PUBMED = (19717, 88648 / 19717)
FLICKR = (89250, 899756 / 89250)
GAT_OUT = ("out", "d_theta", "d_a_src", "d_a_dst", "d_bias", "d_input")


@pytest.fixture(scope="module")
def d():
    from paper_2308_12093_b200 import device

    return device


@pytest.fixture(scope="module")
def ref():
    import refpy  # oracle/_ref: the reference compiled in place (the checker)

    if not refpy.available():
        pytest.fail("oracle/_ref/libsgnn_ref.so missing: run __graft_entry__.build() first")
    return refpy


_graphs = {}


def graph(d, shape):
    if shape not in _graphs:
        _graphs[shape] = d.synthetic_graph(shape[0], shape[1], SEED)
    return _graphs[shape]


def h64(t):
    return t.detach().double().cpu().numpy()


def check_all(orc, pairs):
    """pairs: (name, device tensor or None, reference array or None); every
    error is computed before asserting so a failure reports all of them."""
    errs = {}
    for nm, g, w in pairs:
        if w is None:
            assert g is None, nm
            continue
        errs[nm] = orc.max_rel_diff(h64(g), w)
    bad = {k: f"{v:.3e}" for k, v in errs.items() if not v <= TOL}
    assert not bad, f"max_rel_diff > {TOL}: {bad} (all: { {k: f'{v:.2e}' for k, v in errs.items()} })"
    return errs


# ---- GCN: the bench step and config 2 (Arxiv 128 -> k) --------------------------
_gcn_ref = {}


def gcn_case(d, ref, m, k, fg, policy="adaptive", caching=True):
    n = ARXIV[0]
    src, dst = graph(d, ARXIV)
    A = d.Adjacency.gcn_operator(n, src, dst, torch.float32, "csc")
    X = d.random_uniform(n, m, SEED + 11)
    G = d.random_uniform(n, k, SEED + 12)
    theta, bias = d.gcn_params(m, k, SEED + 13)
    s = d.resolve_scheme(policy, m, k, fg, caching)
    out, cache = d.gcn_forward(A, X, theta, bias, s)
    dth, db, dx = d.gcn_backward(A, G, theta, cache, fg)
    if "coo" not in _gcn_ref:
        _gcn_ref["coo"] = ref.gcn_normalize(n, src.numpy(), dst.numpy())
    want = ref.gcn_layer(n, _gcn_ref["coo"], 2, h64(X), h64(theta), h64(bias),
                         (s.forward, s.backward, s.caching), h64(G), fg)
    return s, (out, dth, db, dx), want


def test_headline_step_full_size(d, ref, orc):
    """bench.py's timed step: Arxiv 128 -> 256, fg, adaptive + caching
    (-> propagate_first_cached + split_propagate_cached), CSC."""
    s, got, want = gcn_case(d, ref, 128, 256, True)
    assert (s.forward, s.backward, s.caching) == (2, 2, True)
    check_all(orc, zip(("out", "d_theta", "d_bias", "d_input"), got, want))


@pytest.mark.parametrize("k", [8, 64, 256, 1024])
@pytest.mark.parametrize("fg", [False, True])
def test_config2_arxiv_sweep(d, ref, orc, k, fg):
    s, got, want = gcn_case(d, ref, 128, k, fg)
    check_all(orc, zip(("out", "d_theta", "d_bias", "d_input"), got, want))


@pytest.mark.parametrize("policy,caching", [("transform-first", False), ("propagate-first", False),
                                            ("propagate-first", True)])
@pytest.mark.parametrize("k", [8, 64])
def test_config2_forced_schemes(d, ref, orc, policy, caching, k):
    s, got, want = gcn_case(d, ref, 128, k, True, policy=policy, caching=caching)
    check_all(orc, zip(("out", "d_theta", "d_bias", "d_input"), got, want))


def test_config1_cora(d, ref, orc):
    """Cora-shaped 1433 -> 16, CSC, caching on (-> transform_first + fused)."""
    n, q = 2708, 10556
    src, dst = d.synthetic_graph(n, q / n, SEED)
    A = d.Adjacency.gcn_operator(n, src, dst, torch.float32, "csc")
    X = d.random_uniform(n, 1433, SEED + 11)
    G = d.random_uniform(n, 16, SEED + 12)
    theta, bias = d.gcn_params(1433, 16, SEED + 13)
    s = d.resolve_scheme("adaptive", 1433, 16, True, True)
    assert (s.forward, s.backward, s.caching) == (0, 0, False)
    out, cache = d.gcn_forward(A, X, theta, bias, s)
    got = (out,) + d.gcn_backward(A, G, theta, cache, True)
    coo = ref.gcn_normalize(n, src.numpy(), dst.numpy())
    want = ref.gcn_layer(n, coo, 2, h64(X), h64(theta), h64(bias), (0, 0, 0), h64(G), True)
    check_all(orc, zip(("out", "d_theta", "d_bias", "d_input"), got, want))


# ---- GAT: config 3 (PubMed / Flickr, 500 -> 8 x k, every cache level) -----------
# The LeakyReLU derivative jumps at y = s_i + d_j = 0: an edge whose float32
# score falls on the other side of zero than the float64 one takes the other
# slope in the backward pass (an O(1) change of its dy, which moves d_theta /
# d_a_src / d_input by up to ~1e-2 at these sizes; measured).  Those decisions
# are ill-conditioned, not wrong, so the gradients are checked against the
# float64 restatement (oracle/gat_f64.py, pinned to the reference) evaluated
# with the device's LeakyReLU decisions, and every decision that differs from
# the float64 one must sit at |y| < 1e-5 of the score scale.  The forward
# output (continuous in y) is checked against the reference itself.
def gat_case(d, ref, orc, shape, h, k, m, levels):
    import gat_f64

    n = shape[0]
    src, dst = graph(d, shape)
    P = d.Pattern.gat_pattern(n, src, dst)
    X = d.random_uniform(n, m, SEED + 11)
    G = d.random_uniform(n, h * k, SEED + 12)
    th, a_s, a_d, b = d.gat_params(m, h, k, SEED + 13)
    pa = P.arrays()
    rp, cl = pa["rowptr"].cpu().numpy(), pa["cols"].cpu().numpy()
    args = [h64(x) for x in (X, th, a_s, a_d, b)]
    want_out = ref.gat_layer(n, rp, cl, *args, h, 3, h64(G), False)[0]
    out_ref, st = gat_f64.forward(rp, cl, *args, h)
    assert orc.max_rel_diff(out_ref, want_out) < 1e-12  # restatement == reference
    dev_mask = None
    results = {}
    for level in levels:
        out, cache = d.gat_forward(P, X, th, a_s, a_d, b, h, 0.2, level)
        # the decisions of THIS level's backward: levels recompute the scores
        # by different routes (the fused GEMM epilogue at none, node_scores
        # from the cached M at features), whose roundings may put a |y| ~ 0
        # edge on different sides
        _, mk = cache.edge_values(P, th, a_s, a_d)
        mask = mk.t().cpu().numpy().astype(bool)  # edge-major q x h
        if dev_mask is None or not np.array_equal(mask, dev_mask):
            dev_mask = mask
            flips, far = gat_f64.ill_conditioned_flips(st["y"], dev_mask)
            assert far == 0, f"{far} of {flips} LeakyReLU decisions differ at |y| >= 1e-5 scale"
            want_g = gat_f64.backward(rp, cl, h64(G), args[0], args[1], args[2], args[3], h,
                                      fg=True, mask=dev_mask)
        grads = d.gat_backward(P, G, th, a_s, a_d, cache, True)
        names = [f"{level}:{x}" for x in GAT_OUT]
        results[level] = check_all(orc, zip(names, (out,) + grads, (want_out,) + want_g))
    return flips, results


@pytest.mark.parametrize("shape", [PUBMED, FLICKR], ids=["pubmed", "flickr"])
@pytest.mark.parametrize("k", [8, 64])
def test_config3_gat_levels(d, ref, orc, shape, k):
    gat_case(d, ref, orc, shape, 8, k, 500, ("none", "features", "node-attn", "full"))


def test_gat_layer_arxiv_bench_shape(d, ref, orc):
    """bench.py's gat_layer line: Arxiv h=8 k=32, level full, fg."""
    gat_case(d, ref, orc, ARXIV, 8, 32, 128, ("full",))


# ---- config 4: 2-layer models, full training step with MSE ----------------------
@pytest.mark.parametrize("kind,hid", [("gcn2", 256), ("gat2", 256), ("gat2", 32)],
                         ids=["gcn2_128-256-40", "gat2_128-8x256-8x40", "gat2_128-8x32-8x40"])
def test_config4_model_step(d, ref, orc, kind, hid):
    n, m, o, h = ARXIV[0], 128, 40, 8
    src, dst = graph(d, ARXIV)
    X = d.random_uniform(n, m, SEED + 11)
    if kind == "gcn2":
        g = d.Adjacency.gcn_operator(n, src, dst, torch.float32, "csc")
        model = d.Model("gcn2", m, hid, o, scheme="adaptive", caching=True, seed=SEED + 13)
        tgt = d.random_uniform(n, o, SEED + 12)
        want = ref.model_step(0, n, ARXIV[1], SEED, m, hid, o, policy=0, caching=True)
    else:
        g = d.Pattern.gat_pattern(n, src, dst)
        model = d.Model("gat2", m, hid, o, heads=h, gat_level="full", seed=SEED + 13)
        tgt = d.random_uniform(n, h * o, SEED + 12)
        want = ref.model_step(1, n, ARXIV[1], SEED, m, hid, o, heads=h, level=3)
    loss, out, grads, _ = model.train_step(g, X, tgt)
    flat = torch.cat([t.reshape(-1) for t in grads])
    check_all(orc, [("prediction", out, want[1]), ("gradients", flat, want[2])])
    gw, gg = want[2], h64(flat)
    print(f"\n{kind} hid={hid}: gradient error / max|gradient| = "
          f"{np.abs(gg - gw).max() / np.abs(gw).max():.3e}")
    assert abs(float(loss) - want[0]) <= TOL * max(1.0, abs(want[0]))


# ---- config 5 at one GPU: the large power-law graph ----------------------------
LARGE = (2449029, 61859140 / 2449029)


def test_config5_powerlaw_gcn_layer(d, ref, orc):
    """A config-5 GCN layer (100 -> 256, fg, adaptive + caching) on the
    2.45M-node / 64M-edge power-law graph (maximum degree ~1e5: the hub-row
    segment plans) against the reference in float64 on the same COO."""
    n, m, k = LARGE[0], 100, 256
    src, dst = d.powerlaw_graph(n, LARGE[1], 2.5, SEED)
    A = d.Adjacency.gcn_operator(n, src, dst, torch.float32, "csc")
    X = d.random_uniform(n, m, SEED + 11)
    G = d.random_uniform(n, k, SEED + 12)
    theta, bias = d.gcn_params(m, k, SEED + 13)
    s = d.resolve_scheme("adaptive", m, k, True, True)
    out, cache = d.gcn_forward(A, X, theta, bias, s)
    got = (out,) + d.gcn_backward(A, G, theta, cache, True)
    coo = ref.gcn_normalize(n, src.cpu().numpy(), dst.cpu().numpy())
    assert coo[0].size == A.nnz
    want = ref.gcn_layer(n, coo, 2, h64(X), h64(theta), h64(bias),
                         (s.forward, s.backward, s.caching), h64(G), True)
    check_all(orc, zip(("out", "d_theta", "d_bias", "d_input"), got, want))


def test_config5_powerlaw_gat_forward(d, ref, orc):
    """The config-5 GAT layer's forward (100 -> 8 x 32) on the power-law
    pattern against the reference in float64 (the output is continuous in
    the scores; the LeakyReLU-decision caveat above concerns gradients)."""
    n, m, h, k = LARGE[0], 100, 8, 32
    src, dst = d.powerlaw_graph(n, LARGE[1], 2.5, SEED)
    P = d.Pattern.gat_pattern(n, src, dst)
    X = d.random_uniform(n, m, SEED + 11)
    th, a_s, a_d, b = d.gat_params(m, h, k, SEED + 13)
    out, _ = d.gat_forward(P, X, th, a_s, a_d, b, h, 0.2, "none")
    pa = P.arrays()
    rp, cl = pa["rowptr"].cpu().numpy(), pa["cols"].cpu().numpy()
    G0 = np.zeros((n, h * k))
    want = ref.gat_layer(n, rp, cl, *[h64(x) for x in (X, th, a_s, a_d, b)], h, 0, G0, False)[0]
    check_all(orc, [("out", out, want)])
