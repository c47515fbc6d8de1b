"""The operator-reordered GAT layer (csrc/gat_reorder.cuh, sgnn_gat_forward_ex
SGNN_GAT_REORDER): wide heads (k > m) run with the attention scores as
X (Theta_t a_t), the aggregation over the m-wide input rows and the per-head
transforms after it -- outputs and all five gradients against the float64
oracle at the north star's float32 bar (1e-4) at every cache level, with and
without input gradients; the gate (k <= m, hub rows, float64) falls back to
the reference order."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def d():
    from paper_2308_12093_b200 import device

    return device


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()


def h64(t):
    return t.detach().double().cpu().numpy()


def _case(d, orc, n, deg, m, h, k, seed):
    _, s, t = orc.synthetic_graph(n, deg, seed)
    pat = orc.gat_pattern(n, s, t)
    P = d.Pattern(pat.n, torch.from_numpy(pat.rowptr).cuda(), torch.from_numpy(pat.cols).cuda())
    X = orc.random_uniform(n, m, seed + 1)
    th, a_s, a_d, bi = orc.gat_params(m, h, k, seed + 2)
    G = orc.random_uniform(n, h * k, seed + 3)
    return pat, P, X, (th, a_s, a_d, bi), G


SHAPES = [(2000, 8.0, 16, 8, 32), (1500, 6.0, 12, 4, 64), (1200, 9.0, 32, 2, 128),
          (900, 5.0, 64, 1, 256), (800, 7.0, 128, 8, 256), (600, 6.0, 256, 4, 512),
          (500, 5.0, 20, 8, 40), (700, 30.0, 100, 2, 104), (64, 3.0, 8, 8, 12)]


@pytest.mark.parametrize("n,deg,m,h,k", SHAPES)
@pytest.mark.parametrize("fg", [False, True])
def test_reordered_layer_vs_oracle(d, orc, n, deg, m, h, k, fg):
    pat, P, X, prm, G = _case(d, orc, n, deg, m, h, k, n + h + k)
    th, a_s, a_d, bi = prm
    ref_out = orc.gat_forward(pat, X, th, a_s, a_d, bi, h, 0.2)
    ref = orc.gat_backward(pat, G, X, th, a_s, a_d, h, 0.2, fg)
    names = ("d_theta", "d_a_src", "d_a_dst", "d_bias", "d_input")
    for level in ("none", "features", "node-attn", "full"):
        out, cache = d.gat_forward(P, cu(X), cu(th), cu(a_s), cu(a_d), cu(bi), h, 0.2, level,
                                   reorder=True)
        assert cache.reordered, level
        assert orc.max_rel_diff(h64(out), ref_out) < 1e-4, level
        # the cache keeps Z (n x h x m) where the reference keeps M (n x h k)
        want = {"none": 0, "features": 4 * n * h * m, "node-attn": 4 * n * h * m + 8 * n * h,
                "full": 4 * n * h * m + 5 * pat.cols.size * h}[level]
        assert cache.extra_bytes() == want, level
        got = d.gat_backward(P, cu(G), cu(th), cu(a_s), cu(a_d), cache, fg, 0.2)
        for nm, gv, rv in zip(names, got, ref):
            if gv is None or rv is None:
                assert not fg and nm == "d_input"
                continue
            assert orc.max_rel_diff(h64(gv), rv) < 1e-4, (level, nm)


@pytest.mark.parametrize("level", ["none", "node-attn", "full"])
def test_reordered_edge_values(d, orc, level):
    """Attention of a reordered cache (kept or recomputed from X W) against the
    oracle's alpha, and its LeakyReLU mask against the reference order's."""
    n, m, h, k = 1000, 16, 4, 48
    pat, P, X, (th, a_s, a_d, bi), _ = _case(d, orc, n, 7.0, m, h, k, 41)
    _, cache = d.gat_forward(P, cu(X), cu(th), cu(a_s), cu(a_d), cu(bi), h, 0.2, level,
                             reorder=True)
    assert cache.reordered
    alpha, mask = cache.edge_values(P, cu(th), cu(a_s), cu(a_d))
    _, base = d.gat_forward(P, cu(X), cu(th), cu(a_s), cu(a_d), cu(bi), h, 0.2, level)
    assert not base.reordered
    a0, m0 = base.edge_values(P, cu(th), cu(a_s), cu(a_d))
    assert orc.max_rel_diff(h64(alpha), h64(a0)) < 1e-5
    # scores summed in another order may flip the sign decision only at y ~ 0
    assert (mask != m0).float().mean().item() < 1e-3


def test_reorder_gate(d, orc):
    """k <= m, float64 and hub rows keep the reference order."""
    n = 900
    pat, P, X, (th, a_s, a_d, bi), _ = _case(d, orc, n, 6.0, 64, 4, 64, 5)
    _, c = d.gat_forward(P, cu(X), cu(th), cu(a_s), cu(a_d), cu(bi), 4, 0.2, "full",
                         reorder=True)
    assert not c.reordered  # k == m
    f64 = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    pat, P, X, (th, a_s, a_d, bi), _ = _case(d, orc, n, 6.0, 16, 4, 64, 6)
    _, c = d.gat_forward(P, f64(X), f64(th), f64(a_s), f64(a_d), f64(bi), 4, 0.2, "full",
                         reorder=True)
    assert not c.reordered  # float64
    s, t = d.powerlaw_graph(4000, 12.0, 2.1, 3)
    P = d.Pattern.gat_pattern(4000, s, t)
    X = d.random_uniform(4000, 16, 1)
    th, a_s, a_d, bi = d.gat_params(16, 4, 64, 2)
    _, c = d.gat_forward(P, X, th, a_s, a_d, bi, 4, 0.2, "full", reorder=True)
    assert not c.reordered  # hub rows (> 128 edges)


def test_reordered_model_matches_reference_order(d, monkeypatch):
    """Gat2 with a wide hidden layer (128 -> 8 x 256) runs layer 1 reordered;
    its loss, prediction and gradients agree with the reference-order run
    (SGNN_GAT_REORDER=0 in a child process) at the float32 bar."""
    import subprocess
    import sys

    code = r"""
import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_2308_12093_b200 import device as d
n = 4000
s, t = d.synthetic_graph(n, 9.0, 3)
P = d.Pattern.gat_pattern(n, s, t)
X = d.random_uniform(n, 128, 4)
tg = d.random_uniform(n, 8 * 40, 5)
m = d.Model("gat2", 128, 256, 40, heads=8, gat_level=sys.argv[1], seed=6)
loss, out, grads, _ = m.train_step(P, X, tg)
flat = torch.cat([g.reshape(-1) for g in grads])
np.save(sys.argv[2], np.concatenate([[float(loss)], out.double().cpu().numpy().ravel(),
                                     flat.double().cpu().numpy()]))
"""
    import os
    import tempfile

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with tempfile.TemporaryDirectory() as tmp:
        for level in ("none", "full"):
            res = []
            for flag in ("1", "0"):
                f = os.path.join(tmp, f"{level}{flag}.npy")
                env = dict(os.environ, SGNN_GAT_REORDER=flag)
                subprocess.run([sys.executable, "-c", code, level, f], cwd=root, env=env,
                               check=True, timeout=300)
                res.append(np.load(f))
            a, b = res
            rel = np.abs(a - b).max() / np.abs(b).max()
            assert rel < 1e-4, (level, rel)


def test_fused_attention_aggregation_bit_identical():
    """The forward's fused attention + aggregation kernel (k_gat_attnagg) and
    the backward's fused SDDMM + softmax backward (k_gat_sddmm_sbwd, register
    head reductions P2 = 1 and P2 = 2) give the same bits as k_gat_attn4 +
    k_gat_agg2 / k_gat_sddmm2 + k_gat_sbwd4 (SGNN_GAT_FUSE=0, child process)
    for outputs, cached attention and the backward, on a uniform graph and on a
    power-law graph with hub rows (those keep the segment path)."""
    import os
    import subprocess
    import sys
    import tempfile

    code = r"""
import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_2308_12093_b200 import device as d
res = []
for kind, h, k in (("er", 8, 32), ("er", 4, 40), ("er", 2, 64), ("er", 1, 256), ("pl", 8, 8)):
    n = 3000
    s, t = d.synthetic_graph(n, 9.0, 3) if kind == "er" else d.powerlaw_graph(n, 12.0, 2.1, 5)
    P = d.Pattern.gat_pattern(n, s, t)
    X = d.random_uniform(n, 48, 4)
    th, a_s, a_d, b = d.gat_params(48, h, k, 6)
    G = d.random_uniform(n, h * k, 7)
    for level in ("none", "full"):
        out, c = d.gat_forward(P, X, th, a_s, a_d, b, h, 0.2, level)
        al, mk = c.edge_values(P, th, a_s, a_d)
        g = d.gat_backward(P, G, th, a_s, a_d, c, True)
        res += [out.cpu().numpy().ravel(), al.cpu().numpy().ravel(), mk.cpu().numpy().ravel()]
        res += [x.cpu().numpy().ravel() for x in g]
np.save(sys.argv[1], np.concatenate([r.astype(np.float64) for r in res]))
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with tempfile.TemporaryDirectory() as tmp:
        out = []
        for flag in ("1", "0"):
            f = os.path.join(tmp, f"{flag}.npy")
            subprocess.run([sys.executable, "-c", code, f], cwd=root,
                           env=dict(os.environ, SGNN_GAT_FUSE=flag), check=True, timeout=300)
            out.append(np.load(f))
        assert np.array_equal(out[0], out[1])
