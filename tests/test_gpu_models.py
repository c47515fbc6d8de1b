"""Two-layer models (model.hpp: Gcn2 GCN-ReLU-GCN, Gat2 GAT-ELU-GAT, MSE loss)
on the device against the oracle, which is pinned to the reference's own
model step (tests/golden/models.npz, oracle/gen_golden.py models)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

CASES = ["gcn2_adaptive_cached", "gcn2_adaptive_fg", "gcn2_tf", "gat2_h2", "gat2_h8"]


def _case(golden, tag):
    g = golden("models")
    kind, n, seed, m, hid, o, h, pol, ca, lv, ig = (int(x) for x in g[f"{tag}_cfg"])
    return g, dict(kind=kind, n=n, seed=seed, m=m, hid=hid, o=o, h=h, pol=pol, ca=ca, lv=lv,
                   ig=ig, deg=float(g[f"{tag}_deg"][0]))


@pytest.mark.parametrize("tag", CASES)
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_model_step_vs_reference(golden, orc, tag, dtype):
    from paper_2308_12093_b200 import device as d

    g, c = _case(golden, tag)
    n = c["n"]
    src, dst = d.synthetic_graph(n, c["deg"], c["seed"])
    X = d.random_uniform(n, c["m"], c["seed"] + 11, dtype=dtype)
    if c["kind"] == 0:
        graph = d.Adjacency.gcn_operator(n, src, dst, dtype, "csc")
        model = d.Model("gcn2", c["m"], c["hid"], c["o"], scheme=c["pol"], caching=c["ca"],
                        input_grad=c["ig"], seed=c["seed"] + 13, dtype=dtype)
        ow = c["o"]
    else:
        graph = d.Pattern.gat_pattern(n, src, dst)
        model = d.Model("gat2", c["m"], c["hid"], c["o"], heads=c["h"], gat_level=c["lv"],
                        input_grad=c["ig"], seed=c["seed"] + 13, dtype=dtype)
        ow = c["h"] * c["o"]
    target = d.random_uniform(n, ow, c["seed"] + 12, dtype=dtype)
    loss, out, grads, dx = model.train_step(graph, X, target)
    flat = torch.cat([t.reshape(-1) for t in grads]).double().cpu().numpy()
    tol = 1e-10 if dtype == torch.float64 else 1e-4
    assert orc.max_rel_diff(out.double().cpu().numpy(), g[f"{tag}_pred"]) < tol
    assert orc.max_rel_diff(flat, g[f"{tag}_grads"]) < tol
    assert abs(float(loss) - g[f"{tag}_loss"][0]) <= tol * max(1.0, abs(g[f"{tag}_loss"][0]))
    assert (dx is not None) == bool(c["ig"])


def test_model_params_are_reference_init(orc):
    from paper_2308_12093_b200 import device as d

    m = d.Model("gcn2", 7, 5, 3, seed=11, dtype=torch.float64)
    want = orc.gcn2_params(7, 5, 3, 11)
    for (name, t), w in zip(m.params, want):
        assert np.array_equal(t.cpu().numpy(), w), name
    g = d.Model("gat2", 6, 4, 2, heads=3, seed=5, dtype=torch.float64)
    want = orc.gat2_params(6, 3, 4, 2, 5)
    for (name, t), w in zip(g.params, want):
        assert np.array_equal(t.cpu().numpy(), w), name
    assert [nm for nm, _ in g.params] == ["l1.theta", "l1.a_src", "l1.a_dst", "l1.bias",
                                          "l2.theta", "l2.a_src", "l2.a_dst", "l2.bias"]


@pytest.mark.parametrize("graph_kind,hid", [("er", 32), ("er", 256), ("er", 40),
                                            ("powerlaw", 32)])
def test_gat2_fused_elu_bit_identical(monkeypatch, graph_kind, hid):
    """Gat2's ELU fused into the layer-1 aggregation epilogue and its backward
    fused into the layer-2 d_input GEMM give the same bits as the separate
    activation passes (SGNN_NO_ACT_FUSION=1).  The power-law graph has hub
    rows, where the forward keeps the separate pass and the backward fuses."""
    from paper_2308_12093_b200 import device as d

    n = 3000
    if graph_kind == "er":
        src, dst = d.synthetic_graph(n, 9.0, 5)
    else:
        src, dst = d.powerlaw_graph(n, 12.0, 2.2, 3)
    P = d.Pattern.gat_pattern(n, src, dst)
    X = d.random_uniform(n, 48, 16)
    target = d.random_uniform(n, 8 * 24, 17)
    model = d.Model("gat2", 48, hid, 24, heads=8, gat_level="full", seed=18)
    runs = []
    for off in ("0", "1"):
        monkeypatch.setenv("SGNN_NO_ACT_FUSION", off)
        loss, out, grads, _ = model.train_step(P, X, target)
        torch.cuda.synchronize()
        runs.append((loss.clone(), out.clone(), [g.clone() for g in grads]))
    (l0, o0, g0), (l1, o1, g1) = runs
    assert torch.equal(o0, o1) and torch.equal(l0, l1)
    for a, b in zip(g0, g1):
        assert torch.equal(a, b)
