"""Central-difference gradient checks of the device models in float64 -- the
reference's own correctness property (model.hpp gradient_check, used by
test_gcn.cpp / test_gat.cpp and `sgnn-bench gradcheck`): perturb a parameter
coordinate by +-eps, re-evaluate the MSE loss on the device, compare with the
analytic gradient of the backward pass under rel_err (dense.hpp:318-320)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _rel_err(a, b):
    return abs(a - b) / max(1.0, abs(a), abs(b))


def _check(model, graph, X, target, coords=12, eps=1e-6, seed=0):
    loss, _, grads, _ = model.train_step(graph, X, target)
    rng = np.random.default_rng(seed)
    worst = 0.0
    for (name, p), g in zip(model.params, grads):
        flat, gflat = p.view(-1), g.view(-1).cpu().numpy()
        for i in rng.choice(flat.numel(), size=min(coords, flat.numel()), replace=False):
            saved = float(flat[i])
            flat[i] = saved + eps
            up = float(model.train_step(graph, X, target)[0])
            flat[i] = saved - eps
            down = float(model.train_step(graph, X, target)[0])
            flat[i] = saved
            worst = max(worst, _rel_err(gflat[i], (up - down) / (2 * eps)))
    return worst


@pytest.mark.parametrize("caching,policy", [(True, "adaptive"), (False, "transform-first"),
                                            (False, "propagate-first")])
def test_gcn2_gradients_match_central_differences(caching, policy):
    from paper_2308_12093_b200 import device as d

    n = 400
    src, dst = d.synthetic_graph(n, 6.0, 5)
    A = d.Adjacency.gcn_operator(n, src, dst, torch.float64, "csc")
    m = d.Model("gcn2", 9, 7, 4, scheme=policy, caching=caching, seed=3, dtype=torch.float64)
    X = d.random_uniform(n, 9, 11, dtype=torch.float64)
    t = d.random_uniform(n, 4, 12, dtype=torch.float64)
    assert _check(m, A, X, t) < 1e-6


@pytest.mark.parametrize("level", ["none", "full"])
def test_gat2_gradients_match_central_differences(level):
    from paper_2308_12093_b200 import device as d

    n = 300
    src, dst = d.synthetic_graph(n, 5.0, 7)
    P = d.Pattern.gat_pattern(n, src, dst)
    m = d.Model("gat2", 6, 3, 2, heads=2, gat_level=level, seed=4, dtype=torch.float64)
    X = d.random_uniform(n, 6, 11, dtype=torch.float64)
    t = d.random_uniform(n, 4, 12, dtype=torch.float64)
    assert _check(m, P, X, t) < 1e-6
