"""Row-partitioned GCN layer on the GPU.

* world_size 1 over NCCL: DistGcnLayer with the product backend (DeviceOps ->
  libsgnn_cuda.so) against the oracle, every scheme.
* virtual partitions on one GPU: the row blocks A'_p / A'^T_p that rank p
  would own propagate bit-identically to the rows of the single-GPU product
  (the accumulation order inside a row is unchanged by the partition)."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl_world1():
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("scheme", [(0, 0, 0), (1, 1, 0), (2, 2, 1), (0, 1, 0), (1, 0, 0)])
@pytest.mark.parametrize("fg", [False, True])
def test_dist_layer_nccl_world1(nccl_world1, orc, scheme, fg):
    from paper_2308_12093_b200 import dist as pd

    n, m, k = 3000, 48, 40
    _, s, t = orc.synthetic_graph(n, 9.0, 5)
    op = orc.gcn_operator(n, s, t)
    X = orc.random_uniform(n, m, 11)
    th, bi = orc.gcn_params(m, k, 13)
    G = orc.random_uniform(n, k, 12)
    ref = orc.gcn_layer(op, X, th, bi, scheme, G, fg)
    layer = pd.DistGcnLayer(n, op.rows, op.cols, op.vals, pd.DeviceOps("cuda:0"), torch.float64)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    out, cache = layer.forward(cu(X), cu(th), cu(bi), scheme)
    dth, db, dx = layer.backward(cu(G), cu(th), cache, fg)
    assert orc.max_rel_diff(out.cpu().numpy(), ref[0]) < 1e-12
    assert orc.max_rel_diff(dth.cpu().numpy(), ref[1]) < 1e-10
    assert orc.max_rel_diff(db.cpu().numpy(), ref[2]) < 1e-12
    if fg:
        assert orc.max_rel_diff(dx.cpu().numpy(), ref[3]) < 1e-10


@pytest.mark.parametrize("parts", [2, 3, 8])
def test_partition_blocks_bit_identical(orc, parts):
    from paper_2308_12093_b200 import device as d
    from paper_2308_12093_b200 import dist as pd

    n, f = 20000, 128
    _, s, t = orc.synthetic_graph(n, 13.77, 1)
    op = orc.gcn_operator(n, s, t)
    rowptr = np.concatenate([[0], np.cumsum(np.bincount(op.rows, minlength=n))])
    bounds = pd.partition_rows(rowptr, parts)
    ops = pd.DeviceOps("cuda:0")
    cu = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dt)  # noqa: E731
    full = d.Adjacency(n, n, cu(op.rows, torch.int32), cu(op.cols, torch.int32),
                       cu(op.vals, torch.float32), "csc")
    B = d.random_uniform(n, f, 7)
    ref = full.spmm(B)
    refT = full.spmm(B, transposed=True)
    for p in range(parts):
        r0, r1 = bounds[p], bounds[p + 1]
        rb = pd.row_block(op.rows, op.cols, op.vals.astype(np.float32), r0, r1)
        A_p = ops.adjacency(r1 - r0, n, *rb, torch.float32)
        assert torch.equal(A_p.spmm(B), ref[r0:r1])
        tb = pd.transposed_block(op.rows, op.cols, op.vals.astype(np.float32), r0, r1)
        AT_p = ops.adjacency(r1 - r0, n, *tb, torch.float32)
        assert torch.equal(AT_p.spmm(B), refT[r0:r1])


def test_dist_step_host_matches_device_path(nccl_world1, orc):
    from paper_2308_12093_b200 import dist as pd

    n, m, k = 2500, 32, 24
    _, s, t = orc.synthetic_graph(n, 8.0, 2)
    op = orc.gcn_operator(n, s, t)
    layer = pd.DistGcnLayer(n, op.rows, op.cols, op.vals, pd.DeviceOps("cuda:0"), torch.float32)
    X = torch.rand(n, m) * 2 - 1
    G = torch.rand(n, k) * 2 - 1
    th, bi = (torch.from_numpy(a.astype(np.float32)).cuda() for a in orc.gcn_params(m, k, 13))
    for scheme in [(0, 0, 0), (2, 2, 1), (1, 1, 0)]:
        out, cache = layer.forward(X.cuda(), th, bi, scheme)
        ref = (out,) + layer.backward(G.cuda(), th, cache, True)
        pin = lambda *sh: torch.empty(sh).pin_memory()  # noqa: E731
        hs = (pin(n, k), pin(m, k), pin(k), pin(n, m))
        layer.step_host(X.pin_memory(), th, bi, scheme, G.pin_memory(), True, *hs)
        torch.cuda.synchronize()
        for a, b in zip(hs, ref):
            assert torch.equal(a, b.cpu()), scheme


@pytest.mark.parametrize("dtype,tol", [(torch.float64, 1e-10), (torch.float32, 1e-4)])
def test_dist_gcn2_matches_oracle_model(nccl_world1, orc, dtype, tol):
    """Partitioned 2-layer GCN step (world 1) against oracle.gcn2_step, which is
    pinned to the reference's Gcn2Model step."""
    from paper_2308_12093_b200 import dist as pd

    n, m, hid, o, seed = 1500, 20, 16, 6, 4
    _, s, t = orc.synthetic_graph(n, 7.0, 3)
    op = orc.gcn_operator(n, s, t)
    layer = pd.DistGcnLayer(n, op.rows, op.cols, op.vals, pd.DeviceOps("cuda:0"), dtype)
    model = pd.DistGcn2(layer, m, hid, o, seed, caching=True, input_grad=False, dtype=dtype)
    X = orc.random_uniform(n, m, seed + 11)
    target = orc.random_uniform(n, o, seed + 12)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dtype)  # noqa: E731
    loss, out, grads, _ = model.train_step(cu(X), cu(target))
    rl, rout, rgrads, _ = orc.gcn2_step(op, X, orc.gcn2_params(m, hid, o, seed), target, 0, True,
                                        False)
    assert abs(float(loss) - rl) <= tol * max(1.0, abs(rl))
    assert orc.max_rel_diff(out.double().cpu().numpy(), rout) < tol
    for g, r in zip(grads, rgrads):
        assert orc.max_rel_diff(g.double().cpu().numpy(), r) < tol


def test_activation_and_loss_entry_points(orc):
    from paper_2308_12093_b200 import device as d

    x = torch.randn(1000, 7, dtype=torch.float64, device="cuda")
    for kind, prm in (("relu", 0.0), ("elu", 1.0)):
        h, mask = d.activation(x, kind)
        rh, rmask = orc.activation(x.cpu().numpy(), kind, prm)
        assert orc.max_rel_diff(h.cpu().numpy(), rh) < 1e-15
        assert np.array_equal(mask.cpu().numpy(), rmask)
        g = torch.randn_like(x)
        gi = d.activation_backward(g, mask, kind, saved=h)
        rgi = orc.activation_backward(g.cpu().numpy(), rmask, kind, prm, rh)
        assert orc.max_rel_diff(gi.cpu().numpy(), rgi) < 1e-15
    tgt = torch.randn_like(x)
    loss, grad = d.loss_mse(x, tgt)
    rl, rg = orc.loss_mse(x.cpu().numpy(), tgt.cpu().numpy())
    assert abs(float(loss) - rl) < 1e-12 and orc.max_rel_diff(grad.cpu().numpy(), rg) < 1e-15


@pytest.mark.parametrize("h,k,exchange", [(8, 32, "edges"), (4, 12, "edges"), (2, 64, "edges"),
                                          (8, 32, "stats"), (4, 16, "stats"), (2, 256, "stats"),
                                          (1, 512, "stats")])
def test_dist_gat_layer_world1(nccl_world1, orc, h, k, exchange):
    """Partitioned GAT layer (world 1).  exchange="edges": the single-GPU
    layer's kernels in the same order (bit-identical results).  "stats": the
    column pass rebuilds alpha / dy from per-row statistics (alpha bit-identical,
    dAlpha re-reduced), checked against the oracle at the north-star 1e-4."""
    from paper_2308_12093_b200 import device as d
    from paper_2308_12093_b200 import dist as pd

    n, m = 2200, 24
    _, s, t = orc.synthetic_graph(n, 8.0, 6)
    pat = orc.gat_pattern(n, s, t)
    layer = pd.DistGatLayer(n, pat.rowptr, pat.cols, h, k, "cuda:0", exchange=exchange)
    assert layer.exchange == exchange
    th, a_s, a_d, b = (torch.from_numpy(x.astype(np.float32)).cuda()
                       for x in orc.gat_params(m, h, k, 21))
    X = orc.random_uniform(n, m, 11)
    G = orc.random_uniform(n, h * k, 12)
    Xc = torch.from_numpy(X.astype(np.float32)).cuda()
    Gc = torch.from_numpy(G.astype(np.float32)).cuda()
    out, cache = layer.forward(Xc, th, a_s, a_d, b)
    grads = layer.backward(Gc, th, a_s, a_d, cache, True)
    P = d.Pattern(n, torch.from_numpy(pat.rowptr).cuda(), torch.from_numpy(pat.cols).cuda())
    o1, c1 = d.gat_forward(P, Xc, th, a_s, a_d, b, h, 0.2, "full")
    g1 = d.gat_backward(P, Gc, th, a_s, a_d, c1, True)
    assert torch.equal(out, o1)
    if exchange == "edges":
        for a_, b_ in zip(grads, g1):
            assert torch.equal(a_, b_)
    ref_o = orc.gat_forward(pat, X, *orc.gat_params(m, h, k, 21), h, 0.2)
    assert orc.max_rel_diff(out.double().cpu().numpy(), ref_o) < 1e-4
    ref_g = orc.gat_backward(pat, G, X, *orc.gat_params(m, h, k, 21)[:3], h, 0.2, True)
    for g, r in zip(grads, ref_g):
        assert orc.max_rel_diff(g.double().cpu().numpy(), r) < 1e-4


@pytest.mark.parametrize("exchange", ["edges", "stats"])
def test_dist_gat_layer_world1_hub_rows(nccl_world1, orc, exchange):
    """The partitioned GAT layer on a power-law graph (hub rows / columns run
    through the block entry points' row plans): forward bit-identical to the
    single-GPU layer, gradients bit-identical ("edges") or within the fp32
    bar of it ("stats")."""
    from paper_2308_12093_b200 import device as d
    from paper_2308_12093_b200 import dist as pd

    n, m, h, k = 3000, 16, 8, 8
    s, t = d.powerlaw_graph(n, 10.0, 2.1, 9)
    P = d.Pattern.gat_pattern(n, s, t)
    pa = P.arrays()
    assert int(torch.diff(pa["rowptr"]).max()) > 500
    layer = pd.DistGatLayer(n, pa["rowptr"], pa["cols"], h, k, "cuda:0", exchange=exchange)
    th, a_s, a_d, b = d.gat_params(m, h, k, 3)
    X = d.random_uniform(n, m, 1)
    G = d.random_uniform(n, h * k, 2)
    out, cache = layer.forward(X, th, a_s, a_d, b)
    grads = layer.backward(G, th, a_s, a_d, cache, True)
    o1, c1 = d.gat_forward(P, X, th, a_s, a_d, b, h, 0.2, "full")
    g1 = d.gat_backward(P, G, th, a_s, a_d, c1, True)
    assert torch.equal(out, o1)
    for x, y in zip(grads, g1):
        if exchange == "edges":
            assert torch.equal(x, y)
        else:
            assert orc.max_rel_diff(x.double().cpu().numpy(), y.double().cpu().numpy()) < 1e-4


def test_dist_gat2_matches_oracle_model(nccl_world1, orc):
    """Partitioned 2-layer GAT step (world 1) against oracle.gat2_step, pinned
    to the reference's Gat2Model step."""
    from paper_2308_12093_b200 import dist as pd

    n, m, h, hid, o, seed = 1400, 20, 4, 8, 4, 5
    _, s, t = orc.synthetic_graph(n, 7.0, 2)
    pat = orc.gat_pattern(n, s, t)
    l1 = pd.DistGatLayer(n, pat.rowptr, pat.cols, h, hid, "cuda:0", exchange="stats")
    l2 = pd.DistGatLayer(n, pat.rowptr, pat.cols, h, o, "cuda:0", exchange="stats")
    assert l1.exchange == "stats" and l2.exchange == "stats"
    model = pd.DistGat2(l1, l2, m, hid, o, h, seed)
    X = orc.random_uniform(n, m, seed + 11)
    tgt = orc.random_uniform(n, h * o, seed + 12)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()  # noqa: E731
    loss, out, grads, _ = model.train_step(cu(X), cu(tgt))
    prm = [p.double().cpu().numpy() for p in model.p]  # the device's float32 parameters
    rl, rout, rgrads, _ = orc.gat2_step(pat, X, prm, h, tgt, 0.2, False)
    assert abs(float(loss) - rl) <= 1e-4 * max(1.0, abs(rl))
    assert orc.max_rel_diff(out.double().cpu().numpy(), rout) < 1e-4
    for g, r in zip(grads, rgrads):
        assert orc.max_rel_diff(g.double().cpu().numpy(), r) < 1e-4
