"""The row-partitioned layers at world 2 and 3 on ONE B200: every rank is a
thread with its own sgnn context (stream), and the collectives are simulated
in process (slot copies and a rank-ordered sum between the threads, at the
points the NCCL calls sit).  The device kernels then run on the padded
multi-rank layouts -- remapped column ids, perm into the gathered edge slots,
gathered per-row statistics, hub-row plans of the rank's blocks -- which the
world-1 NCCL tests cannot reach.  Every rank's rows of the outputs and the
all-reduced gradients are checked against the single-process oracle."""
import threading

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


class _Shared:
    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.deposit = [None] * world


class SimExchange:
    """In-process stand-in for dist._Exchange (all-gather of rank slots,
    all-reduce in rank order) between rank threads on one GPU."""

    def __init__(self, shared, rank):
        self.sh, self.rank, self.world = shared, rank, shared.world

    def start(self, buf, slots):
        sh = self.sh
        torch.cuda.current_stream().synchronize()  # my slot is written
        sh.deposit[self.rank] = buf
        sh.barrier.wait()
        for p in range(self.world):
            if p != self.rank:
                buf[p * slots:(p + 1) * slots].copy_(sh.deposit[p][p * slots:(p + 1) * slots])
        torch.cuda.current_stream().synchronize()
        sh.barrier.wait()  # nobody reuses its buffer before every peer copied
        return None

    @staticmethod
    def wait(work):
        return None

    def allreduce(self, flat):
        sh = self.sh
        torch.cuda.current_stream().synchronize()
        sh.deposit[self.rank] = flat.clone()
        sh.barrier.wait()
        total = sh.deposit[0].clone()
        for p in range(1, self.world):
            total += sh.deposit[p]
        sh.barrier.wait()
        flat.copy_(total)
        torch.cuda.current_stream().synchronize()
        return flat


class SimGroup:
    def __init__(self, shared, rank):
        self.sh, self.rank = shared, rank

    def rank_world(self):
        return self.rank, self.sh.world

    def exchange(self, rank, world):
        return SimExchange(self.sh, rank)


def run_ranks(world, fn):
    """fn(rank, group, ops_factory) on `world` threads; returns their results."""
    from paper_2308_12093_b200 import device as d
    from paper_2308_12093_b200 import dist as pd

    sh = _Shared(world)
    out, errs = [None] * world, []

    def ops_for(kind):
        ops = (pd.GatDeviceOps if kind == "gat" else pd.DeviceOps)("cuda:0")
        ops.ctx = d.Context(0, stream=torch.cuda.Stream())  # the rank's own stream
        return ops

    def body(r):
        try:
            torch.cuda.set_device(0)
            out[r] = fn(r, SimGroup(sh, r), ops_for)
            torch.cuda.synchronize()
        except BaseException as ex:  # noqa: BLE001 -- re-raised in the main thread
            errs.append(ex)
            sh.barrier.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    if errs:
        raise errs[0]
    return out


def h64(t):
    return t.detach().double().cpu().numpy()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("scheme", [(0, 0, 0), (0, 1, 0), (1, 0, 0), (1, 1, 0), (2, 2, 1)])
@pytest.mark.parametrize("dtype,tol", [(torch.float64, 1e-12), (torch.float32, 1e-4)])
def test_sim_gcn_layer(orc, world, scheme, dtype, tol):
    from paper_2308_12093_b200 import dist as pd

    n, m, k, fg = 3000, 24, 40, True
    _, s, t = orc.synthetic_graph(n, 7.0, 3)
    op = orc.gcn_operator(n, s, t)
    X = orc.random_uniform(n, m, 11)
    th, bi = orc.gcn_params(m, k, 13)
    G = orc.random_uniform(n, k, 12)
    ref = orc.gcn_layer(op, X, th, bi, scheme, G, fg)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dtype)  # noqa: E731

    def rank(r, group, ops_for):
        layer = pd.DistGcnLayer(n, op.rows, op.cols, op.vals, ops_for("gcn"), dtype, group=group)
        r0, r1 = layer.r0, layer.r1
        out, cache = layer.forward(cu(X[r0:r1]), cu(th), cu(bi), scheme)
        dth, db, dx = layer.backward(cu(G[r0:r1]), cu(th), cache, fg)
        return r0, r1, h64(out), h64(dth), h64(db), h64(dx)

    res = run_ranks(world, rank)
    assert sum(r1 - r0 for r0, r1, *_ in res) == n
    for r0, r1, out, dth, db, dx in res:
        assert orc.max_rel_diff(out, ref[0][r0:r1]) < tol
        assert orc.max_rel_diff(dth, ref[1]) < tol and orc.max_rel_diff(db, ref[2]) < tol
        assert orc.max_rel_diff(dx, ref[3][r0:r1]) < tol


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("exchange", ["stats", "edges"])
@pytest.mark.parametrize("h,k,graph", [(8, 32, "uniform"), (4, 16, "uniform"), (8, 8, "powerlaw")])
def test_sim_gat_layer(orc, world, exchange, h, k, graph):
    """DistGatLayer on the multi-rank layouts, both exchange modes (the
    statistics column pass k_gat_col3 and the shipped-edge column pass), hub
    rows and columns on the power-law graph, against the float64 oracle."""
    from paper_2308_12093_b200 import device as d
    from paper_2308_12093_b200 import dist as pd

    n, m = 2600, 20
    if graph == "powerlaw":
        s, t = d.powerlaw_graph(n, 10.0, 2.1, 9)
        s, t = s.cpu().numpy(), t.cpu().numpy()
    else:
        _, s, t = orc.synthetic_graph(n, 8.0, 6)
    pat = orc.gat_pattern(n, s, t)
    if graph == "powerlaw":
        assert np.diff(pat.rowptr).max() > 500  # hub rows / columns present
    th, a_s, a_d, b = orc.gat_params(m, h, k, 21)
    X = orc.random_uniform(n, m, 11)
    G = orc.random_uniform(n, h * k, 12)
    ref_o = orc.gat_forward(pat, X, th, a_s, a_d, b, h, 0.2)
    ref_g = orc.gat_backward(pat, G, X, th, a_s, a_d, h, 0.2, True)
    f32 = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()  # noqa: E731

    def rank(r, group, ops_for):
        layer = pd.DistGatLayer(n, pat.rowptr, pat.cols, h, k, ops_for("gat"), group=group,
                                exchange=exchange)
        r0, r1 = layer.r0, layer.r1
        out, cache = layer.forward(f32(X[r0:r1]), f32(th), f32(a_s), f32(a_d), f32(b))
        grads = layer.backward(f32(G[r0:r1]), f32(th), f32(a_s), f32(a_d), cache, True)
        return r0, r1, h64(out), [h64(g) for g in grads]

    res = run_ranks(world, rank)
    for r0, r1, out, grads in res:
        assert orc.max_rel_diff(out, ref_o[r0:r1]) < 1e-4
        for g, want in zip(grads[:4], ref_g[:4]):
            assert orc.max_rel_diff(g, want) < 1e-4
        assert orc.max_rel_diff(grads[4], ref_g[4][r0:r1]) < 1e-4


@pytest.mark.parametrize("world", [2, 3])
def test_sim_models(orc, world):
    """DistGcn2 and DistGat2 steps (fused ReLU / ELU paths included) against
    the oracle's Gcn2Model / Gat2Model steps."""
    from paper_2308_12093_b200 import dist as pd

    n, m = 2000, 16
    _, s, t = orc.synthetic_graph(n, 7.0, 2)
    op = orc.gcn_operator(n, s, t)
    pat = orc.gat_pattern(n, s, t)
    X = orc.random_uniform(n, m, 31)
    gp = orc.gcn2_params(m, 24, 6, 7)
    tg = orc.random_uniform(n, 6, 32)
    ap = orc.gat2_params(m, 4, 8, 4, 9)
    ta = orc.random_uniform(n, 16, 33)
    f32 = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()  # noqa: E731
    # reference on the float32-rounded parameters and inputs the device uses
    r32 = lambda a: np.asarray(a, np.float32).astype(np.float64)  # noqa: E731
    g_ref = orc.gcn2_step(op, r32(X), [r32(p) for p in gp], r32(tg), 0, True, True)
    a_ref = orc.gat2_step(pat, r32(X), [r32(p) for p in ap], 4, r32(ta), 0.2, True)

    def rank(r, group, ops_for):
        gl = pd.DistGcnLayer(n, op.rows, op.cols, op.vals, ops_for("gcn"), torch.float32,
                             group=group)
        g2 = pd.DistGcn2(gl, m, 24, 6, 7, caching=True, input_grad=True,
                         params=[f32(p) for p in gp])
        r0, r1 = gl.r0, gl.r1
        gres = g2.train_step(f32(X[r0:r1]), f32(tg[r0:r1]))
        gops = ops_for("gat")
        l1 = pd.DistGatLayer(n, pat.rowptr, pat.cols, 4, 8, gops, group=group)
        l2 = pd.DistGatLayer(n, pat.rowptr, pat.cols, 4, 4, gops, group=group)
        a2 = pd.DistGat2(l1, l2, m, 8, 4, 4, 9, input_grad=True, params=[f32(p) for p in ap])
        ares = a2.train_step(f32(X[r0:r1]), f32(ta[r0:r1]))
        pack = lambda res: (float(res[0]), h64(res[1]), [h64(x) for x in res[2]], h64(res[3]))  # noqa: E731
        return r0, r1, pack(gres), pack(ares), l1.exchange

    res = run_ranks(world, rank)
    for r0, r1, gres, ares, ex in res:
        assert ex == "stats"
        for (loss, out, grads, dx), ref in ((gres, g_ref), (ares, a_ref)):
            rl, rout, rgrads, rdx = ref
            assert abs(loss - rl) <= 1e-4 * max(1.0, abs(rl))
            assert orc.max_rel_diff(out, rout[r0:r1]) < 1e-4
            for g, w in zip(grads, rgrads):
                assert orc.max_rel_diff(g, w) < 1e-4
            assert orc.max_rel_diff(dx, rdx[r0:r1]) < 1e-4
