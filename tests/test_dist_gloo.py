"""Row-partitioned GCN / GAT layers and 2-layer models with
world_size 2..4 over gloo on the CPU.  The partition / all-gather / all-reduce logic of
paper_2308_12093_b200.dist runs unchanged; the per-rank compute backend is a
small CPU implementation injected by the test (the product backend is
libsgnn_cuda.so).  Every rank's row block of the outputs and gradients is
compared with the single-process oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from _cpu_ops import CpuOps


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, root)
        sys.path.insert(0, os.path.join(root, "oracle"))
        import oracle as orc
        from paper_2308_12093_b200 import dist as pd

        n, m, k, scheme, fg = case
        _, s, t = orc.synthetic_graph(n, 6.0, 3)
        op = orc.gcn_operator(n, s, t)
        X = orc.random_uniform(n, m, 11)
        th, bi = orc.gcn_params(m, k, 13)
        G = orc.random_uniform(n, k, 12)
        ref = orc.gcn_layer(op, X, th, bi, scheme, G, fg)
        layer = pd.DistGcnLayer(n, op.rows, op.cols, op.vals, CpuOps(), torch.float64)
        r0, r1 = layer.r0, layer.r1
        out, cache = layer.forward(torch.from_numpy(X[r0:r1]), torch.from_numpy(th),
                                   torch.from_numpy(bi), scheme)
        dth, db, dx = layer.backward(torch.from_numpy(G[r0:r1]), torch.from_numpy(th), cache, fg)
        errs = [orc.max_rel_diff(out.numpy(), ref[0][r0:r1]),
                orc.max_rel_diff(dth.numpy(), ref[1]), orc.max_rel_diff(db.numpy(), ref[2])]
        if fg:
            errs.append(orc.max_rel_diff(dx.numpy(), ref[3][r0:r1]))
        q.put((rank, max(errs), r1 - r0, layer.bounds))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("scheme", [(0, 0, 0), (1, 1, 0), (2, 2, 1), (0, 1, 0), (1, 0, 0)])
@pytest.mark.parametrize("fg", [False, True])
def test_row_partitioned_gcn_matches_single_process(scheme, fg):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, (120, 7, 5, scheme, fg), q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    total = 0
    for rank, err, rows, bounds in results:
        assert err < 1e-12, (rank, err)
        total += rows
    assert total == 120
    assert bounds[0] == 0 and bounds[-1] == 120


def test_partition_rows_balances_nnz():
    from paper_2308_12093_b200.dist import partition_rows, transposed_block

    rng = np.random.default_rng(0)
    deg = rng.integers(1, 50, 1000)
    rowptr = np.concatenate([[0], np.cumsum(deg)])
    for parts in (1, 2, 4, 8):
        b = partition_rows(rowptr, parts)
        assert b[0] == 0 and b[-1] == 1000 and all(b[i] <= b[i + 1] for i in range(parts))
        loads = [rowptr[b[i + 1]] - rowptr[b[i]] for i in range(parts)]
        assert max(loads) - min(loads) <= 2 * deg.max()
    r, c, v = transposed_block(np.array([0, 0, 1, 2]), np.array([1, 2, 0, 1]),
                               np.array([1.0, 2.0, 3.0, 4.0]), 1, 3)
    assert list(r) == [0, 0, 1] and list(c) == [0, 2, 0] and list(v) == [1.0, 4.0, 2.0]


def test_gat_blocks_reproduce_the_csc_view():
    """Host index arrays of the partitioned GAT layer: over the ranks, the
    column blocks are the pattern's CSC (rows ascending within a column) and
    perm points at the right edges of the gathered edge-major layout."""
    from paper_2308_12093_b200.dist import gat_blocks, partition_rows

    rng = np.random.default_rng(3)
    n = 300
    A = (rng.random((n, n)) < 0.03) | np.eye(n, dtype=bool)
    rows, cols = np.nonzero(A)
    rowptr = np.concatenate([[0], np.cumsum(A.sum(1))])
    for world in (1, 2, 3, 4):
        bounds = partition_rows(rowptr, world)
        mx = max(bounds[p + 1] - bounds[p] for p in range(world))
        blocks = [gat_blocks(rowptr, cols, bounds, p) for p in range(world)]
        emx = blocks[0]["emx"]
        canon = {}
        for p, b in enumerate(blocks):
            for i in range(b["edges"]):
                canon[p * emx + i] = rowptr[bounds[p]] + i
        for p, b in enumerate(blocks):
            r0 = bounds[p]
            assert np.array_equal(b["rowptr"], rowptr[r0:bounds[p + 1] + 1] - rowptr[r0])
            for jl in range(bounds[p + 1] - r0):
                j = r0 + jl
                lo, hi = b["colptr"][jl], b["colptr"][jl + 1]
                want = list(np.nonzero(A[:, j])[0])
                got = [bounds[q // mx] + q % mx for q in b["rows"][lo:hi]]
                assert got == want
                for q, r in zip(b["perm"][lo:hi], want):
                    e = canon[int(q)]
                    assert rows[e] == r and cols[e] == j


# ---------------------------------------------------------------------------
# partitioned GAT layer and the 2-layer models
# ---------------------------------------------------------------------------
def _gat_worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, root)
        sys.path.insert(0, os.path.join(root, "oracle"))
        import oracle as orc
        from _cpu_ops import GatCpuOps
        from paper_2308_12093_b200 import dist as pd

        kind, n, m, h, k, exchange, fg = case
        _, s, t = orc.synthetic_graph(n, 6.0, 5)
        pat = orc.gat_pattern(n, s, t)
        ops = GatCpuOps()
        T = torch.from_numpy
        if kind == "layer":
            layer = pd.DistGatLayer(n, pat.rowptr, pat.cols, h, k, ops, exchange=exchange)
            r0, r1 = layer.r0, layer.r1
            th, a_s, a_d, b = orc.gat_params(m, h, k, 21)
            X = orc.random_uniform(n, m, 11)
            G = orc.random_uniform(n, h * k, 12)
            out, cache = layer.forward(T(X[r0:r1]), T(th), T(a_s), T(a_d), T(b))
            grads = layer.backward(T(G[r0:r1]), T(th), T(a_s), T(a_d), cache, fg)
            ref_o = orc.gat_forward(pat, X, th, a_s, a_d, b, h, 0.2)
            ref_g = orc.gat_backward(pat, G, X, th, a_s, a_d, h, 0.2, fg)
            errs = [orc.max_rel_diff(out.numpy(), ref_o[r0:r1])]
            errs += [orc.max_rel_diff(g.numpy(), r) for g, r in zip(grads[:4], ref_g[:4])]
            if fg:
                errs.append(orc.max_rel_diff(grads[4].numpy(), ref_g[4][r0:r1]))
            q.put((rank, max(errs), r1 - r0, layer.exchange))
        elif kind == "gat2":
            hid, o = k, 3
            l1 = pd.DistGatLayer(n, pat.rowptr, pat.cols, h, hid, ops, exchange=exchange)
            l2 = pd.DistGatLayer(n, pat.rowptr, pat.cols, h, o, ops, exchange=exchange)
            prm = orc.gat2_params(m, h, hid, o, 7)
            model = pd.DistGat2(l1, l2, m, hid, o, h, 7, input_grad=fg,
                                params=[T(p) for p in prm])
            r0, r1 = l1.r0, l1.r1
            X = orc.random_uniform(n, m, 18)
            tgt = orc.random_uniform(n, h * o, 19)
            loss, out, grads, dx = model.train_step(T(X[r0:r1]), T(tgt[r0:r1]))
            rl, rout, rgrads, rdx = orc.gat2_step(pat, X, prm, h, tgt, 0.2, fg)
            errs = [abs(float(loss) - rl) / max(1.0, abs(rl)),
                    orc.max_rel_diff(out.numpy(), rout[r0:r1])]
            errs += [orc.max_rel_diff(g.numpy(), r) for g, r in zip(grads, rgrads)]
            if fg:
                errs.append(orc.max_rel_diff(dx.numpy(), rdx[r0:r1]))
            q.put((rank, max(errs), r1 - r0, exchange))
        else:  # gcn2
            op = orc.gcn_operator(n, s, t)
            layer = pd.DistGcnLayer(n, op.rows, op.cols, op.vals, ops, torch.float64)
            hid, o = k, 4
            prm = orc.gcn2_params(m, hid, o, 9)
            model = pd.DistGcn2(layer, m, hid, o, 9, caching=True, input_grad=fg,
                                params=[T(p) for p in prm])
            r0, r1 = layer.r0, layer.r1
            X = orc.random_uniform(n, m, 20)
            tgt = orc.random_uniform(n, o, 21)
            loss, out, grads, dx = model.train_step(T(X[r0:r1]), T(tgt[r0:r1]))
            rl, rout, rgrads, rdx = orc.gcn2_step(op, X, prm, tgt, 0, True, fg)
            errs = [abs(float(loss) - rl) / max(1.0, abs(rl)),
                    orc.max_rel_diff(out.numpy(), rout[r0:r1])]
            errs += [orc.max_rel_diff(g.numpy(), r) for g, r in zip(grads, rgrads)]
            if fg:
                errs.append(orc.max_rel_diff(dx.numpy(), rdx[r0:r1]))
            q.put((rank, max(errs), r1 - r0, None))
    finally:
        dist.destroy_process_group()


def _run(world, case, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gat_worker, args=(r, world, port, case, q))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sum(r[2] for r in results) == n
    return results


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("exchange", ["stats", "edges"])
@pytest.mark.parametrize("h,k", [(4, 3), (2, 5)])
def test_row_partitioned_gat_layer(world, exchange, h, k):
    """DistGatLayer over gloo: each rank's rows of out / dX and the
    all-reduced dTheta, dA_src, dA_dst, db against the single-process oracle,
    shipping either per-row statistics (alpha / dy rebuilt in the column pass)
    or the edge values."""
    n = 90
    for rank, err, _, ex in _run(world, ("layer", n, 6, h, k, exchange, True), n):
        assert ex == exchange
        assert err < 1e-12, (rank, err)


@pytest.mark.parametrize("world", [2, 3])
def test_row_partitioned_gat2_step(world):
    """DistGat2 (Gat2Model over the partition: GAT -> ELU -> GAT, MSE) against
    the oracle's Gat2Model step (pinned to the reference's)."""
    n = 80
    for rank, err, _, _ in _run(world, ("gat2", n, 5, 2, 3, "stats", True), n):
        assert err < 1e-12, (rank, err)


@pytest.mark.parametrize("world", [2, 4])
def test_row_partitioned_gcn2_step(world):
    """DistGcn2 against the oracle's Gcn2Model step (pinned to the reference's)."""
    n = 100
    for rank, err, _, _ in _run(world, ("gcn2", n, 6, 1, 5, None, True), n):
        assert err < 1e-12, (rank, err)
