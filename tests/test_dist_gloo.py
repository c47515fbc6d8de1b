"""Row-partitioned GCN layer with world_size 2 over gloo on the
CPU.  The partition / all-gather / all-reduce logic of
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


class CpuOps:
    """Test-only backend: CSR SpMM in stored order, numpy GEMMs, float64."""

    class Adj:
        def __init__(self, n_rows, rows, cols, vals):
            self.rowptr = np.zeros(n_rows + 1, np.int64)
            np.add.at(self.rowptr, np.asarray(rows, np.int64) + 1, 1)
            self.rowptr = np.cumsum(self.rowptr)
            self.cols, self.vals = np.asarray(cols), np.asarray(vals, np.float64)

    def adjacency(self, n_rows, n_cols, rows, cols, vals, dtype):
        return CpuOps.Adj(n_rows, rows, cols, vals)

    def spmm(self, adj, B, bias=None):
        B = B.numpy()
        out = np.zeros((len(adj.rowptr) - 1, B.shape[1]))
        for i in range(len(adj.rowptr) - 1):
            for e in range(adj.rowptr[i], adj.rowptr[i + 1]):
                out[i] += adj.vals[e] * B[adj.cols[e]]
        t = torch.from_numpy(out)
        return t if bias is None else t + bias

    def empty(self, rows, cols, dtype):
        return torch.empty((rows, cols), dtype=dtype)

    def gemm(self, A, B, ta=False, tb=False, bias=None, out=None, colsum_b=None):
        a = A.T if ta else A
        b = B.T if tb else B
        r = a @ b
        if bias is not None:
            r = r + bias
        if colsum_b is not None:
            colsum_b.copy_(B.sum(0))
        if out is None:
            return r
        out.copy_(r)
        return out

    def colsum(self, X):
        return X.sum(0)


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
