"""Test-only CPU backends for the row-partitioned layers (paper_2308_12093_b200.dist):
float64 numpy restatements of each block entry point's contract, so the
partition / exchange / all-reduce logic runs unchanged under gloo on the CPU.
The product backends are DeviceOps / GatDeviceOps (libsgnn_cuda.so)."""
import numpy as np
import torch


def _n(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


class CpuOps:
    """GCN pieces: CSR SpMM in stored order, numpy GEMMs, float64."""

    class Adj:
        def __init__(self, n_rows, rows, cols, vals):
            rows = _n(rows).astype(np.int64)
            self.rowptr = np.zeros(n_rows + 1, np.int64)
            np.add.at(self.rowptr, rows + 1, 1)
            self.rowptr = np.cumsum(self.rowptr)
            self.cols, self.vals = _n(cols).astype(np.int64), _n(vals).astype(np.float64)

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
        return torch.empty((rows, cols), dtype=torch.float64 if dtype.is_floating_point else dtype)

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

    # model pieces (dense.hpp:196-270, model.hpp loss_mse)
    def activation(self, X, kind, out=None):
        x = X.numpy()
        if kind == "relu":
            h = np.where(x > 0, x, 0.0)
        else:
            h = np.where(x > 0, x, np.expm1(x))
        mask = torch.from_numpy((x > 0).astype(np.uint8))
        h = torch.from_numpy(h)
        if out is not None:
            out.copy_(h)
            h = out
        return h, mask

    def activation_backward(self, g, mask, kind, saved=None, out=None):
        gg, m = g.numpy(), mask.numpy().astype(bool)
        if kind == "relu":
            r = np.where(m, gg, 0.0)
        else:
            r = np.where(m, gg, gg * (saved.numpy() + 1.0))
        r = torch.from_numpy(r)
        if out is not None:
            out.copy_(r)
            r = out
        return r

    def mask(self, rows, cols):
        return torch.empty((rows, cols), dtype=torch.uint8)

    def gemm_act(self, A, B, act, mask, ta=False, tb=False, bias=None, saved=None):
        r = self.gemm(A, B, ta, tb, bias=bias)
        if act == "relu":
            r, m = self.activation(r, "relu", out=r)
            mask.copy_(m)
            return r
        return self.activation_backward(r, mask, "relu" if act == "relu_backward" else "elu",
                                        saved=saved)

    def loss_mse(self, out, target, total):
        d = out.numpy() - target.numpy()
        return torch.tensor(float((d * d).sum()) / total, dtype=torch.float64), \
            torch.from_numpy(2.0 * d / total)


def _lrelu(y, beta):
    return np.where(y > 0, y, beta * y)


class GatCpuOps(CpuOps):
    """The sgnn_gat_* block entry points restated in float64."""

    def index(self, a):
        return torch.from_numpy(_n(a).astype(np.int64))

    def rowplan(self, n_rows, rowptr):
        return None

    def free_rowplan(self, h):
        pass

    def stats_supported(self, h, k):
        return True

    def transform(self, X, theta, h, k, a_src, a_dst, M, s, d):
        m = (X @ theta).numpy()
        M.copy_(torch.from_numpy(m))
        m3 = m.reshape(len(m), h, k)
        s.copy_(torch.from_numpy((m3 * a_src.numpy()[None]).sum(-1)))
        d.copy_(torch.from_numpy((m3 * a_dst.numpy()[None]).sum(-1)))

    def attention(self, nl, rowptr, cols, h, s, d, beta, alpha, mask, stats, plan):
        rp, cl = rowptr.numpy(), cols.numpy()
        s, d = s.numpy(), d.numpy()
        a, mk = alpha.numpy(), mask.numpy()
        st = stats.numpy() if stats is not None else None
        for i in range(nl):
            es = slice(rp[i], rp[i + 1])
            y = s[i][None, :] + d[cl[es]]
            w = _lrelu(y, beta)
            mx = w.max(0)
            ex = np.exp(w - mx)
            inv = 1.0 / ex.sum(0)
            a[es] = ex * inv
            mk[es] = (y > 0).astype(np.uint8)
            if st is not None:  # [row][head][4] = (s, max, 1 / sum, dot)
                q = st[i].reshape(h, 4)
                q[:, 0], q[:, 1], q[:, 2] = s[i], mx, inv

    def aggregate(self, nl, rowptr, cols, h, k, alpha, M, bias, out, plan):
        rp, cl, a = rowptr.numpy(), cols.numpy(), alpha.numpy()
        M3 = M.numpy().reshape(M.shape[0], h, k)
        o = out.numpy().reshape(nl, h, k)
        for i in range(nl):
            es = slice(rp[i], rp[i + 1])
            o[i] = (a[es][:, :, None] * M3[cl[es]]).sum(0)
        o += bias.numpy().reshape(1, h, k)

    def sddmm(self, nl, rowptr, cols, h, k, M, G, da, plan):
        rp, cl = rowptr.numpy(), cols.numpy()
        M3 = M.numpy().reshape(M.shape[0], h, k)
        G3 = G.numpy().reshape(G.shape[0], h, k)
        out = da.numpy()
        for i in range(nl):
            es = slice(rp[i], rp[i + 1])
            out[es] = (G3[i][None] * M3[cl[es]]).sum(-1)

    def softmax_backward(self, nl, rowptr, h, alpha, mask, da, beta, dy, dS, stats, plan):
        rp, a, g, mk = rowptr.numpy(), alpha.numpy(), da.numpy(), mask.numpy()
        y, ds = dy.numpy(), dS.numpy()
        st = stats.numpy() if stats is not None else None
        for i in range(nl):
            es = slice(rp[i], rp[i + 1])
            dot = (a[es] * g[es]).sum(0)
            dw = a[es] * (g[es] - dot)
            y[es] = np.where(mk[es] > 0, dw, beta * dw)
            ds[i] = y[es].sum(0)
            if st is not None:
                st[i].reshape(h, 4)[:, 3] = dot

    def _finish(self, j, h, k, acc, dd, dS, a_src, a_dst, dD, dM):
        dD.numpy()[j] = dd
        o = acc + dS.numpy()[j][:, None] * a_src.numpy() + dd[:, None] * a_dst.numpy()
        dM.numpy()[j] = o.reshape(-1)

    def column_pass(self, nl, colptr, rows, perm, h, k, G, alpha, dy, dS, a_src, a_dst, dD, dM,
                    plan):
        cp, rw, pm = colptr.numpy(), rows.numpy(), perm.numpy()
        G3 = G.numpy().reshape(G.shape[0], h, k)
        a, y = alpha.numpy(), dy.numpy()
        for j in range(nl):
            ps = slice(cp[j], cp[j + 1])
            acc = (a[pm[ps]][:, :, None] * G3[rw[ps]]).sum(0)
            self._finish(j, h, k, acc, y[pm[ps]].sum(0), dS, a_src, a_dst, dD, dM)

    def column_pass_stats(self, nl, colptr, rows, h, k, G, stats, d_own, M_own, beta, dS,
                          a_src, a_dst, dD, dM, plan):
        cp, rw = colptr.numpy(), rows.numpy()
        G3 = G.numpy().reshape(G.shape[0], h, k)
        M3 = M_own.numpy().reshape(M_own.shape[0], h, k)
        st, dj = stats.numpy(), d_own.numpy()
        for j in range(nl):
            r = rw[cp[j]:cp[j + 1]]
            q4 = st[r].reshape(len(r), h, 4)
            s, mx, inv, dot = (q4[:, :, q] for q in range(4))
            y = s + dj[j][None]
            a = np.exp(_lrelu(y, beta) - mx) * inv
            dalpha = (G3[r] * M3[j][None]).sum(-1)
            dw = a * (dalpha - dot)
            dyv = np.where(y > 0, dw, beta * dw)
            acc = (a[:, :, None] * G3[r]).sum(0)
            self._finish(j, h, k, acc, dyv.sum(0), dS, a_src, a_dst, dD, dM)

    def param_grads(self, nl, h, k, G, M, dS, dD, d_b, d_as, d_ad):
        G_, M3 = G.numpy(), M.numpy().reshape(nl, h, k)
        d_b.copy_(torch.from_numpy(G_.sum(0)))
        d_as.copy_(torch.from_numpy((dS.numpy()[:, :, None] * M3).sum(0)))
        d_ad.copy_(torch.from_numpy((dD.numpy()[:, :, None] * M3).sum(0)))
