"""Generate tests/golden/*.npz by running the REFERENCE itself.

Runs only in the build container (needs /root/reference to have built
oracle/_ref/libsgnn_ref.so).  Inputs are produced by the reference's own
generators (synthetic_graph, DenseMatrix::random_uniform, GcnParams/GatParams
init) or by a fixed numpy RNG and stored next to the outputs, so the tests
can rebuild every case from the fixture alone.  Re-run with
    make -C oracle && python oracle/gen_golden.py
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import refpy  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests",
                   "golden")
L = refpy.load()
L.ref_set_num_threads(1)


def save(name, **arrays):
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **arrays)
    print("wrote", name, {k: np.asarray(v).shape for k, v in arrays.items()})


def ref_graph(n, deg, seed):
    ne = L.ref_synthetic_graph(n, deg, seed, None, None)
    src, dst = np.empty(ne, np.int32), np.empty(ne, np.int32)
    L.ref_synthetic_graph(n, deg, seed, src.ctypes.data_as(C.c_void_p),
                          dst.ctypes.data_as(C.c_void_p))
    return src, dst


def ref_uniform(r, c, seed, lo=-1.0, hi=1.0):
    o = np.empty((r, c))
    L.ref_random_uniform(r, c, seed, lo, hi, o)
    return o


def ref_canon(nr, nc, r, c, v):
    q = len(r)
    ro, co, vo = np.empty(q, np.int32), np.empty(q, np.int32), np.empty(q)
    w = L.ref_coo_canonicalize(nr, nc, q, r, c, v, ro, co, vo)
    assert w >= 0
    return ro[:w], co[:w], vo[:w]


def ref_normalize(n, r, c, v):
    q = len(r)
    ro, co, vo = np.empty(q + n, np.int32), np.empty(q + n, np.int32), np.empty(q + n)
    w = L.ref_gcn_normalize(n, q, r, c, v, ro, co, vo)
    assert w >= 0
    return ro[:w], co[:w], vo[:w]


def ref_csr_csc(nr, nc, r, c, v):
    rp, cp = np.empty(nr + 1, np.int32), np.empty(nc + 1, np.int32)
    cr, cv = np.empty(len(r), np.int32), np.empty(len(r))
    L.ref_csr_csc(nr, nc, len(r), r, c, v, rp, cp, cr, cv)
    return rp, cp, cr, cv


def ref_pattern(n, rp, cols):
    q = int(rp[n])
    cp, rows, perm, diag = (np.empty(n + 1, np.int32), np.empty(q, np.int32),
                            np.empty(q, np.int32), np.empty(n, np.int32))
    flag = L.ref_pattern(n, rp, cols, cp, rows, perm, diag)
    return cp, rows, perm, diag, flag


def vp(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def main():
    rng = np.random.default_rng(20230823)

    # -- rng.hpp / dense.hpp:45-53 --------------------------------------------
    save("rng", u_7x5_s42=ref_uniform(7, 5, 42), u_3x11_s0_pm2=ref_uniform(3, 11, 0, -2, 2),
         u_1x1000_s99=ref_uniform(1, 1000, 99, 0.0, 1.0))

    # -- graph.hpp:160-190 ------------------------------------------------------
    s1, d1 = ref_graph(500, 6.0, 7)
    s2, d2 = ref_graph(2708, 10556 / 2708, 1)  # Cora-shaped
    s3, d3 = ref_graph(97, 3.3, 123)
    save("synthetic_graph", src_500_6_7=s1, dst_500_6_7=d1, src_cora_1=s2, dst_cora_1=d2,
         src_97_3p3_123=s3, dst_97_3p3_123=d3)

    # -- sparse.hpp: canonicalize (dups keep last), normalize, csr/csc ---------
    nr, nc, q = 40, 33, 400
    r = rng.integers(0, nr, q).astype(np.int32)
    c = rng.integers(0, nc, q).astype(np.int32)
    v = rng.uniform(0.1, 1.0, q)
    cr, cc, cv = ref_canon(nr, nc, r, c, v)
    rp, cp, crows, cvals = ref_csr_csc(nr, nc, cr, cc, cv)
    # square weighted graph for normalize (with some explicit diagonal values)
    n = 60
    qr = rng.integers(0, n, 420).astype(np.int32)
    qc = rng.integers(0, n, 420).astype(np.int32)
    qv = rng.uniform(0.1, 1.0, 420)
    nr_, nc_, nv_ = ref_normalize(n, qr, qc, qv)
    nq = len(nr_)
    nv32 = np.empty(nq, np.float32)
    r32, c32 = np.empty(nq, np.int32), np.empty(nq, np.int32)
    L.ref_gcn_normalize_f32(n, len(qr), qr, qc, qv.astype(np.float32), r32, c32, nv32)
    save("sparse", in_rows=r, in_cols=c, in_vals=v, n_rows=nr, n_cols=nc, canon_rows=cr,
         canon_cols=cc, canon_vals=cv, rowptr=rp, colptr=cp, csc_rows=crows, csc_vals=cvals,
         norm_n=n, norm_in_rows=qr, norm_in_cols=qc, norm_in_vals=qv, norm_rows=nr_,
         norm_cols=nc_, norm_vals=nv_, norm_vals_f32=nv32)

    # -- pattern.hpp:19-59 on a graph with and without all self loops ----------
    gs, gd = ref_graph(50, 4.0, 5)
    pr, pc, pv = ref_canon(50, 50, gs, gd, np.ones(len(gs)))
    prp, _, _, _ = ref_csr_csc(50, 50, pr, pc, pv)
    pat0 = ref_pattern(50, prp, pc)
    lr, lc, lv = ref_normalize(50, gs, gd, np.ones(len(gs)))  # has all self loops
    lrp, _, _, _ = ref_csr_csc(50, 50, lr, lc, lv)
    pat1 = ref_pattern(50, lrp, lc)
    save("pattern", rowptr0=prp, cols0=pc, colptr0=pat0[0], rows0=pat0[1], perm0=pat0[2],
         diag0=pat0[3], all0=pat0[4], rowptr1=lrp, cols1=lc, colptr1=pat1[0], rows1=pat1[1],
         perm1=pat1[2], diag1=pat1[3], all1=pat1[4])

    # -- kernels.hpp: spmm in every format (f64 and f32), sddmm, softmax -------
    f = 9
    B = rng.standard_normal((nc, f))
    outs = {}
    for name, fmt in [("coo", 0), ("csr", 1), ("csc", 2), ("ellpack", 3), ("hybrid", 4)]:
        Cm = np.empty((nr, f))
        assert L.ref_spmm(fmt, nr, nc, len(r), r, c, v, B, f, Cm) == 0
        outs["C_" + name] = Cm
    B32 = rng.standard_normal((nc, 33)).astype(np.float32)
    v32 = v.astype(np.float32)
    C32 = np.empty((nr, 33), np.float32)
    assert L.ref_spmm_f32(1, nr, nc, len(r), r, c, v32, B32, 33, C32) == 0
    # sddmm on a square pattern
    sn = 30
    sr = rng.integers(0, sn, 150).astype(np.int32)
    sc = rng.integers(0, sn, 150).astype(np.int32)
    SB = rng.standard_normal((sn, 5))
    SC = rng.standard_normal((5, sn))
    svals = np.empty(150)
    sq = L.ref_sddmm(sn, 150, sr, sc, SB, 5, SC, svals)
    # edge softmax incl. +-500 scores (needs self loops)
    er = np.concatenate([sr, np.arange(sn, dtype=np.int32)])
    ec = np.concatenate([sc, np.arange(sn, dtype=np.int32)])
    er_c, ec_c, _ = ref_canon(sn, sn, er, ec, np.ones(len(er)))
    scores = rng.uniform(-500, 500, len(er_c))
    alpha = np.empty(len(er_c))
    assert L.ref_edge_softmax(sn, len(er), er, ec, scores, alpha) == 0
    save("kernels", rows=r, cols=c, vals=v, n_rows=nr, n_cols=nc, B=B, B32=B32, C32=C32,
         sddmm_n=sn, sddmm_rows=sr, sddmm_cols=sc, sddmm_B=SB, sddmm_C=SC,
         sddmm_vals=svals[:sq], softmax_rows=er, softmax_cols=ec, softmax_scores=scores,
         softmax_alpha=alpha, **outs)

    # -- cost.hpp: selector grid + cost formulas -------------------------------
    ms = np.array([1 << i for i in range(11)], np.int64)
    ks = np.arange(1, 1025, dtype=np.int64)
    sel = np.zeros((3, len(ms), len(ks), 2, 2, 3), np.int8)
    a, b, cch = C.c_int(), C.c_int(), C.c_int()
    for pi in range(3):
        for mi, m in enumerate(ms):
            for ki, k in enumerate(ks):
                for fg in (0, 1):
                    for ca in (0, 1):
                        L.ref_select_scheme(pi, int(m), int(k), fg, ca, C.byref(a), C.byref(b),
                                            C.byref(cch))
                        sel[pi, mi, ki, fg, ca] = (a.value, b.value, cch.value)
    costs = []
    fl, by, oi = C.c_longlong(), C.c_longlong(), C.c_double()
    for fn_i, fn in enumerate([L.ref_spmm_cost, L.ref_sddmm_cost]):
        for (nn, qq, pp) in [(2708, 10556, 168), (169343, 1166243, 436), (100, 0, 3)]:
            for fmt in range(4):
                for ff in (1, 8, 64, 256):
                    for sb in (4, 8):
                        rc = fn(fmt, nn, qq, pp, ff, sb, 4, C.byref(fl), C.byref(by),
                                C.byref(oi))
                        costs.append((fn_i, nn, qq, pp, fmt, ff, sb, rc, fl.value, by.value,
                                      oi.value))
    save("cost", ms=ms, ks=ks, select=sel, costs=np.array(costs, np.float64))

    # -- gcn.hpp: one layer, every scheme combination, f64 ---------------------
    gn = 64
    gsrc, gdst = ref_graph(gn, 5.0, 3)
    Ar, Ac, Av = ref_normalize(gn, gsrc, gdst, np.ones(len(gsrc)))
    gcn = {"n": gn, "rows": Ar, "cols": Ac, "vals": Av}
    for (m, k) in [(7, 5), (5, 9)]:
        X = ref_uniform(gn, m, 11)
        th, bi = np.empty((m, k)), np.empty(k)
        L.ref_gcn_params(m, k, 13, th, bi)
        G = ref_uniform(gn, k, 12)
        gcn[f"X_{m}_{k}"], gcn[f"theta_{m}_{k}"], gcn[f"bias_{m}_{k}"], gcn[f"G_{m}_{k}"] = \
            X, th, bi, G
        for (fw, bw, ca) in [(0, 0, 0), (0, 1, 0), (1, 0, 0), (1, 1, 0), (2, 2, 1)]:
            for fmt in (1, 2):
                for fg in (0, 1):
                    o, dth, db, dx = np.empty((gn, k)), np.empty((m, k)), np.empty(k), \
                        np.empty((gn, m))
                    assert L.ref_gcn_layer(gn, len(Ar), Ar, Ac, Av, fmt, X, m, th, bi, k, fw,
                                           bw, ca, vp(G), fg, o, vp(dth), vp(db), vp(dx)) == 0
                    tag = f"{m}_{k}_{fw}{bw}_{fmt}_{fg}"
                    gcn["out_" + tag], gcn["dtheta_" + tag], gcn["dbias_" + tag] = o, dth, db
                    if fg:
                        gcn["dinput_" + tag] = dx
    save("gcn", **gcn)

    # -- Cora-shaped config 1 (1433 -> 16, CSC, caching) -----------------------
    cn, cm, ck = 2708, 1433, 16
    Cr, Cc, Cv = ref_normalize(cn, s2, d2, np.ones(len(s2)))
    X = ref_uniform(cn, cm, 11)
    th, bi = np.empty((cm, ck)), np.empty(ck)
    L.ref_gcn_params(cm, ck, 13, th, bi)
    G = ref_uniform(cn, ck, 12)
    L.ref_select_scheme(0, cm, ck, 1, 1, C.byref(a), C.byref(b), C.byref(cch))
    o, dth, db, dx = np.empty((cn, ck)), np.empty((cm, ck)), np.empty(ck), np.empty((cn, cm))
    assert L.ref_gcn_layer(cn, len(Cr), Cr, Cc, Cv, 2, X, cm, th, bi, ck, a.value, b.value,
                           cch.value, vp(G), 1, o, vp(dth), vp(db), vp(dx)) == 0
    save("gcn_cora", nnz=len(Cr), scheme=np.array([a.value, b.value, cch.value]), out=o,
         dtheta=dth, dbias=db, dinput_colsum=dx.sum(axis=0), dinput_rows=dx[::97].copy(),
         norm_vals_sample=Cv[::13].copy())

    # -- gat.hpp: one multi-head layer, every cache level ----------------------
    an, am, ah, ak = 40, 6, 3, 4
    asrc, adst = ref_graph(an, 4.0, 9)
    base_r, base_c, base_v = ref_canon(an, an, asrc, adst, np.ones(len(asrc)))
    # add_self_loops == normalize's structure; the pattern only needs the structure
    lr, lc, _ = ref_normalize(an, asrc, adst, np.ones(len(asrc)))
    arp, _, _, _ = ref_csr_csc(an, an, lr, lc, np.ones(len(lr)))
    X = ref_uniform(an, am, 21)
    th, a_s, a_d, bi = np.empty((am, ah * ak)), np.empty((ah, ak)), np.empty((ah, ak)), \
        np.empty(ah * ak)
    L.ref_gat_params(am, ah, ak, 23, th, a_s, a_d, bi)
    G = ref_uniform(an, ah * ak, 22)
    gat = {"n": an, "rowptr": arp, "cols": lc, "X": X, "theta": th, "a_src": a_s,
           "a_dst": a_d, "bias": bi, "G": G, "heads": ah, "k": ak, "beta": 0.2}
    q = len(lc)
    for level in range(4):
        o = np.empty((an, ah * ak))
        al, mk = np.empty((ah, q)), np.empty((ah, q), np.uint8)
        dth, das, dad, db, dx = np.empty((am, ah * ak)), np.empty((ah, ak)), np.empty((ah, ak)), \
            np.empty(ah * ak), np.empty((an, am))
        assert L.ref_gat_layer(an, arp, lc, X, am, th, a_s, a_d, bi, ah, ak, 0.2, level,
                               vp(G), 1, o, vp(al), vp(mk), vp(dth), vp(das), vp(dad), vp(db),
                               vp(dx)) == 0
        for nm, arr in [("out", o), ("alpha", al), ("mask", mk), ("dtheta", dth),
                        ("da_src", das), ("da_dst", dad), ("dbias", db), ("dinput", dx)]:
            gat[f"{nm}_{level}"] = arr
    save("gat", **gat)


# two-layer models (model.hpp): (kind, n, deg, seed, m, hidden, out, heads,
# policy, caching, level, input_grad)
MODEL_CASES = {
    "gcn2_adaptive_cached": (0, 300, 6.0, 5, 12, 16, 5, 1, 0, 1, 0, 0),
    "gcn2_adaptive_fg": (0, 300, 6.0, 5, 12, 16, 5, 1, 0, 0, 0, 1),
    "gcn2_tf": (0, 250, 4.0, 9, 20, 8, 3, 1, 1, 0, 0, 1),
    "gat2_h2": (1, 200, 5.0, 7, 10, 4, 3, 2, 0, 0, 3, 1),
    "gat2_h8": (1, 220, 6.0, 3, 16, 8, 4, 8, 0, 0, 3, 0),
}


def models():
    out = {}
    for tag, (kind, n, deg, seed, m, hid, o, h, pol, ca, lv, ig) in MODEL_CASES.items():
        ow = o if kind == 0 else h * o
        sizes = ([m * hid, hid, hid * o, o] if kind == 0 else
                 [m * h * hid, h * hid, h * hid, h * hid, h * hid * h * o, h * o, h * o, h * o])
        loss = C.c_double()
        pred = np.empty((n, ow))
        grads = np.empty(sum(sizes))
        assert L.ref_model_step(kind, n, deg, seed, m, hid, o, h, pol, ca, lv, ig,
                                C.byref(loss), pred, grads) == 0, L.ref_last_error()
        out[f"{tag}_loss"] = np.array([loss.value])
        out[f"{tag}_pred"] = pred
        out[f"{tag}_grads"] = grads
        out[f"{tag}_cfg"] = np.array([kind, n, seed, m, hid, o, h, pol, ca, lv, ig], np.int64)
        out[f"{tag}_deg"] = np.array([deg])
    save("models", **out)


if __name__ == "__main__":
    if sys.argv[1:] == ["models"]:
        models()
    else:
        main()
        models()
