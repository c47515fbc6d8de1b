"""CPU-only checks of the C-ABI library: it loads without a GPU, exports every
symbol include/sgnn_cuda.h declares, and its host-pure entry points (scheme
selector, analytic cost model, synthetic graph generator) are bit-identical to
the reference golden vectors.  No device compute is called here."""
import itertools
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "sgnn_cuda.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sgnn_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2308_12093_b200 import _capi

    declared = _declared()
    assert len(declared) >= 45
    for name in declared:
        assert hasattr(_capi.lib, name), name
    assert set(declared) == set(_capi.SYMBOLS)
    assert "sm_100a" in _capi.version()


def test_library_is_sm100a_fatbin():
    import subprocess

    so = os.path.join(ROOT, "paper_2308_12093_b200", "libsgnn_cuda.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_selector_matches_reference_grid(golden):
    from paper_2308_12093_b200 import device as d

    g = golden("cost")
    sel = g["select"]
    pol = ["adaptive", "transform-first", "propagate-first"]
    for pi, (mi, m) in itertools.product(range(3), enumerate(g["ms"])):
        for ki, k in enumerate(g["ks"]):
            for fg, ca in itertools.product((0, 1), (0, 1)):
                s = d.resolve_scheme(pol[pi], int(m), int(k), fg, ca)
                assert (s.forward, s.backward, s.caching) == tuple(sel[pi, mi, ki, fg, ca])
    with pytest.raises(ValueError, match="m and k must be >= 1"):
        d.resolve_scheme("adaptive", 0, 4)
    with pytest.raises(ValueError, match="unknown scheme"):
        d.resolve_scheme("bogus", 4, 4)


def test_cost_model_matches_reference(golden):
    from paper_2308_12093_b200 import sgnn

    g = golden("cost")
    names = ["coo", "csr", "csc", "ellpack"]
    for fn_i, n, q, p, fmt, f, sb, rc, fl, by, oi in g["costs"]:
        fn = sgnn.spmm_cost if fn_i == 0 else sgnn.sddmm_cost
        args = (names[int(fmt)], int(n), int(q), int(p), int(f), int(sb))
        if rc != 0:
            with pytest.raises(ValueError):
                fn(*args)
            continue
        got = fn(*args)
        assert (got["flops"], got["bytes"], got["operational_intensity"]) == (int(fl), int(by), oi)
    # reference python smoke values (tests/python/test_smoke.py:34-51)
    assert abs(sgnn.spmm_cost("csr", 169343, 1166243, f=64)["operational_intensity"] - 1.066) <= .005
    assert abs(sgnn.spmm_cost("ellpack", 2708, 10556, p=168, f=64)["operational_intensity"]
               - 0.236) <= 0.005
    assert sgnn.gat_cache_footprint("none", 3, 2, 4, 5) == 0
    assert sgnn.gat_cache_footprint("full", 3, 2, 4, 5) == 146
    with pytest.raises(ValueError):
        sgnn.gat_cache_footprint("bogus", 3, 2, 4, 5)


def test_flop_and_transient_formulas(orc):
    from paper_2308_12093_b200._capi import lib

    for s, (n, m, k, q) in itertools.product(range(3), [(4, 2, 3, 6), (1000, 128, 256, 5000)]):
        assert lib.sgnn_gcn_forward_flops(s, n, m, k, q) == orc.gcn_forward_flops(s, n, m, k, q)
        assert lib.sgnn_gcn_forward_transients(s, n, m, k) == \
            orc.gcn_forward_transients(s, n, m, k)
        for fg in (0, 1):
            assert lib.sgnn_gcn_backward_flops(s, n, m, k, q, fg) == \
                orc.gcn_backward_flops(s, n, m, k, q, fg)
            assert lib.sgnn_gcn_backward_transients(s, n, m, k, fg) == \
                orc.gcn_backward_transients(s, n, m, k, fg)
    assert lib.sgnn_gcn_forward_flops(0, 4, 2, 3, 6) == 84  # test_cost.cpp:148


@pytest.mark.parametrize("n,deg,seed,tag", [(500, 6.0, 7, "500_6_7"),
                                            (2708, 10556 / 2708, 1, "cora_1")])
def test_synthetic_graph_bit_exact(golden, n, deg, seed, tag):
    from paper_2308_12093_b200 import sgnn

    g = golden("synthetic_graph")
    n2, s, d = sgnn.synthetic_graph(n, deg, seed)
    assert n2 == n
    assert np.array_equal(s, g["src_" + tag]) and np.array_equal(d, g["dst_" + tag])


def test_synthetic_graph_arxiv_edge_count():
    from paper_2308_12093_b200._capi import lib

    # the generator is symmetric: 1,166,243 requested -> 2 * 583,122 pairs
    assert lib.sgnn_synthetic_graph_edges(169343, 1166243 / 169343) == 1166244


def test_load_graph(tmp_path):
    from paper_2308_12093_b200 import sgnn

    p = tmp_path / "g.el"
    p.write_text("# comment\n0 1\n1 2 0.5\n1 2 0.25\n")
    g = sgnn.load_graph(str(p))
    assert g["n"] == 3
    assert list(g["src"]) == [0, 1] and list(g["dst"]) == [1, 2]
    assert g["weight"][1] == 0.25  # duplicates keep the last weight
    mm = tmp_path / "g.mtx"
    mm.write_text("%%MatrixMarket matrix coordinate real symmetric\n3 3 2\n2 1 0.5\n3 3 2.0\n")
    g = sgnn.load_graph(str(mm), "matrix-market")
    assert g["n"] == 3 and list(g["src"]) == [0, 1, 2] and list(g["dst"]) == [1, 0, 2]
    with pytest.raises(RuntimeError):
        sgnn.load_graph(str(tmp_path / "missing.el"))
