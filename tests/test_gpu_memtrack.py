"""Device memory accounting (memtrack.hpp:19-94 MemTracker) on the device
engine: the reference's own pins restated on the GPU path --
  * transient peaks of every scheme equal gcn_forward_transients /
    gcn_backward_transients (test_gcn.cpp:170-194);
  * the cached scheme retains no more than the uncached one (:196-208);
  * cache-class live bytes of a GAT forward equal gat_cache_footprint at
    every level, 4- and 8-byte scalars (test_gat.cpp:165-190)."""
import pytest
import torch

pytestmark = pytest.mark.gpu

SCHEMES = [(0, 0, 0), (0, 1, 0), (1, 0, 0), (1, 1, 0), (2, 2, 1)]


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_transient_peaks_match_the_scheme_table(orc, dtype):
    from paper_2308_12093_b200 import device as d

    n, m, k = 3000, 24, 40
    _, s, t = orc.synthetic_graph(n, 6.0, 61)
    A = d.Adjacency.gcn_operator(n, torch.from_numpy(s), torch.from_numpy(t), dtype)
    X = d.random_uniform(n, m, 62, dtype=dtype)
    th, b = d.gcn_params(m, k, 63, dtype=dtype)
    G = d.random_uniform(n, k, 64, dtype=dtype)
    sb = torch.finfo(dtype).bits // 8
    for sc in SCHEMES:
        scheme = d.make_scheme(*sc)
        for fg in (False, True):
            torch.cuda.synchronize()
            live0 = d.memory_stats("transient")[0]
            d.reset_memory_peaks()
            out, cache = d.gcn_forward(A, X, th, b, scheme)
            fwd_peak = d.memory_stats("transient")[1] - live0
            assert fwd_peak == sb * orc.gcn_forward_transients(sc[0], n, m, k), (sc, fg)
            d.reset_memory_peaks()
            d.gcn_backward(A, G, th, cache, fg)
            bwd_peak = d.memory_stats("transient")[1] - live0
            assert bwd_peak == sb * orc.gcn_backward_transients(sc[1], n, m, k, fg), (sc, fg)
            assert d.memory_stats("transient")[0] == live0  # transients released
            del cache


def test_cached_scheme_retains_no_more_than_uncached(orc):
    from paper_2308_12093_b200 import device as d

    n, m = 2000, 6
    _, s, t = orc.synthetic_graph(n, 5.0, 71)
    A = d.Adjacency.gcn_operator(n, torch.from_numpy(s), torch.from_numpy(t), torch.float64)
    X = d.random_uniform(n, m, 72, dtype=torch.float64)
    for k in (4, 6, 12):
        th, b = d.gcn_params(m, k, 73, dtype=torch.float64)
        c0 = d.memory_stats("cache")[0]
        _, cached = d.gcn_forward(A, X, th, b, d.make_scheme(2, 2, 1))
        assert d.memory_stats("cache")[0] - c0 == n * m * 8  # P reclassified into the cache
        _, uncached = d.gcn_forward(A, X, th, b, d.make_scheme(1, 1, 0))
        assert cached.retained_bytes() <= uncached.retained_bytes()
        del cached, uncached
        assert d.memory_stats("cache")[0] == c0


@pytest.mark.parametrize("dtype,sb", [(torch.float32, 4), (torch.float64, 8)])
def test_gat_cache_class_bytes_equal_the_footprint(orc, dtype, sb):
    from paper_2308_12093_b200 import device as d

    n, m, h, k = 1100, 4, 3, 5
    _, s, t = orc.synthetic_graph(n, 4.0, 101)
    P = d.Pattern.gat_pattern(n, torch.from_numpy(s), torch.from_numpy(t))
    q = P.nnz
    X = d.random_uniform(n, m, 102, dtype=dtype)
    th, a_s, a_d, b = d.gat_params(m, h, k, 103, dtype=dtype)
    for level, lv in (("none", 0), ("features", 1), ("node-attn", 2), ("full", 3)):
        c0 = d.memory_stats("cache")[0]
        out, cache = d.gat_forward(P, X, th, a_s, a_d, b, h, 0.2, level)
        want = orc.gat_cache_footprint(level, n, h, k, q, sb)
        assert cache.extra_bytes() == want
        assert d.memory_stats("cache")[0] - c0 == want, level
        del cache
        assert d.memory_stats("cache")[0] == c0
