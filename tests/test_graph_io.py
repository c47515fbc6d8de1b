"""Graph-file loaders vs the reference's own loaders (graph.hpp:62-147).

tests/golden/graph_io/expected.json holds what the reference returned for
every fixture file (oracle/gen_graph_io.py, through oracle/_ref): the
canonical edge list, or the runtime_error text for malformed input (header
lines skipped, a malformed weight read as 0, trailing tokens, ranges...)."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

DIR = os.path.join(GOLDEN, "graph_io")
with open(os.path.join(DIR, "expected.json")) as _fh:
    EXPECTED = json.load(_fh)


@pytest.mark.parametrize("name", sorted(EXPECTED))
def test_loader_matches_reference(name, monkeypatch):
    from paper_2308_12093_b200 import _graph_io

    monkeypatch.chdir(DIR)  # the reference's error text carries the path as given
    fmt = "matrix-market" if name.endswith(".mtx") else "edge-list"
    want = EXPECTED[name]
    if "error" in want:
        with pytest.raises(RuntimeError) as ei:
            _graph_io.load_graph(name, fmt)
        assert str(ei.value) == want["error"]
        return
    g = _graph_io.load_graph(name, fmt)
    assert g["n"] == want["n"]
    assert g["src"].dtype == np.int32 and g["dst"].dtype == np.int32
    assert g["src"].tolist() == want["src"] and g["dst"].tolist() == want["dst"]
    assert [float(x).hex() for x in g["weight"]] == want["weight"]


def test_missing_file():
    from paper_2308_12093_b200 import _graph_io

    with pytest.raises(RuntimeError, match="cannot open"):
        _graph_io.load_graph(os.path.join(DIR, "does-not-exist.el"))
