"""Golden cases for the graph-file loaders -- TEST INFRASTRUCTURE ONLY.

Writes small edge-list / MatrixMarket fixtures (well-formed, header lines,
comments, malformed tokens, trailing tokens, duplicate edges, ...) under
tests/golden/graph_io/ and records what the reference's own loaders
(graph.hpp:62-147, through oracle/_ref's ref_load_graph) return for each:
the canonical edge list or the runtime_error text.  Run in the dev container
(needs oracle/_ref):  python oracle/gen_graph_io.py
"""
import ctypes as C
import json
import os

import numpy as np

import refpy

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "..", "tests", "golden", "graph_io")

CASES = {
    # edge lists
    "plain.el": "0 1\n1 2 2.5\n2 0\n",
    "header.el": "source target\n0 1\n1 2\n",
    "comments.el": "# a comment\n\n0 1 # trailing comment\n   \n1 0 3\n",
    "dups.el": "0 1 1.0\n0 1 2.0\n1 0\n0 1 3.0\n",
    "missing_dst.el": "0 1\n2\n",
    "bad_dst.el": "0 1\n2 x\n",
    "trailing.el": "0 1 1.0 extra\n",
    "bad_weight.el": "0 1 abc\n1 2\n",
    "weight_suffix.el": "0 1 2.5x\n",
    "negative.el": "0 -1\n",
    "float_src.el": "1.5 2\n",
    "int_prefix.el": "12abc 3\n",
    "plus_sign.el": "+1 +2 +3.5\n",
    "empty.el": "",
    "sci_weight.el": "0 1 1e-3\n1 0 -2E2\n",
    # MatrixMarket
    "general.mtx": "%%MatrixMarket matrix coordinate real general\n% c\n3 3 3\n1 2 0.5\n2 3 1\n3 1 2\n",
    "symmetric.mtx": "%%MatrixMarket matrix coordinate real symmetric\n3 3 2\n2 1 4\n3 3 1\n",
    "pattern.mtx": "%%MatrixMarket matrix coordinate pattern general\n2 2 2\n1 2\n2 1\n",
    "integer.mtx": "%%MatrixMarket matrix coordinate integer general\n2 2 1\n1 2 7\n",
    "bad_header.mtx": "%%MatrixMarket matrix array real general\n2 2\n",
    "bad_field.mtx": "%%MatrixMarket matrix coordinate complex general\n2 2 1\n1 2 1 0\n",
    "not_square.mtx": "%%MatrixMarket matrix coordinate real general\n2 3 1\n1 2 1\n",
    "bad_size.mtx": "%%MatrixMarket matrix coordinate real general\n2 x 1\n",
    "no_size.mtx": "%%MatrixMarket matrix coordinate real general\n% only comments\n",
    "missing_value.mtx": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2\n",
    "out_of_range.mtx": "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n",
    "short.mtx": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 2 1\n",
    "bad_entry.mtx": "%%MatrixMarket matrix coordinate real general\n2 2 1\nx 2 1\n",
    "blank_entry.mtx": "%%MatrixMarket matrix coordinate real general\n2 2 1\n   \n1 2 1\n",
    "extra_tokens.mtx": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 1 9 9\n",
    "empty.mtx": "",
    "dups.mtx": "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 2 1\n1 2 5\n2 1 2\n",
}


def main():
    os.makedirs(OUT, exist_ok=True)
    lib = refpy.lib()
    expected = {}
    for name, text in sorted(CASES.items()):
        path = os.path.join(OUT, name)
        with open(path, "w") as fh:
            fh.write(text)
        mm = int(name.endswith(".mtx"))
        n = C.c_int(0)
        # relative path in the error text: run from the golden directory
        cwd = os.getcwd()
        os.chdir(OUT)
        try:
            cnt = lib.ref_load_graph(name.encode(), mm, C.byref(n), None, None, None)
            if cnt < 0:
                expected[name] = {"error": lib.ref_last_error().decode()}
                continue
            src = np.zeros(cnt, np.int32)
            dst = np.zeros(cnt, np.int32)
            w = np.zeros(cnt, np.float64)
            lib.ref_load_graph(name.encode(), mm, C.byref(n), src.ctypes.data, dst.ctypes.data,
                               w.ctypes.data)
        finally:
            os.chdir(cwd)
        expected[name] = {"n": n.value, "src": src.tolist(), "dst": dst.tolist(),
                          "weight": [float(x).hex() for x in w]}
    with open(os.path.join(OUT, "expected.json"), "w") as fh:
        json.dump(expected, fh, indent=1, sort_keys=True)
    print(json.dumps(expected, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
