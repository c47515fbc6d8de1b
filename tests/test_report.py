"""BenchReport (bench.hpp:52-71, 292-437): the analytic counter restatement
of paper_2308_12093_b200/report.py against the reference's own
run_benchmark reports over 400 configurations (tests/golden/bench_reports.json,
oracle/gen_bench_reports.py), and the report emission formats."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

with open(os.path.join(GOLDEN, "bench_reports.json")) as _fh:
    GOLD = json.load(_fh)
FORMATS = ("coo", "csr", "csc", "ellpack", "hybrid")
LEVELS = ("none", "features", "node-attn", "full")


@pytest.fixture(scope="module")
def shapes(orc):
    from paper_2308_12093_b200 import report as R

    spec = dict(kv.split("=") for kv in GOLD["dataset"][len("synth:"):].split(","))
    n = int(spec["n"])
    _, s, t = orc.synthetic_graph(n, float(spec["deg"]), int(spec["seed"]))
    op = orc.gcn_operator(n, s, t)  # gcn_normalize(A): the Gcn2 operator
    pat = orc.gat_pattern(n, s, t)  # add_self_loops(A): the Gat2 pattern
    rc = np.bincount(op.rows, minlength=n)
    cc = np.bincount(op.cols, minlength=n)
    return n, {f: R.OperatorShape(f, n, rc, cc) for f in FORMATS}, int(pat.rowptr[-1])


def _case_ids():
    return [f"{c['config']['gat2']}-{i}" for i, c in enumerate(GOLD["cells"])]


@pytest.mark.parametrize("idx", range(len(GOLD["cells"])), ids=_case_ids())
def test_counters_equal_the_reference_report(idx, shapes, orc):
    from paper_2308_12093_b200 import report as R

    cell = GOLD["cells"][idx]
    cfg, want = cell["config"], cell["report"]
    n, ops, q_gat = shapes
    op = ops[FORMATS[cfg["fmt"]]]
    sb = 4 if cfg["f32"] else 8
    if cfg["gat2"]:
        assert want["q"] == q_gat
        c = R.step_counters("gat2", op, n, cfg["in_features"], cfg["hidden"], cfg["classes"],
                            heads=cfg["heads"], gat_level=LEVELS[cfg["level"]],
                            fwdbwd=bool(cfg["fwdbwd"]), input_grad=bool(cfg["fg"]),
                            scalar_bytes=sb)
    else:
        assert want["q"] == op.q
        pol, cach, fg = cfg["policy"], bool(cfg["level"]), bool(cfg["fg"])
        s1 = orc.resolve_scheme(pol, cfg["in_features"], cfg["hidden"], fg, cach)
        s2 = orc.resolve_scheme(pol, cfg["hidden"], cfg["classes"], True, cach)
        c = R.step_counters("gcn2", op, n, cfg["in_features"], cfg["hidden"], cfg["classes"],
                            scheme=((s1[0], s1[1]), (s2[0], s2[1])),
                            fwdbwd=bool(cfg["fwdbwd"]), input_grad=fg, scalar_bytes=sb)
    rep = R.fill_counters(R.new_report(), c)
    for key in ("flops", "bytes", "gemm_flops", "spmm_flops", "sddmm_flops", "edge_flops",
                "elementwise_flops"):
        assert rep[key] == want[key], (key, cfg)


def test_report_emission_round_trip(tmp_path):
    from paper_2308_12093_b200 import report as R

    r = R.new_report(dataset="g.el", format="csr", model="gcn2", hidden=8,
                     scheme="adaptive", caching="features", precision="f32",
                     block_seconds=[1e-3, 2e-3, 3e-3])
    r["pass"] = "fwdbwd"
    r["median_s"], r["std_s"] = R.timing_stats(r["block_seconds"])
    assert r["median_s"] == 2e-3 and abs(r["std_s"] - (2 / 3) ** 0.5 * 1e-3) < 1e-15
    bad = dict(r, error="boom, \"quoted\"", dataset="a,b")
    R.emit([r, bad], "json", str(tmp_path / "r.json"))
    j = json.loads((tmp_path / "r.json").read_text())
    assert j["schema_version"] == 1 and len(j["reports"]) == 2
    assert R.report_from_json(j["reports"][0]) == R.report_from_json(R.report_to_json(r))
    assert j["reports"][1]["error"] == "boom, \"quoted\""
    csv = R.reports_to_csv([r, bad]).splitlines()
    assert csv[0] == R.csv_header() and len(csv) == 3
    assert csv[1].split(",")[8] == "2.000000000e-03"
    assert csv[2].startswith('"a,b",csr') and csv[2].endswith(",,,,,,")
