"""sgnn-bench on the GPU: the reference's CLI smoke sequence
(tools/cli_smoke.cmake: gen -> bench --emit json with schema_version 1 ->
sweep a gat2 grid into a 5-line CSV), finite-difference gradcheck of both
models, and BenchReport parity with the reference's own run_benchmark
(oracle/_ref): n, q, every counter and cache_mem equal."""
import ctypes as C
import json
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_2308_12093_b200.bench_cli", *args],
                          cwd=ROOT, capture_output=True, text=True, timeout=600)


def test_cli_smoke_sequence(tmp_path):
    g = tmp_path / "g.el"
    assert _cli("gen", "--n", "300", "--avg-degree", "5", "--seed", "3",
                "--out", str(g)).returncode == 0
    r = _cli("bench", "--dataset", str(g), "--model", "gcn2", "--in-features", "8",
             "--hidden", "8", "--classes", "4", "--pass", "fwdbwd", "--warmups", "1",
             "--blocks", "2", "--runs", "1", "--emit", "json", "--out", str(tmp_path / "r.json"))
    assert r.returncode == 0, r.stderr
    text = (tmp_path / "r.json").read_text()
    assert '"schema_version": 1' in text
    rep = json.loads(text)["reports"][0]
    assert rep["median_s"] > 0 and len(rep["block_seconds"]) == 2 and "error" not in rep
    r = _cli("sweep", "--dataset", str(g), "--model", "gat2", "--in-features", "8",
             "--hidden", "8,16", "--heads", "8", "--classes", "4", "--caching", "none,full",
             "--warmups", "0", "--blocks", "1", "--runs", "1", "--out", str(tmp_path / "s.csv"))
    assert r.returncode == 0, r.stderr
    assert len((tmp_path / "s.csv").read_text().splitlines()) == 5  # header + 2 x 2


@pytest.mark.parametrize("model,extra", [("gcn2", []), ("gat2", []),
                                         ("gcn2", ["--caching", "features"]),
                                         ("gat2", ["--caching", "full"])])
def test_gradcheck_passes(model, extra):
    r = _cli("gradcheck", "--model", model, *extra)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout


CASES = [
    # model, format, scheme, caching, pass, feature-grad, precision
    ("gcn2", "csc", "adaptive", "features", "fwdbwd", "off", "f32"),
    ("gcn2", "ellpack", "transform-first", "none", "fwdbwd", "on", "f64"),
    ("gcn2", "hybrid", "propagate-first", "features", "fwd", "off", "f64"),
    ("gat2", "csr", "adaptive", "full", "fwdbwd", "off", "f32"),
    ("gat2", "coo", "adaptive", "node-attn", "fwdbwd", "on", "f64"),
    ("gat2", "csc", "adaptive", "features", "fwd", "off", "f32"),
]


@pytest.mark.parametrize("case", CASES)
def test_report_matches_the_reference_run_benchmark(case, tmp_path):
    import refpy

    model, fmt, scheme, caching, pss, fg, prec = case
    ds = "synth:n=1500,deg=6,seed=4"
    r = _cli("bench", "--dataset", ds, "--model", model, "--format", fmt, "--scheme", scheme,
             "--caching", caching, "--pass", pss, "--feature-grad", fg, "--precision", prec,
             "--in-features", "12", "--hidden", "8", "--heads", "4", "--classes", "5",
             "--warmups", "0", "--blocks", "2", "--runs", "1", "--emit", "json")
    assert r.returncode == 0, r.stderr
    ours = json.loads(r.stdout)["reports"][0]
    lib = refpy.lib()
    buf = C.create_string_buffer(1 << 16)
    lv = ["none", "features", "node-attn", "full"].index(caching)
    n = lib.ref_bench_report_json(ds.encode(), int(model == "gat2"),
                                  ["coo", "csr", "csc", "ellpack", "hybrid"].index(fmt), 8, 4,
                                  ["adaptive", "transform-first", "propagate-first"].index(scheme),
                                  lv, int(pss == "fwdbwd"), int(fg == "on"), int(prec == "f32"),
                                  12, 5, 0, buf, 1 << 16)
    assert n > 0, lib.ref_last_error()
    ref = json.loads(buf.value.decode())
    for key in ("schema_version", "dataset", "format", "model", "hidden", "heads", "scheme",
                "caching", "pass", "precision", "n", "q", "flops", "bytes", "gemm_flops",
                "spmm_flops", "sddmm_flops", "edge_flops", "elementwise_flops", "cache_mem"):
        assert ours[key] == ref[key], (key, ours[key], ref[key])
