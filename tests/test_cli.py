"""sgnn-bench CLI (tools/sgnn_bench.cpp) host-side subcommands: cost (the
reference's cost CSV for its recorded dataset statistics), gen (the reference's
save_edge_list format of its seeded generator) and argument validation."""
import subprocess
import sys

from conftest import ROOT


def _cli(*args, env=None):
    return subprocess.run([sys.executable, "-m", "paper_2308_12093_b200.bench_cli", *args],
                          cwd=ROOT, capture_output=True, text=True, timeout=300, env=env)


def test_cost_csv_matches_the_cost_model(orc):
    r = _cli("cost", "--dataset-stats", "cora", "--f", "64")
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    assert lines[0] == "op,format,n,q,p,f,flops,bytes,oi"
    assert len(lines) == 9  # csr, csc, coo, ellpack x spmm, sddmm
    for ln in lines[1:]:
        op, fmt, n, q, p, f, flops, by, oi = ln.split(",")
        fn = orc.spmm_cost if op == "spmm" else orc.sddmm_cost
        c = fn(fmt, int(n), int(q), int(p), int(f))
        assert (int(flops), int(by)) == (c["flops"], c["bytes"]), ln
        assert oi == "%.6f" % c["operational_intensity"]
    # test_smoke.py:35-37 reference values
    assert lines[1].startswith("spmm,csr,2708,10556,0,64,") and lines[1].endswith(",0.621219")


def test_gen_writes_the_reference_edge_list(tmp_path, orc):
    out = tmp_path / "g.el"
    r = _cli("gen", "--n", "300", "--avg-degree", "5", "--seed", "3", "--out", str(out))
    assert r.returncode == 0, r.stderr
    _, s, t = orc.synthetic_graph(300, 5.0, 3)
    want = [f"# nodes 300 edges {len(s)}"] + [f"{a} {b}" for a, b in zip(s, t)]
    assert out.read_text().splitlines() == want


def test_usage_errors():
    r = _cli("bench", "--dataset", "synth:n=10,deg=2", "--format", "dense")
    assert r.returncode == 2 and "unknown format 'dense'" in r.stderr
    r = _cli("sweep", "--dataset", "synth:n=10,deg=2", "--model", "gcn2", "--caching", "full")
    assert r.returncode == 2 and "gcn2 supports none or features" in r.stderr
    r = _cli("cost", "--dataset-stats", "nope")
    assert r.returncode == 2
