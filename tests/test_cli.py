"""The command-line front end (mirror of polynewt.cli with --backend cuda):
output against the reference's own serialized systems and trace
(tests/golden/cli.json, make_cli_golden.py), exit codes, CSV report."""

import json
import os
import subprocess
import sys

import pytest

from conftest import GOLDEN, ROOT


def _cli(*args, **kw):
    return subprocess.run([sys.executable, "-m", "paper_1402_2626_b200", *args], capture_output=True, text=True,
                          cwd=ROOT, timeout=600, **kw)


def _golden():
    with open(os.path.join(GOLDEN, "cli.json")) as f:
        return json.load(f)


def test_gen_cyclic_matches_reference():
    """cyclic needs no arithmetic (all coefficients are +-1): host only."""
    g = _golden()["gen"]
    for name in ("cdd", "rqd", "cd", "cqd"):
        base, cplx = name[1:], name[0] == "c"
        r = _cli("gen", "--benchmark", "cyclic", "--n", "5", "--prec", base, "--complex" if cplx else "--real")
        assert r.returncode == 0, r.stderr
        assert r.stdout == g[f"cyclic 5 {name}"]


def test_usage_and_parse_errors_exit_2(tmp_path):
    bad = tmp_path / "bad.txt"
    bad.write_text("1 2\n3*x0 + ;\n")
    r = _cli("newton", "--file", str(bad))
    assert r.returncode == 2 and "line 2, column" in r.stderr
    r = _cli("qr", "--m", "3", "--n", "5")
    assert r.returncode == 2 and "need m >= n >= 1" in r.stderr
    r = _cli("newton", "--benchmark", "cyclic", "--n", "4", "--real", "--homotopy")
    assert r.returncode == 2 and "need --complex" in r.stderr


def test_report_writes_reference_csv(tmp_path):
    trace = tmp_path / "t.jsonl"
    trace.write_text(_golden()["newton_chandrasekhar_12_cdd"] + json.dumps({"summary": {}}) + "\n")
    r = _cli("report", "--trace", str(trace), "--out-dir", str(tmp_path / "out"))
    assert r.returncode == 0, r.stderr
    rows = (tmp_path / "out" / "trace.csv").read_text().splitlines()
    assert rows[0] == "iter,f_norm,dx_norm,b0,dx0,x0" and len(rows) == 7
    first = json.loads(_golden()["newton_chandrasekhar_12_cdd"].splitlines()[0])
    assert rows[1].startswith(f"1,{first['f_norm']},{first['dx_norm']},\"({first['b0'][0]},{first['b0'][1]})\"")


@pytest.mark.gpu
def test_gen_chandrasekhar_matches_reference(gpu):
    """H-equation coefficients are formed in working precision on the GPU."""
    g = _golden()["gen"]
    for name in ("cdd", "rqd", "cd", "cqd"):
        base, cplx = name[1:], name[0] == "c"
        r = _cli("gen", "--benchmark", "chandrasekhar", "--n", "6", "--prec", base, "--complex" if cplx else "--real")
        assert r.returncode == 0, r.stderr
        assert r.stdout == g[f"chandrasekhar 6 {name}"]


@pytest.mark.gpu
def test_newton_trace_matches_reference(gpu, tmp_path):
    g = _golden()
    out = tmp_path / "trace.jsonl"
    r = _cli("newton", "--benchmark", "chandrasekhar", "--n", "12", "--iters", "6", "--tol", "0",
             "--output", str(out), "--report-dir", str(tmp_path / "rep"), "--dump-qr", str(tmp_path / "qr.txt"))
    assert r.returncode == 0, r.stderr
    lines = out.read_text().splitlines(keepends=True)
    assert "".join(lines[:-1]) == g["newton_chandrasekhar_12_cdd"]
    summary = json.loads(lines[-1])["summary"]
    for k, v in g["newton_summary"].items():
        assert summary[k] == v, k
    assert summary["backend"] == "cuda"
    assert (tmp_path / "rep" / "trace.csv").exists()
    assert (tmp_path / "qr.txt").read_text().startswith("Q 12 12\n")


@pytest.mark.gpu
def test_qr_check_and_evaldiff(gpu):
    r = _cli("qr", "--m", "40", "--n", "17", "--prec", "qd", "--check")
    assert r.returncode == 0, r.stderr
    d = json.loads(r.stdout)
    assert d["m"] == 40 and d["qr_residual"] < 1e-60 and d["backend"] == "cuda"
    r = _cli("evaldiff", "--m", "4", "--n", "64", "--prec", "dd")
    assert r.returncode == 0, r.stderr
    d = json.loads(r.stdout)
    # the product tree's analytic counts (test_acceptance.py:46-61): n-1 and 2n-4 per product
    assert d["tree"]["eval_mults"] == 4 * 63 and d["tree"]["grad_mults"] == 4 * 124
    assert d["sequential"]["eval_mults"] == 4 * 63 and d["sequential"]["grad_mults"] == 4 * 124


@pytest.mark.gpu
def test_newton_from_text_file_matches_benchmark(gpu, tmp_path):
    """gen -> file -> newton --file (native text ingestion): the rendered
    32-digit coefficients parse back to (nearly) the same system, so the run
    converges like the benchmark's (quadratically, to the dd floor)."""
    g = _golden()
    path = tmp_path / "chandra12.txt"
    r = _cli("gen", "--benchmark", "chandrasekhar", "--n", "12", "--output", str(path))
    assert r.returncode == 0, r.stderr
    out = tmp_path / "t.jsonl"
    r = _cli("newton", "--file", str(path), "--iters", "6", "--tol", "0", "--output", str(out))
    assert r.returncode == 0, r.stderr
    lines = out.read_text().splitlines()
    summary = json.loads(lines[-1])["summary"]
    assert summary["iterations"] == 6 and summary["final_f_norm"] < 1e-28
    assert json.loads(lines[0])["f_norm"] == json.loads(g["newton_chandrasekhar_12_cdd"].splitlines()[0])["f_norm"]
