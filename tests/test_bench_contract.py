"""bench.py's reference arm (`--impl reference`) runs the oracle port on the
host only, so its JSON line can be checked here without a GPU: the keys the
driver reads, the reference-arm extras, whole measured steps, the identical
config dict as our arm, and that the arm never maps the product library
(bench.py contract)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

ARGV = ["--impl", "reference", "--dim", "48", "--terms", "24", "--k", "6", "--base", "dd", "--steps", "2",
        "--warmup", "1", "--cpu-budget", "1"]

PROBE = """
import runpy, sys, json
sys.argv = ["bench.py"] + json.loads(sys.argv[1])
runpy.run_path("bench.py", run_name="__main__")
maps = open("/proc/self/maps").read()
print("PRODUCT_LIB_MAPPED=" + str("libpolynewt_b200" in maps))
print("ORACLE_LIB_MAPPED=" + str("libpn_oracle" in maps))
"""


def _run_reference():
    out = subprocess.run([sys.executable, "-c", PROBE, json.dumps(ARGV)], capture_output=True, text=True,
                         timeout=600, cwd=ROOT, env={**os.environ, "RANK": "0", "WORLD_SIZE": "1",
                                                     "LOCAL_RANK": "0"})
    assert out.returncode == 0, out.stderr[-2000:]
    lines = out.stdout.strip().splitlines()
    d = json.loads([ln for ln in lines if ln.startswith("{")][-1])
    return d, lines


def test_reference_arm_json_line():
    d, lines = _run_reference()
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference"
    assert d["unit"] == "steps/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["single_core"]["cores"] == 1
    # whole steps, measured: the reported mean is the mean of the timed steps
    assert d["steps"] == 2 and len(d["step_seconds"]) == 2
    assert abs(d["ms_per_step"] - 1e3 * sum(d["step_seconds"]) / 2) < 1e-6
    assert "extrapolated" not in d["cpu_baseline"]["sample"]
    # no product library in the reference arm; the oracle is what runs
    assert "PRODUCT_LIB_MAPPED=False" in lines
    assert "ORACLE_LIB_MAPPED=True" in lines


def test_reference_arm_config_equals_ours():
    sys.path.insert(0, ROOT)
    import bench
    d, _ = _run_reference()
    ours = bench.step_config(bench.parse(ARGV[2:]), 1)
    assert d["config"] == ours
    assert d["config"]["workload"].startswith("F(48,24,6) complex dd Newton step 48x48")


def test_oracle_generator_matches_product_generator():
    """The reference arm's inputs (oracle generator) equal our arm's (the
    product's C generator), array for array."""
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import oracle
    from paper_1402_2626_b200.generators import random_sparse_system
    from paper_1402_2626_b200.xprec import precision_level
    for base, kmin, maxexp in (("qd", None, 1), ("dd", 1, 3)):
        p = random_sparse_system(40, 17, 6, precision_level(base, True), seed=5, maxexp=maxexp, m=45, kmin=kmin)
        c = oracle.random_sparse_csr(40, 17, 6, oracle.Level(base, True), seed=5, maxexp=maxexp, m=45, kmin=kmin)
        for a, b in ((p.poly_ptr, c.poly_ptr), (p.mon_ptr, c.mon_ptr), (p.var_idx, c.var_idx), (p.exps, c.exps),
                     (p.coeffs, c.coeffs)):
            assert np.array_equal(np.asarray(a), np.asarray(b))


REDUCE_PROBE = """
import os, sys, json
import torch.distributed as dist
sys.path.insert(0, os.getcwd())
import bench
dist.init_process_group("gloo")
r = dist.get_rank()
mx = bench.reduce_ranks([1.0 + r, 10.0 - r], "max")
sm = bench.reduce_ranks([1.0 + r], "sum")
print(json.dumps({"rank": r, "max": mx, "sum": sm}))
dist.destroy_process_group()
"""


def test_max_over_ranks_gloo_world2(tmp_path):
    """The timing reductions of an N-rank bench run (max of the elapsed times,
    sum of the work) over two gloo ranks (PN_BENCH_SHARED_GPU: host tensors)."""
    probe = tmp_path / "probe.py"
    probe.write_text(REDUCE_PROBE)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(probe)]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT,
                         env={**os.environ, "PN_BENCH_SHARED_GPU": "1", "OMP_NUM_THREADS": "1"})
    assert out.returncode == 0, out.stderr[-2000:]
    recs = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert sorted(r["rank"] for r in recs) == [0, 1]
    for r in recs:
        assert r["max"] == [2.0, 10.0] and r["sum"] == [3.0]


def _port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]
