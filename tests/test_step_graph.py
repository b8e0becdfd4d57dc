"""Graph-replayed Newton step (pn_newton_step on small systems: the device
step is captured once into a CUDA graph and replayed).  The replay launches
the same kernels on the same buffers, so every run_newton trace must equal
the direct path's and the oracle's bit for bit (newton.py:82-132)."""

import os
from contextlib import contextmanager

import numpy as np
import pytest

import oracle
from conftest import level_from_name, same

pytestmark = pytest.mark.gpu


@contextmanager
def env(**kv):
    old = {k: os.environ.get(k) for k in kv}
    os.environ.update(kv)
    try:
        yield
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


@pytest.mark.parametrize("lv,n,T,k", [("cd", 32, 32, 8), ("cdd", 24, 20, 6), ("cqd", 16, 12, 4), ("rdd", 20, 16, 5)])
def test_graph_replay_matches_direct_and_oracle(gpu, lv, n, T, k):
    from paper_1402_2626_b200.generators import random_sparse_system
    from paper_1402_2626_b200.newton import NewtonConfig, run_newton
    from paper_1402_2626_b200.polyrep import PackedSystem
    level = level_from_name(lv)
    p = random_sparse_system(n, T, k, level, seed=n + T + k)
    rng = np.random.default_rng(n)
    x0 = np.ascontiguousarray(rng.uniform(0.5, 2.0, level.cshape + (n,)))
    traces = {}
    for g in ("1", "0"):
        with env(PN_GRAPH=g):
            tr = run_newton(p, x0, NewtonConfig(level=level, max_iters=4, tol=0.0))
        traces[g] = tr
    assert traces["1"].to_json_lines() == traces["0"].to_json_lines()
    assert same(level.to_planes(traces["1"].x), level.to_planes(traces["0"].x))
    L = oracle.Level(level.base, level.cplx)
    lines, _, _ = oracle.run_newton_trace(L, oracle.CSR.from_packed(p), x0, 4, tol=0.0, nthreads=4)
    assert traces["1"].to_json_lines() == lines
