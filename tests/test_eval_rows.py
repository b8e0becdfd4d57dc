"""The row evaluation (k_eval_rows: one CTA per polynomial at a time,
contributions of a chunk in shared memory, per-variable binary-counter
stacks) against the oracle and against the two-kernel path (K1 + K2), bit
for bit, on every precision level, tree base, exponent pattern and
polynomial shape the plan accepts (evaldiff.py:142-266)."""

import os

import numpy as np
import pytest

import oracle
from conftest import LEVEL_NAMES, level_from_name, oracle_level, same

pytestmark = pytest.mark.gpu


def _point(level, n, seed):
    rng = np.random.default_rng(seed)
    x = rng.uniform(0.5, 2.0, level.cshape + (n,)) * rng.choice([-1.0, 1.0], level.cshape + (n,))
    x.reshape(-1, n)[[i for i in range(level.es) if i % level.ncomp != 0]] *= 1e-17
    return np.ascontiguousarray(x)


def _eval(monkeypatch, p, x, rows):
    """Evaluate with the row path forced on (rows=True) or off."""
    from paper_1402_2626_b200.evaldiff import PreparedSystem, evaluate_system
    monkeypatch.setenv("PN_EVAL_ROWS", "1")
    prep = PreparedSystem(p)
    monkeypatch.setenv("PN_EVAL_ROWS", "1" if rows else "0")
    ev = evaluate_system(prep, x)
    monkeypatch.delenv("PN_EVAL_ROWS", raising=False)
    return ev, prep


@pytest.mark.parametrize("lv", LEVEL_NAMES)
@pytest.mark.parametrize("maxexp", [1, 3])
def test_rows_vs_oracle_and_two_kernel_path(gpu, monkeypatch, lv, maxexp):
    from paper_1402_2626_b200.generators import random_sparse_system
    level = level_from_name(lv)
    p = random_sparse_system(70, 45, 6, level, seed=11 + maxexp, maxexp=maxexp)
    x = _point(level, 70, 3)
    ev, prep = _eval(monkeypatch, p, x, rows=True)
    assert prep.rows_plan()["ok"]
    ref, _ = _eval(monkeypatch, p, x, rows=False)
    f, J, counts = oracle.evaluate(oracle_level(lv), oracle.CSR.from_packed(p), x)
    assert same(ev.f, f) and same(ev.J, J)
    assert same(ref.f, ev.f) and same(ref.J, ev.J)
    assert (ev.counter.eval_mults, ev.counter.grad_mults) == counts


@pytest.mark.parametrize("lv", ["cd", "cdd", "cqd", "rd"])
def test_rows_many_chunks_and_long_runs(gpu, monkeypatch, lv):
    """T = 700 monomials per polynomial (several chunks, a ragged last one)
    over 9 variables of k = 5: long Jacobian-entry runs (deep stacks) that
    cross chunk boundaries, and a value stack over chunks."""
    from paper_1402_2626_b200.generators import random_sparse_system
    level = level_from_name(lv)
    p = random_sparse_system(9, 700, 5, level, seed=4, m=6, maxexp=2)
    x = _point(level, 9, 4)
    x.reshape(level.es, 9)[0] = np.abs(x.reshape(level.es, 9)[0]) * 0.5 + 0.75  # keep the products bounded
    ev, prep = _eval(monkeypatch, p, x, rows=True)
    plan = prep.rows_plan()
    assert plan["ok"] and plan["nchunks"] > 6 and plan["depth"] >= 9
    f, J, _ = oracle.evaluate(oracle_level(lv), oracle.CSR.from_packed(p), x)
    assert same(ev.f, f) and same(ev.J, J)


@pytest.mark.parametrize("K", [2, 3, 5, 8, 16, 17, 31, 32])
def test_rows_every_tree_base(gpu, monkeypatch, K):
    from paper_1402_2626_b200.generators import random_sparse_system
    level = level_from_name("cdd")
    p = random_sparse_system(40, 21, K, level, seed=K)
    x = _point(level, 40, K)
    ev, prep = _eval(monkeypatch, p, x, rows=True)
    assert prep.rows_plan()["ok"] and prep.rows_plan()["K"] == K
    f, J, _ = oracle.evaluate(oracle_level("cdd"), oracle.CSR.from_packed(p), x)
    assert same(ev.f, f) and same(ev.J, J)


@pytest.mark.parametrize("lv", ["cd", "cqd", "rdd"])
def test_rows_ragged_polynomials_constants_and_empty(gpu, monkeypatch, lv):
    """Polynomials of 0, 1, 2, 33 and 70 terms, constants (k = 0, sorted
    first; duplicates kept), duplicate supports, an empty polynomial (f = 0
    and an all-zero Jacobian row, evaldiff.py:261-262)."""
    from paper_1402_2626_b200.polyrep import PackedSystem
    level = level_from_name(lv)
    rng = np.random.default_rng(5)
    n, K = 24, 4
    sizes = [0, 1, 2, 33, 70, 5]
    supports = []
    for T in sizes:
        poly = []
        for t in range(T):
            if t % 11 == 3:
                poly.append([])  # constant term
            else:
                poly.append(sorted(rng.choice(n, K, replace=False).tolist()))
        if T >= 5:
            poly.append(list(poly[1]))  # duplicate support
        supports.append(poly)
    pp = np.array([0] + list(np.cumsum([len(s) for s in supports])), np.int32)
    mons = [mm for s in supports for mm in s]
    mp = np.array([0] + list(np.cumsum([len(mm) for mm in mons])), np.int32)
    var = np.concatenate([np.asarray(mm, np.int32) for mm in mons if mm])
    exps = rng.integers(1, 3, len(var)).astype(np.int32)
    M = len(mons)
    coeffs = rng.uniform(-2, 2, level.cshape + (M,))
    p = PackedSystem(level, n, pp, mp, var, exps, np.ascontiguousarray(coeffs))
    x = _point(level, n, 8)
    ev, prep = _eval(monkeypatch, p, x, rows=True)
    assert prep.rows_plan()["ok"]
    f, J, _ = oracle.evaluate(oracle_level(lv), oracle.CSR.from_packed(p), x)
    assert same(ev.f, f) and same(ev.J, J)
    assert np.all(ev.f[..., 0] == 0.0) and np.all(ev.J[..., 0, :] == 0.0)


def test_rows_plan_declines_mixed_k(gpu):
    """Mixed k (the C2 "mixed" variant) keeps the two-kernel path."""
    from paper_1402_2626_b200.evaldiff import PreparedSystem
    from paper_1402_2626_b200.generators import random_sparse_system
    p = random_sparse_system(30, 10, 8, level_from_name("cd"), seed=1, kmin=2)
    assert not PreparedSystem(p).rows_plan()["ok"]


@pytest.mark.parametrize("lv", ["cd", "cdd", "cqd"])
def test_rows_batched_homotopy_constants(gpu, monkeypatch, lv):
    """The batched path (per-start constants replacing each polynomial's
    constant term) through the row-cluster kernel equals single runs."""
    from paper_1402_2626_b200.batch import homotopy_batch, run_newton_batch
    from paper_1402_2626_b200.evaldiff import PreparedSystem
    from paper_1402_2626_b200.generators import random_sparse_system, random_unit_point
    from paper_1402_2626_b200.newton import NewtonConfig, homotopy_start_system, run_newton
    level = level_from_name(lv)
    p = random_sparse_system(16, 8, 4, level, seed=31, maxexp=2)
    B = 4
    Z = np.stack([level.to_planes(random_unit_point(16, 200 + b, level)) for b in range(B)], axis=-2)
    t = level.from_float(0.99)
    system, consts = homotopy_batch(p, Z, t)
    monkeypatch.setenv("PN_EVAL_ROWS", "1")
    prep = PreparedSystem(system)
    assert prep.rows_plan()["ok"]
    res = run_newton_batch(prep, Z, consts, max_iters=6)
    monkeypatch.setenv("PN_EVAL_ROWS", "0")
    for b in range(B):
        zb = np.ascontiguousarray(Z[..., b, :])
        tr = run_newton(homotopy_start_system(p, zb, t), zb, NewtonConfig(level=level, max_iters=6))
        assert same(res.x[..., b, :], level.to_planes(tr.x)), b
        assert res.iters[b] == len(tr.entries)


@pytest.mark.parametrize("lv", ["cd", "cdd", "cqd"])
def test_rows_full_size_c2_vs_oracle(gpu, monkeypatch, lv):
    """C2 at full size through the row-cluster kernel: 8 sampled rows of f
    and J against the oracle."""
    from paper_1402_2626_b200.generators import random_sparse_system
    level = level_from_name(lv)
    p = random_sparse_system(1024, 1024, 32, level, seed=2024)
    x = _point(level, 1024, 11)
    ev, prep = _eval(monkeypatch, p, x, rows=True)
    rows = [0, 1, 255, 511, 512, 777, 1000, 1023]
    f, J, _ = oracle.evaluate(oracle_level(lv), oracle.CSR.from_packed(p).rows(rows), x,
                              nthreads=os.cpu_count() or 1)
    assert same(ev.f[..., rows], f)
    assert same(ev.J[..., rows, :], J)
