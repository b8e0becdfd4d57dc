"""Fused evaluation (k_eval_fused, opt-in with PN_EVAL_FUSED=1): monomial
trees folded straight into per-variable binary-counter stacks, one CTA per
(polynomial, slot).  It must reproduce evaluate_system (evaldiff.py:215-266)
bit for bit, like the two-kernel path."""

import os
from contextlib import contextmanager

import numpy as np
import pytest

import oracle
from conftest import golden, golden_names, level_from_name, oracle_level, same

pytestmark = pytest.mark.gpu


@contextmanager
def fused_env(value):
    old = os.environ.get("PN_EVAL_FUSED")
    os.environ["PN_EVAL_FUSED"] = value
    try:
        yield
    finally:
        if old is None:
            del os.environ["PN_EVAL_FUSED"]
        else:
            os.environ["PN_EVAL_FUSED"] = old


def _packed(g):
    from paper_1402_2626_b200.polyrep import PackedSystem
    level = level_from_name(str(g["level"]))
    return PackedSystem(level, int(g["n_vars"]), g["poly_ptr"].astype(np.int32), g["mon_ptr"].astype(np.int32),
                        g["var_idx"].astype(np.int32), g["exps"].astype(np.int32), np.ascontiguousarray(g["coeffs"]))


def _point(level, n, seed):
    rng = np.random.default_rng(seed)
    x = rng.uniform(0.5, 2.0, level.cshape + (n,)) * rng.choice([-1.0, 1.0], level.cshape + (n,))
    x.reshape(-1, n)[[i for i in range(level.es) if i % level.ncomp != 0]] *= 1e-17
    return np.ascontiguousarray(x)


@pytest.mark.parametrize("name", golden_names("eval_"))
def test_fused_single_evaluation_golden(gpu, name):
    """With PN_EVAL_FUSED=1 at creation, eligible systems evaluate through the
    fused kernel; every golden still matches."""
    from paper_1402_2626_b200.evaldiff import PreparedSystem, evaluate_system
    g = golden(name)
    with fused_env("1"):
        ev = evaluate_system(PreparedSystem(_packed(g)), g["x"])
    assert same(ev.f, g["f"])
    assert same(ev.J, g["J"])


@pytest.mark.parametrize("lv,n,T,k,maxexp", [("cd", 128, 64, 32, 1), ("cdd", 96, 80, 32, 1), ("cqd", 64, 40, 32, 1),
                                             ("rdd", 60, 50, 5, 3), ("cdd", 50, 70, 12, 2), ("cqd", 40, 33, 3, 3),
                                             ("rqd", 48, 65, 20, 2)])
def test_fused_single_evaluation_vs_oracle(gpu, lv, n, T, k, maxexp):
    """Chunks of 32 monomials with ragged last chunks (T = 33, 50, 65, 70, 80),
    folded pairs (ell > 0) and power-table exponents."""
    from paper_1402_2626_b200.evaldiff import PreparedSystem, evaluate_system
    from paper_1402_2626_b200.generators import random_sparse_system
    level = level_from_name(lv)
    p = random_sparse_system(n, T, k, level, seed=n + T + k, maxexp=maxexp)
    x = _point(level, n, 5)
    with fused_env("1"):
        prep = PreparedSystem(p)
        assert prep.stats().segments > 0
        ev = evaluate_system(prep, x)
    f, J, counts = oracle.evaluate(oracle_level(lv), oracle.CSR.from_packed(p), x, nthreads=8)
    assert same(ev.f, f)
    assert same(ev.J, J)
    assert (ev.counter.eval_mults, ev.counter.grad_mults) == counts


@pytest.mark.parametrize("lv", ["cd", "cdd", "cqd"])
def test_fused_batch_values_match_single(gpu, lv):
    """pn_evaldiff_batch (fused, one slot per point) == one-point evaluations
    on the two-kernel path."""
    from paper_1402_2626_b200.batch import evaluate_batch
    from paper_1402_2626_b200.evaldiff import PreparedSystem, evaluate_system
    from paper_1402_2626_b200.generators import random_sparse_system
    level = level_from_name(lv)
    p = random_sparse_system(40, 45, 7, level, seed=77, maxexp=2)
    with fused_env("1"):
        prep = PreparedSystem(p)
        X = np.stack([_point(level, 40, 100 + b) for b in range(5)], axis=-2)
        F = evaluate_batch(prep, X)
    with fused_env("0"):
        for b in range(5):
            ev = evaluate_system(prep, np.ascontiguousarray(X[..., b, :]))
            assert same(F[..., b, :], ev.f), b
