"""Pin the C oracle (oracle/pn_oracle.c) to the reference: golden vectors
produced by running polynewt itself (tests/golden/make_golden.py) and the
reference's own known-answer tests (pkg/tests/test_evaldiff.py,
test_mgs.py, test_newton.py).  CPU only."""

import random
from functools import reduce

import numpy as np
import pytest

import oracle
from conftest import LEVEL_NAMES, golden, golden_names, oracle_level, same


def csr_of(g, prefix=""):
    return oracle.CSR(int(g["n_vars"]), g[prefix + "poly_ptr"], g[prefix + "mon_ptr"], g[prefix + "var_idx"],
                      g[prefix + "exps"], g[prefix + "coeffs"])


# -- L0/L1 arithmetic (test_varith.py:24-70) ---------------------------------------

@pytest.mark.parametrize("lv", LEVEL_NAMES)
def test_vec_ops_match_reference(lv):
    g = golden(f"vec_{lv}")
    L = oracle_level(lv)
    for op in ("add", "sub", "mul", "div"):
        assert same(oracle.vec_op(L, op, g["a"], g["b"]), g[op]), op
    assert same(oracle.vec_op(L, "abs2", g["a"]), g["abs2"])
    assert same(oracle.vec_op(L, "sqrt", g["abs2"]), g["sqrt"])


@pytest.mark.parametrize("lv", LEVEL_NAMES)
def test_tree_sum_matches_reference(lv):
    g = golden(f"vec_{lv}")
    L = oracle_level(lv)
    for n in (1, 2, 3, 5, 7, 8, 33, 100, 257):
        assert same(oracle.tree_sum(L, g[f"tree_in_{n}"]), g[f"tree_out_{n}"]), n


# -- L3 (1)+(2) evaluation ---------------------------------------------------------

@pytest.mark.parametrize("name", golden_names("eval_"))
def test_evaluate_matches_reference(name):
    g = golden(name)
    L = oracle_level(str(g["level"]))
    f, J, counts = oracle.evaluate(L, csr_of(g), g["x"])
    assert same(f, g["f"])
    assert same(J, g["J"])
    assert counts == tuple(int(c) for c in g["counts"])


def _single_monomial(n_vars, exps, coeff=1.0):
    L = oracle.Level("dd", False)
    return L, oracle.CSR.from_polys(n_vars, [[((coeff, 0.0), tuple(exps))]], L)


@pytest.mark.parametrize("n", range(2, 13))
def test_tree_exact_small_integers(n):
    # test_evaldiff.py:50-83: small-integer inputs make every product exact
    rng = random.Random(n)
    for _ in range(5):
        ints = [rng.randint(1, 9) for _ in range(n)]
        L, c = _single_monomial(n, [(v, 1) for v in range(n)])
        x = np.zeros((2, n))
        x[0] = ints
        f, J, _ = oracle.evaluate(L, c, x)
        assert f[0, 0] == reduce(lambda a, b: a * b, ints)
        for i in range(n):
            want = reduce(lambda a, b: a * b, (v for j, v in enumerate(ints) if j != i), 1)
            assert J[0, 0, i] == want


@pytest.mark.parametrize("n", [2, 3, 4, 5, 8, 13, 16, 100])
def test_operation_counts(n):
    # eval = (n-1) tree + 1 value; grad = 2*base-4 + 2*ell + n (test_evaldiff.py:22-47)
    L, c = _single_monomial(n, [(v, 1) for v in range(n)])
    x = np.zeros((2, n))
    x[0] = np.arange(2, n + 2)
    _, _, (em, gm) = oracle.evaluate(L, c, x)
    base = 1 << (n.bit_length() - 1)
    assert em == n
    assert gm == 2 * base - 4 + 2 * (n - base) + n


def test_monomial_hand_values():
    # test_evaldiff.py:96-127
    L = oracle.Level("dd", False)
    c = oracle.CSR.from_polys(2, [[((2.0, 0.0), ((0, 3), (1, 1)))]], L)
    f, J, _ = oracle.evaluate(L, c, np.array([[0.0, 5.0], [0.0, 0.0]]))
    assert f[0, 0] == 0.0 and J[0, 0, 0] == 0.0 and J[0, 0, 1] == 0.0
    c = oracle.CSR.from_polys(1, [[((3.0, 0.0), ((0, 4),))]], L)
    f, J, _ = oracle.evaluate(L, c, np.array([[2.0], [0.0]]))
    assert f[0, 0] == 48.0 and J[0, 0, 0] == 96.0
    c = oracle.CSR.from_polys(2, [[((1.0, 0.0), ((0, 2), (1, 3)))]], L)
    f, J, _ = oracle.evaluate(L, c, np.array([[2.0, 3.0], [0.0, 0.0]]))
    assert f[0, 0] == 108.0 and J[0, 0, 0] == 108.0 and J[0, 0, 1] == 108.0


# -- L3 (3) least squares ------------------------------------------------------------

@pytest.mark.parametrize("name", [n for n in golden_names("mgs_") if "breakdown" not in n])
def test_mgs_matches_reference(name):
    g = golden(name)
    L = oracle_level(str(g["level"]))
    x, z, Q, R = oracle.least_squares(L, g["aug"])
    assert same(Q, g["Q"])
    assert same(R, g["R"])
    assert same(x, g["x"])
    assert z == float(g["z"])


def test_mgs_breakdown_matches_reference():
    g = golden("mgs_breakdown_rdd")
    with pytest.raises(oracle.Breakdown) as e:
        oracle.mgs_qr(oracle_level("rdd"), g["aug"])
    k, rkk, thr = g["breakdown"]
    assert (e.value.k, e.value.rkk, e.value.threshold) == (int(k), rkk, thr)


def test_mgs_parallel_is_bit_identical():
    g = golden("mgs_96x64_cdd")
    L = oracle_level("cdd")
    a = oracle.least_squares(L, g["aug"], nthreads=1)
    b = oracle.least_squares(L, g["aug"], nthreads=4)
    assert all(same(u, v) for u, v in zip((a[0], a[2], a[3]), (b[0], b[2], b[3])))


# -- Newton ------------------------------------------------------------------------------

def test_newton_c1_matches_reference():
    g = golden("newton_c1")
    L = oracle_level("cd")
    xn, f, dx = oracle.newton_step(L, csr_of(g), g["x"])
    assert same(f, g["f"])
    assert same(xn, g["x_next"])


@pytest.mark.parametrize("name", [n for n in golden_names("newton_") if n != "newton_c1"])
def test_newton_trace_matches_reference(name):
    g = golden(name)
    L = oracle_level(str(g["level"]))
    if "shifted_poly_ptr" in g:
        c = csr_of(g, "shifted_")
        x0 = g["z"]
    else:
        c = csr_of(g)
        x0 = g["x0"]
    ref = str(g["trace"])
    iters = ref.count("\n") + (0 if bool(g["converged"]) else 0)
    text, x, conv = oracle.run_newton_trace(L, c, x0, max_iters=max(iters, 1))
    assert text == ref
    assert conv == bool(g["converged"])
    assert same(x, g["x_final"])
