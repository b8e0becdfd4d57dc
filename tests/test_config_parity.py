"""Parity for the BASELINE.json configurations the round-1 suite left
uncompared (VERDICT r01 "Next round" item 1), all bit-exact against the
pinned oracle:

* C4 overdetermined: one full complex quad-double Newton step at
  1536 x 1024 (flow kernel at NT = 192 plus the six-part row-split tail), and
  a 1300 x 400 least-squares case where both the flow kernel and the tail
  carry columns (mgs.py:145-305);
* C4 square: the first two iterations of the homotopy run, JSONL trace
  byte-identical to the oracle's (newton.py:106-159);
* C2 "mixed" variant: k ~ U{1..32}, maxexp = 3 at dim 1024, which drives the
  power table, common factors, the k <= 1 bypass and every tree bucket
  (evaldiff.py:142-180, polyrep.py:120-139);
* criterion 1's shape (test_acceptance.py:44-61): single monomials with
  k = 512 and 1024 variables, and rows of cyclic 1024-roots.
"""

import os

import numpy as np
import pytest

import oracle
from conftest import level_from_name, oracle_level, same

pytestmark = pytest.mark.gpu
NT = os.cpu_count() or 1


def _point(level, n, seed, busy=True):
    rng = np.random.default_rng(seed)
    x = rng.uniform(0.5, 2.0, level.cshape + (n,)) * rng.choice([-1.0, 1.0], level.cshape + (n,))
    x.reshape(-1, n)[[i for i in range(level.es) if i % level.ncomp != 0]] *= 1e-17 if busy else 0.0
    return np.ascontiguousarray(x)


def _busy_aug(lv, m, n, seed):
    L = oracle_level(lv)
    rng = np.random.default_rng(seed)
    aug = rng.uniform(-1, 1, L.cshape + (m, n + 1))
    aug.reshape(L.es, -1)[[i for i in range(L.es) if i % L.nc != 0]] *= 1e-17
    return L, np.ascontiguousarray(aug)


# -- C4 overdetermined ------------------------------------------------------------

def test_c4_overdetermined_cqd_newton_step_1536x1024(gpu):
    """One full cqd Gauss-Newton step on F(1024, 1024, 32) with m = 1536
    equations: 1536 x 1025 MGS in the NT = 192 flow kernel (two CTAs per SM)
    and the six-part tail, back substitution, update."""
    from paper_1402_2626_b200.evaldiff import PreparedSystem
    from paper_1402_2626_b200.generators import random_sparse_system
    from paper_1402_2626_b200.newton import device_step
    level = level_from_name("cqd")
    p = random_sparse_system(1024, 1024, 32, level, seed=2024, m=1536)
    x = _point(level, 1024, 5)
    res = device_step(PreparedSystem(p), x)
    xn, f, dx = oracle.newton_step(oracle_level("cqd"), oracle.CSR.from_packed(p), x, nthreads=NT)
    assert same(res.f, f)
    assert same(res.dx, dx)
    assert same(res.x_next, xn)


@pytest.mark.parametrize("m,n", [(1300, 400), (1536, 300)])
def test_cqd_flow_and_tail_both_carry_columns(gpu, m, n):
    """m > 1024 selects the NT = 192 flow kernel; with n > 148 it keeps the
    first n + 1 - 148 pivots and the row-split tail the rest (1300 rows: five
    full 256-row parts and a ragged 20-row part)."""
    from paper_1402_2626_b200.mgs import AugmentedMatrix, least_squares_solve
    from paper_1402_2626_b200.varith import VecContext
    L, aug = _busy_aug("cqd", m, n, m * 7 + n)
    res = least_squares_solve(AugmentedMatrix(VecContext(level_from_name("cqd")), aug))
    x, z, Q, R = oracle.least_squares(L, aug, nthreads=NT)
    assert same(res.factors.R, R)
    assert same(res.factors.Q, Q)
    assert same(res.x, x)
    assert res.z == z


# -- C4 square: first iterations of the homotopy run --------------------------------

def test_c4_square_homotopy_first_two_iterations_trace(gpu):
    """bench.py --converge's square C4 input (F(1024,1024,32) cqd shifted by
    -t f(z), t = 0.99, x0 = z on the unit circle): the shift constants equal
    the oracle's -(t * f(z)), and two run_newton iterations give the oracle's
    JSONL trace byte for byte and the same iterate."""
    import math
    from paper_1402_2626_b200.evaldiff import PreparedSystem
    from paper_1402_2626_b200.generators import random_sparse_system
    from paper_1402_2626_b200.newton import NewtonConfig, homotopy_start_system, run_newton
    level = level_from_name("cqd")
    L = oracle_level("cqd")
    n = 1024
    p = random_sparse_system(n, 1024, 32, level, seed=2024)
    rng = np.random.default_rng(2024 + 3)
    theta = rng.uniform(0.0, 2.0 * math.pi, n)
    z = np.zeros(level.cshape + (n,))
    z[0, 0], z[1, 0] = np.cos(theta), np.sin(theta)
    t = level.from_float(0.99)
    shifted = homotopy_start_system(p, z, t)
    # the constants: -(t * f_i(z)) (newton.py:144-158), appended last per polynomial
    f_z, _, _ = oracle.evaluate(L, oracle.CSR.from_packed(p), z, nthreads=NT)
    tp = np.repeat(level.to_planes([t]), n, axis=-1)
    want = -oracle.vec_op(L, "mul", tp, f_z)
    last = np.asarray(shifted.poly_ptr[1:]) - 1
    assert np.all(np.diff(shifted.mon_ptr)[last] == 0)
    assert same(shifted.coeffs[..., last], want)
    tr = run_newton(PreparedSystem(shifted), z, NewtonConfig(level=level, max_iters=2))
    lines, x2, _ = oracle.run_newton_trace(L, oracle.CSR.from_packed(shifted), z, max_iters=2, nthreads=NT)
    assert tr.to_json_lines() == lines
    assert same(level.to_planes(tr.x), x2)
    assert tr.entries[1].f_norm < tr.entries[0].f_norm


# -- C2 mixed variant ----------------------------------------------------------------

@pytest.mark.parametrize("lv", ["cqd", "cdd", "cd"])
def test_c2_mixed_variant_rows_vs_oracle(gpu, lv):
    """F(1024, 1024, 32) with k ~ U{1..32} and exponents in [1, 3]: k = 1
    bypass, common factors, power table rows up to degree 3 and all five
    tree buckets, evaluated in full on the GPU; 8 sampled rows compared."""
    from paper_1402_2626_b200.evaldiff import PreparedSystem, evaluate_system
    from paper_1402_2626_b200.generators import random_sparse_system
    level = level_from_name(lv)
    p = random_sparse_system(1024, 1024, 32, level, seed=77, maxexp=3, kmin=1)
    ks = np.diff(p.mon_ptr)
    assert ks.min() == 1 and ks.max() == 32 and p.exps.max() == 3
    x = _point(level, 1024, 13)
    prep = PreparedSystem(p)
    ev = evaluate_system(prep, x)
    rows = [0, 3, 128, 500, 511, 640, 999, 1023]
    sub = oracle.CSR.from_packed(p).rows(rows)
    f, J, _ = oracle.evaluate(oracle_level(lv), sub, x, nthreads=NT)
    assert same(ev.f[..., rows], f)
    assert same(ev.J[..., rows, :], J)


def test_c2_mixed_variant_op_counts_closed_form(gpu):
    """OpCounter totals of the mixed system equal the closed form of SURVEY
    8(a) summed over the monomials (eval = k + c, grad = 2 base - 4 + 2 ell +
    k + c for k >= 2; (1, [d > 1]) for k = 1)."""
    from paper_1402_2626_b200.evaldiff import PreparedSystem
    from paper_1402_2626_b200.generators import random_sparse_system
    level = level_from_name("cd")
    p = random_sparse_system(1024, 256, 32, level, seed=78, maxexp=3, kmin=1)
    got = PreparedSystem(p).counts()
    ev = gr = 0
    for c in range(p.monomials):
        a, b = p.mon_ptr[c], p.mon_ptr[c + 1]
        k = int(b - a)
        cnt = int((p.exps[a:b] >= 2).sum())
        if k == 1:
            ev, gr = ev + 1, gr + cnt
        elif k >= 2:
            base = 1 << (k.bit_length() - 1)
            ev += k + cnt
            gr += 2 * base - 4 + 2 * (k - base) + k + cnt
    assert (got.eval_mults, got.grad_mults) == (ev, gr)


# -- criterion 1's shape: k = 512 / 1024 ----------------------------------------------

def _packed_rows(level, n, supports, coeffs):
    from paper_1402_2626_b200.polyrep import PackedSystem
    poly_ptr = np.array([0] + list(np.cumsum([len(s) for s in supports])), np.int32)
    mons = [m for s in supports for m in s]
    mon_ptr = np.array([0] + list(np.cumsum([len(m) for m in mons])), np.int32)
    var_idx = np.concatenate([np.asarray(m, np.int32) for m in mons]) if mons else np.zeros(0, np.int32)
    exps = np.ones(len(var_idx), np.int32)
    return PackedSystem(level, n, poly_ptr, mon_ptr, var_idx, exps, np.ascontiguousarray(coeffs))


@pytest.mark.parametrize("lv", ["rdd", "cqd", "cdd"])
@pytest.mark.parametrize("k", [512, 1024, 2048, 4096])
def test_single_large_monomial_vs_oracle(gpu, lv, k):
    """One monomial of k variables at x_j = 1 + j/(64k) (the shape of
    test_acceptance.py:46-61, scaled so the k = 4096 product stays finite):
    value, all k partial derivatives and the analytic counts: the product
    tree's k-1 / 2k-4 (test_acceptance.py:46-61) plus the k coefficient
    scalings of eval_monomial_and_derivs, i.e. k / 3k-4 (k a power of two).
    k = 2048 (cqd) and 4096 (cdd, cqd) keep the tree levels in global
    scratch instead of shared memory."""
    from paper_1402_2626_b200.evaldiff import PreparedSystem, evaluate_system
    level = level_from_name(lv)
    coeffs = np.zeros(level.cshape + (1,))
    coeffs.reshape(level.es, 1)[0, 0] = 1.0
    p = _packed_rows(level, k, [[list(range(k))]], coeffs)
    x = np.zeros(level.cshape + (k,))
    x.reshape(level.es, k)[0] = 1.0 + np.arange(k) / (64.0 * k)
    if level.cplx:
        x[1, 0] = 1e-3 * np.cos(np.arange(k))
    ev = evaluate_system(PreparedSystem(p), x)
    f, J, counts = oracle.evaluate(oracle_level(lv), oracle.CSR.from_packed(p), x)
    assert same(ev.f, f)
    assert same(ev.J, J)
    assert counts == (k, 3 * k - 4)
    assert (ev.counter.eval_mults, ev.counter.grad_mults) == counts


@pytest.mark.parametrize("lv", ["cqd", "cdd"])
def test_cyclic_1024_rows_vs_oracle(gpu, lv):
    """Rows of cyclic 1024-roots (bench.py:51-69): polynomial i has 1024
    monomials of i consecutive (cyclic) variables.  Rows with i = 511, 512
    and 1023 (k up to 1023, one CTA per monomial) plus the last row (the
    1024-variable product and the constant -1)."""
    from paper_1402_2626_b200.evaldiff import PreparedSystem, evaluate_system
    n = 1024
    level = level_from_name(lv)
    rows = [511, 512, 1023]
    supports = [[sorted((j + q) % n for q in range(i)) for j in range(n)] for i in rows]
    supports.append([list(range(n)), []])
    M = sum(len(s) for s in supports)
    coeffs = np.zeros(level.cshape + (M,))
    coeffs.reshape(level.es, M)[0] = 1.0
    coeffs.reshape(level.es, M)[0, M - 1] = -1.0
    p = _packed_rows(level, n, supports, coeffs)
    rng = np.random.default_rng(9)
    theta = rng.uniform(0.0, 2.0 * np.pi, n)
    x = np.zeros(level.cshape + (n,))
    x[0, 0], x[1, 0] = np.cos(theta), np.sin(theta)
    ev = evaluate_system(PreparedSystem(p), x)
    f, J, _ = oracle.evaluate(oracle_level(lv), oracle.CSR.from_packed(p), x, nthreads=NT)
    assert same(ev.f, f)
    assert same(ev.J, J)


@pytest.mark.parametrize("warp", ["1", "0"])
@pytest.mark.parametrize("lv", ["cd", "cdd", "cqd", "rqd"])
def test_cyclic_300_all_large_buckets_vs_oracle(gpu, monkeypatch, lv, warp):
    """Full cyclic 300-roots (k = 1 .. 300: tree buckets up to base 32 and
    the large buckets of base 64, 128, 256), evaluated with one warp per
    large monomial (default) and one CTA per monomial (PN_LARGE_WARP=0);
    sampled rows against the oracle."""
    from paper_1402_2626_b200.evaldiff import PreparedSystem, evaluate_system
    from paper_1402_2626_b200.generators import cyclic_packed
    monkeypatch.setenv("PN_LARGE_WARP", warp)
    n = 300
    level = level_from_name(lv)
    p = cyclic_packed(n, level)
    rng = np.random.default_rng(17)
    x = np.zeros(level.cshape + (n,))
    if level.cplx:
        theta = rng.uniform(0.0, 2.0 * np.pi, n)
        x[0, 0], x[1, 0] = np.cos(theta), np.sin(theta)
    else:
        x[0] = rng.uniform(0.9, 1.1, n) * rng.choice([-1.0, 1.0], n)
    ev = evaluate_system(PreparedSystem(p), x)
    rows = [0, 31, 32, 63, 64, 100, 127, 128, 255, 256, 298, 299]
    f, J, _ = oracle.evaluate(oracle_level(lv), oracle.CSR.from_packed(p).rows(rows), x, nthreads=NT)
    assert same(ev.f[..., rows], f)
    assert same(ev.J[..., rows, :], J)


@pytest.mark.parametrize("lv,m,n", [("cdd", 4096, 48), ("cd", 3000, 200), ("rdd", 2100, 130), ("rqd", 4064, 40),
                                    ("rqd", 2100, 90), ("cdd", 2500, 60), ("rqd", 3048, 50)])
@pytest.mark.parametrize("wide", ["2", "1", "0"])
def test_tall_least_squares_wide_flow_vs_oracle(gpu, monkeypatch, lv, m, n, wide):
    """1024 < m <= 4096 rows: d/dd take the 512-thread (dd) or 1024-thread
    flow kernel (default above 2048 rows, PN_FLOW_WIDE) or the dataflow
    kernel, real qd the 512-thread flow kernel or the 256-thread one, against
    the oracle (the shapes of the Chandrasekhar n = 2048..4096 runs)."""
    from paper_1402_2626_b200.mgs import AugmentedMatrix, least_squares_solve
    from paper_1402_2626_b200.varith import VecContext
    monkeypatch.setenv("PN_FLOW_WIDE", wide)
    L, aug = _busy_aug(lv, m, n, m + n)
    res = least_squares_solve(AugmentedMatrix(VecContext(level_from_name(lv)), aug))
    x, z, Q, R = oracle.least_squares(L, aug, nthreads=NT)
    assert same(res.factors.R, R)
    assert same(res.factors.Q, Q)
    assert same(res.x, x)
    assert res.z == z

@pytest.mark.parametrize("lv,m,n", [("cdd", 1600, 120), ("cdd", 1536, 70), ("cdd", 2048, 40)])
@pytest.mark.parametrize("tall", ["1", "0"])
def test_mid_tall_cdd_flow_vs_oracle(gpu, monkeypatch, lv, m, n, tall):
    """complex dd with 1024 < m <= 2048 rows: the flow kernel (default,
    PN_FLOW_TALL) and the dataflow kernel, against the oracle."""
    from paper_1402_2626_b200.mgs import AugmentedMatrix, least_squares_solve
    from paper_1402_2626_b200.varith import VecContext
    monkeypatch.setenv("PN_FLOW_TALL", tall)
    L, aug = _busy_aug(lv, m, n, m + 3 * n)
    res = least_squares_solve(AugmentedMatrix(VecContext(level_from_name(lv)), aug))
    x, z, Q, R = oracle.least_squares(L, aug, nthreads=NT)
    assert same(res.factors.R, R)
    assert same(res.factors.Q, Q)
    assert same(res.x, x)
    assert res.z == z
