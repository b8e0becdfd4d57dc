"""CUDA path vs the reference (golden vectors) and vs the pinned oracle on
larger seeded inputs.  Bit-exact: every component compared with ==."""

import numpy as np
import pytest

import oracle
from conftest import LEVEL_NAMES, golden, golden_names, level_from_name, oracle_level, same

pytestmark = pytest.mark.gpu


def packed_of(g, prefix=""):
    from paper_1402_2626_b200.polyrep import PackedSystem
    level = level_from_name(str(g["level"]))
    return PackedSystem(level, int(g["n_vars"]), g[prefix + "poly_ptr"].astype(np.int32),
                        g[prefix + "mon_ptr"].astype(np.int32), g[prefix + "var_idx"].astype(np.int32),
                        g[prefix + "exps"].astype(np.int32), np.ascontiguousarray(g[prefix + "coeffs"]))


def csr_of(p):
    return oracle.CSR.from_packed(p)


# -- element-wise arithmetic (test_varith.py:24-70) ----------------------------------

@pytest.mark.parametrize("lv", LEVEL_NAMES)
def test_vec_ops(gpu, lv):
    from paper_1402_2626_b200.varith import VecContext
    g = golden(f"vec_{lv}")
    ctx = VecContext(level_from_name(lv))
    assert same(ctx.add(g["a"], g["b"]), g["add"])
    assert same(ctx.sub(g["a"], g["b"]), g["sub"])
    assert same(ctx.mul(g["a"], g["b"]), g["mul"])
    assert same(ctx.div(g["a"], g["b"]), g["div"])
    assert same(ctx.abs2(g["a"]), g["abs2"])
    assert same(ctx.sqrt_real(g["abs2"]), g["sqrt"])


@pytest.mark.parametrize("lv", LEVEL_NAMES)
def test_tree_sum(gpu, lv):
    from paper_1402_2626_b200.varith import VecContext
    g = golden(f"vec_{lv}")
    ctx = VecContext(level_from_name(lv))
    for n in (1, 2, 3, 5, 7, 8, 33, 100, 257):
        assert same(ctx.tree_sum(g[f"tree_in_{n}"], axis=0), g[f"tree_out_{n}"]), n


@pytest.mark.parametrize("lv", LEVEL_NAMES)
def test_tree_sum_long_vs_oracle(gpu, lv):
    # multi-chunk path of the reduction kernel (> 256 * B elements)
    from paper_1402_2626_b200.varith import VecContext
    L = oracle_level(lv)
    rng = np.random.default_rng(5)
    for n in (1000, 4097, 70001):
        a = rng.uniform(-1, 1, L.cshape + (n,))
        ctx = VecContext(level_from_name(lv))
        assert same(ctx.tree_sum(a, axis=0), oracle.tree_sum(L, a)), n


def test_scalar_arithmetic(gpu):
    from paper_1402_2626_b200.xprec import precision_level
    cdd = precision_level("dd", True)
    a, b = cdd.from_float(1.5, -0.25), cdd.from_float(0.75, 2.0)
    g = golden("vec_cdd")
    del g
    prod = a * b
    assert float(prod.re) == 1.5 * 0.75 + 0.25 * 2.0
    assert (a / a).re == cdd.one().re


# -- evaluation ------------------------------------------------------------------------

@pytest.mark.parametrize("name", golden_names("eval_"))
def test_evaluate_golden(gpu, name):
    from paper_1402_2626_b200.evaldiff import evaluate_system
    g = golden(name)
    ev = evaluate_system(packed_of(g), g["x"])
    assert same(ev.f, g["f"])
    assert same(ev.J, g["J"])
    assert (ev.counter.eval_mults, ev.counter.grad_mults) == tuple(int(c) for c in g["counts"])


@pytest.mark.parametrize("name", ["eval_mixed_cqd", "eval_cyclic40_cdd", "eval_f16_rdd"])
def test_canonical_order_matches_oracle(gpu, name):
    from paper_1402_2626_b200.evaldiff import PreparedSystem
    g = golden(name)
    p = packed_of(g)
    assert np.array_equal(PreparedSystem(p).canonical_order(), csr_of(p).canonical_perm())


def _mixed_system(level, n, T, kmax, seed, maxexp=3, m=None, empty_every=0, const_every=0, dup_every=0):
    """Seeded mixed-support system: k ~ U{1..kmax}, exponents in [1, maxexp],
    constant terms, duplicate monomials and empty polynomials (edge cases of
    evaldiff.py:152-165, 261 and polyrep.py:103-107)."""
    from paper_1402_2626_b200.polyrep import PackedSystem
    rng = np.random.default_rng(seed)
    m = n if m is None else m
    pp, mp, vi, ex, co = [0], [0], [], [], []
    for i in range(m):
        if empty_every and i % empty_every == 1:
            pp.append(len(mp) - 1)
            continue
        terms = []
        for t in range(T):
            k = int(rng.integers(1, kmax + 1))
            vs = np.sort(rng.choice(n, size=k, replace=False))
            es = rng.integers(1, maxexp + 1, size=k)
            terms.append((vs, es))
            if dup_every and t % dup_every == 0:
                terms.append((vs, es))
        if const_every and i % const_every == 0:
            terms.insert(len(terms) // 2, (np.zeros(0, int), np.zeros(0, int)))
        for vs, es in terms:
            vi.extend(vs.tolist())
            ex.extend(es.tolist())
            mp.append(len(vi))
            c = rng.uniform(0.5, 2.0, level.es) * rng.choice([-1.0, 1.0], level.es)
            c[1:level.ncomp] *= 1e-17  # populated low components
            if level.cplx:
                c[level.ncomp + 1:] *= 1e-17
            co.append(c)
        pp.append(len(mp) - 1)
    M = len(co)
    coeffs = np.asarray(co).reshape(M, level.es).T.reshape(level.cshape + (M,))
    return PackedSystem(level, n, np.asarray(pp, np.int32), np.asarray(mp, np.int32), np.asarray(vi, np.int32),
                        np.asarray(ex, np.int32), np.ascontiguousarray(coeffs))


def _point(level, n, seed):
    rng = np.random.default_rng(seed)
    x = rng.uniform(0.5, 2.0, level.cshape + (n,)) * rng.choice([-1.0, 1.0], level.cshape + (n,))
    x.reshape(-1, n)[[i for i in range(level.es) if i % level.ncomp != 0]] *= 1e-17
    return np.ascontiguousarray(x)


@pytest.mark.parametrize("lv", LEVEL_NAMES)
def test_evaluate_mixed_vs_oracle(gpu, lv):
    from paper_1402_2626_b200.evaldiff import evaluate_system
    level = level_from_name(lv)
    p = _mixed_system(level, 48, 40, 32, seed=hash(lv) % 1000, empty_every=7, const_every=5, dup_every=9)
    x = _point(level, 48, 3)
    ev = evaluate_system(p, x)
    f, J, counts = oracle.evaluate(oracle_level(lv), csr_of(p), x)
    assert same(ev.f, f)
    assert same(ev.J, J)
    assert (ev.counter.eval_mults, ev.counter.grad_mults) == counts


@pytest.mark.parametrize("lv", ["cd", "cdd", "cqd", "rqd"])
def test_evaluate_k32_vs_oracle(gpu, lv):
    from paper_1402_2626_b200.evaldiff import evaluate_system
    from paper_1402_2626_b200.generators import random_sparse_system
    level = level_from_name(lv)
    p = random_sparse_system(128, 64, 32, level, seed=42)
    x = _point(level, 128, 4)
    ev = evaluate_system(p, x)
    f, J, _ = oracle.evaluate(oracle_level(lv), csr_of(p), x, nthreads=8)
    assert same(ev.f, f)
    assert same(ev.J, J)


def test_evaluate_large_k_vs_oracle(gpu):
    # k > 32 takes the shared-memory tree kernel (cyclic n-roots family)
    from paper_1402_2626_b200.evaldiff import evaluate_system
    level = level_from_name("cqd")
    p = _mixed_system(level, 300, 6, 260, seed=8, maxexp=2, m=5)
    x = _point(level, 300, 9)
    ev = evaluate_system(p, x)
    f, J, _ = oracle.evaluate(oracle_level("cqd"), csr_of(p), x)
    assert same(ev.f, f)
    assert same(ev.J, J)


def test_evaluate_reference_objects(gpu):
    """The drop-in path: a PolySystem built from Monomial objects."""
    from paper_1402_2626_b200 import evaluate_system
    from paper_1402_2626_b200.generators import cyclic_n_roots, random_point
    from paper_1402_2626_b200.xprec import precision_level
    cdd = precision_level("dd", True)
    g = golden("eval_cyclic5_cdd")
    ev = evaluate_system(cyclic_n_roots(5, cdd), random_point(5, 3, cdd))
    assert same(ev.f, g["f"]) and same(ev.J, g["J"])
    assert ev.values[0] == cdd.from_components(g["f"][..., 0].reshape(-1).tolist())


# -- least squares -----------------------------------------------------------------------

@pytest.fixture(params=["flow", "dataflow", "sweeps", "pipe/late0", "pipe/late1", "pipe/pair", "small"])
def mgs_mode(request, monkeypatch):
    """Every MGS schedule (priority flow, dataflow, launch per sweep, TMA pipe
    with the prefetch before the reduction or after its first barrier, the
    pipe on 2-CTA clusters with q pushed through distributed shared memory
    (d), one CTA)."""
    mode, _, opt = request.param.partition("/")
    monkeypatch.setenv("PN_MGS_MODE", mode)
    if opt.startswith("late"):
        monkeypatch.setenv("PN_PIPE_LATE", opt[4:])
    if opt == "pair":
        monkeypatch.setenv("PN_PIPE_PAIR", "1")
    return mode


@pytest.mark.parametrize("name", [n for n in golden_names("mgs_") if "breakdown" not in n])
def test_least_squares_golden(gpu, mgs_mode, name):
    from paper_1402_2626_b200.mgs import AugmentedMatrix, least_squares_solve, mgs_qr
    from paper_1402_2626_b200.varith import VecContext
    g = golden(name)
    ctx = VecContext(level_from_name(str(g["level"])))
    aug = AugmentedMatrix(ctx, g["aug"])
    res = least_squares_solve(aug)
    assert same(res.factors.Q, g["Q"])
    assert same(res.factors.R, g["R"])
    assert same(res.x, g["x"])
    assert res.z == float(g["z"])
    f = mgs_qr(aug)
    assert same(f.R, g["R"])


def test_breakdown_golden(gpu, mgs_mode):
    from paper_1402_2626_b200.mgs import AugmentedMatrix, MgsBreakdownError, mgs_qr
    from paper_1402_2626_b200.varith import VecContext
    g = golden("mgs_breakdown_rdd")
    with pytest.raises(MgsBreakdownError) as e:
        mgs_qr(AugmentedMatrix(VecContext(level_from_name("rdd")), g["aug"]))
    k, rkk, thr = g["breakdown"]
    assert (e.value.k, e.value.rkk, e.value.threshold) == (int(k), rkk, thr)


@pytest.mark.parametrize("lv,m,n", [("cqd", 160, 128), ("cdd", 513, 200), ("rdd", 1030, 64), ("cd", 256, 256),
                                    ("cdd", 768, 300), ("rd", 512, 512), ("cdd", 1024, 160), ("rdd", 512, 200),
                                    ("cdd", 256, 100), ("cqd", 700, 90), ("rqd", 768, 64), ("cqd", 300, 120)])
def test_least_squares_vs_oracle(gpu, mgs_mode, lv, m, n):
    from paper_1402_2626_b200.mgs import AugmentedMatrix, least_squares_solve
    from paper_1402_2626_b200.varith import VecContext
    L = oracle_level(lv)
    rng = np.random.default_rng(m * n)
    aug = rng.uniform(-1, 1, L.cshape + (m, n + 1))
    aug.reshape(L.es, -1)[[i for i in range(L.es) if i % L.nc != 0]] *= 1e-17
    aug = np.ascontiguousarray(aug)
    res = least_squares_solve(AugmentedMatrix(VecContext(level_from_name(lv)), aug))
    x, z, Q, R = oracle.least_squares(L, aug, nthreads=8)
    assert same(res.factors.R, R)
    assert same(res.factors.Q, Q)
    assert same(res.x, x)
    assert res.z == z


@pytest.mark.parametrize("lv,m", [("cdd", 300), ("rqd", 300), ("cd", 300), ("cdd", 512), ("rd", 512)])
def test_breakdown_mid_factorisation_vs_oracle(gpu, mgs_mode, lv, m):
    """A dependent column deep in the matrix: every CTA of the dataflow kernel
    must stop cleanly and report the reference's (k, rkk, threshold)."""
    from paper_1402_2626_b200.mgs import AugmentedMatrix, MgsBreakdownError, mgs_qr
    from paper_1402_2626_b200.varith import VecContext
    L = oracle_level(lv)
    rng = np.random.default_rng(17)
    aug = rng.uniform(-1, 1, L.cshape + (m, 201))
    aug[..., 157] = aug[..., 3] * 0.5  # exact multiple of column 3
    aug = np.ascontiguousarray(aug)
    with pytest.raises(oracle.Breakdown) as want:
        oracle.mgs_qr(L, aug, nthreads=8)
    with pytest.raises(MgsBreakdownError) as got:
        mgs_qr(AugmentedMatrix(VecContext(level_from_name(lv)), aug))
    assert (got.value.k, got.value.rkk, got.value.threshold) == (want.value.k, want.value.rkk, want.value.threshold)


@pytest.mark.parametrize("bmode", ["look", "single"])
@pytest.mark.parametrize("lv,n", [("cqd", 77), ("cqd", 300), ("cdd", 1000), ("rd", 33), ("cd", 1500), ("rqd", 64),
                                  ("cqd", 31), ("cqd", 64), ("cqd", 1030)])
def test_back_substitution_vs_oracle(gpu, monkeypatch, bmode, lv, n):
    from paper_1402_2626_b200.mgs import back_substitute
    from paper_1402_2626_b200.varith import VecContext
    if bmode == "single" and n > 1024:
        pytest.skip("single-CTA variant is limited to n <= 1024")
    monkeypatch.setenv("PN_BACKSUB_MODE", bmode)
    L = oracle_level(lv)
    rng = np.random.default_rng(n)
    Ra = np.zeros(L.cshape + (n + 1, n + 1))
    Ra[...] = rng.uniform(-1, 1, Ra.shape)
    Ra.reshape(L.es, n + 1, n + 1)[[i for i in range(L.es) if i % L.nc != 0]] *= 1e-17
    Ra[..., np.tril_indices(n + 1, -1)[0], np.tril_indices(n + 1, -1)[1]] = 0.0
    Ra.reshape(L.es, n + 1, n + 1)[0, np.arange(n), np.arange(n)] += 4.0  # well conditioned
    Ra = np.ascontiguousarray(Ra)
    ctx = VecContext(level_from_name(lv))
    got = back_substitute(Ra[..., :n, :n], Ra[..., :n, n], ctx)
    assert same(got, oracle.back_substitute(L, Ra))


@pytest.mark.parametrize("lv", ["cdd", "cqd"])
def test_singular_back_substitution(gpu, lv):
    from paper_1402_2626_b200.mgs import SingularMatrixError, back_substitute
    from paper_1402_2626_b200.varith import VecContext
    ctx = VecContext(level_from_name(lv))
    R = np.zeros(ctx.cshape + (4, 4))
    R[0, 0] = np.eye(4)
    R[0, 0, 2, 2] = 0.0
    with pytest.raises(SingularMatrixError) as e:
        back_substitute(R, np.ones(ctx.cshape + (4,)), ctx)
    assert e.value.index == 2


# -- Newton --------------------------------------------------------------------------------

def test_newton_c1_golden(gpu):
    from paper_1402_2626_b200.evaldiff import PreparedSystem
    from paper_1402_2626_b200.newton import NewtonConfig, newton_step
    g = golden("newton_c1")
    p = packed_of(g)
    level = p.level
    x1, entry, counter, secs = newton_step(PreparedSystem(p), g["x"], NewtonConfig(level=level))
    assert same(level.to_planes(x1), g["x_next"])
    entry.iteration = 0
    assert entry.to_json() == str(g["trace"])


@pytest.mark.parametrize("name", [n for n in golden_names("newton_") if n != "newton_c1"])
def test_run_newton_trace_golden(gpu, name):
    from paper_1402_2626_b200.newton import NewtonConfig, run_newton
    g = golden(name)
    if "shifted_poly_ptr" in g:
        p, x0 = packed_of(g, "shifted_"), g["z"]
    else:
        p, x0 = packed_of(g), g["x0"]
    ref = str(g["trace"])
    trace = run_newton(p, x0, NewtonConfig(level=p.level, max_iters=ref.count("\n")))
    assert trace.to_json_lines() == ref
    assert trace.converged == bool(g["converged"])
    assert same(p.level.to_planes(trace.x), g["x_final"])


@pytest.mark.parametrize("name", ["newton_homotopy_cdd", "newton_homotopy_cqd", "newton_cyclic8_cdd"])
def test_homotopy_start_system_golden(gpu, name):
    from paper_1402_2626_b200.newton import homotopy_start_system
    g = golden(name)
    p = packed_of(g)
    level = p.level
    t = level.from_planes(g["t"])[0]
    s = homotopy_start_system(p, g["z"], t)
    for key in ("poly_ptr", "mon_ptr", "var_idx", "exps"):
        assert np.array_equal(getattr(s, key), g["shifted_" + key]), key
    assert same(s.coeffs, g["shifted_coeffs"])


# -- residual_check (mgs.py:311-357) -----------------------------------------------------

def _residual_goldens():
    import json
    import os
    from conftest import GOLDEN
    with open(os.path.join(GOLDEN, "residuals.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("name", sorted(k for k in _residual_goldens() if k.startswith("mgs_")))
def test_residual_check_golden(gpu, name):
    """GPU residual_check (next precision, GEMM-tiled) == the reference's float."""
    from paper_1402_2626_b200.mgs import residual_check
    g = golden(name)
    level = level_from_name(str(g["level"]))
    n = g["Q"].shape[-1]
    got = residual_check(g["aug"][..., :, :n], g["Q"], g["R"], level)
    assert got == _residual_goldens()[name]


def test_residual_check_fixed_point_is_exact(gpu):
    """The qd check accumulates exactly: Q = I, R = A gives A - QR = 0."""
    from paper_1402_2626_b200.mgs import residual_check
    level = level_from_name("cqd")
    rng = np.random.default_rng(3)
    n = 24
    a = np.zeros(level.cshape + (n, n))
    a[0, 0], a[1, 0] = rng.uniform(-1, 1, (n, n)), rng.uniform(-1, 1, (n, n))
    a[0, 1] = a[0, 0] * 1e-17
    q = np.zeros_like(a)
    q[0, 0] = np.eye(n)
    assert residual_check(a, q, a, level) == 0.0
