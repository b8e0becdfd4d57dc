"""Generate the golden fixtures in tests/golden/ by running the REFERENCE
implementation (polynewt, /root/reference/pkg/src) in this container.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference cannot travel to the GPU box, so its outputs are committed as
small .npz files; tests compare both the C oracle (CPU) and the CUDA path
(GPU) against them.  Every array is in the reference's component-plane
layout (varith.py:3-8).
"""

from __future__ import annotations

import json
import os
import random
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from polynewt import bench, evaldiff, mgs, newton, polyrep, varith, xprec  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
LEVELS = {f"{'c' if c else 'r'}{b}": xprec.precision_level(b, c) for b in ("d", "dd", "qd") for c in (False, True)}


def lname(level):
    return ("c" if level.cplx else "r") + level.base


def planes(level, values):
    return varith.VecContext(level).from_scalars(list(values))


def random_sparse(n, T, k, level, seed, maxexp=1, m=None, kmin=None, const_every=0):
    """SURVEY 8(d) F(n, T, k, level, seed, maxexp, m) with the reference's
    own Monomial/PolySystem.  kmin: k ~ U{kmin..k} (mixed variant);
    const_every > 0 appends a constant term to every const_every-th poly."""
    rng = random.Random(seed)
    m = n if m is None else m
    polys = []
    for i in range(m):
        terms = []
        for _ in range(T):
            kk = k if kmin is None else rng.randint(kmin, k)
            vs = sorted(rng.sample(range(n), kk))
            exps = tuple((v, rng.randint(1, maxexp)) for v in vs)
            re = rng.uniform(0.5, 2) * rng.choice((-1.0, 1.0))
            im = rng.uniform(0.5, 2) * rng.choice((-1.0, 1.0))
            terms.append(polyrep.Monomial(level.from_float(re, im if level.cplx else 0.0), exps))
        if const_every and i % const_every == 0:
            terms.append(polyrep.Monomial(level.from_float(0.75, -0.25 if level.cplx else 0.0), ()))
        polys.append(terms)
    return polyrep.PolySystem(n, polys)


def csr(system, level):
    pp, mp, vi, ex, co = [0], [0], [], [], []
    for poly in system.polys:
        for mon in poly:
            for v, d in mon.exponents:
                vi.append(v)
                ex.append(d)
            mp.append(len(vi))
            co.append(mon.coeff)
        pp.append(len(mp) - 1)
    return dict(poly_ptr=np.asarray(pp, np.int32), mon_ptr=np.asarray(mp, np.int32),
                var_idx=np.asarray(vi, np.int32), exps=np.asarray(ex, np.int32), coeffs=planes(level, co))


def eval_case(name, system, x, level):
    ev = evaldiff.evaluate_system(system, x)
    ctx = varith.VecContext(level)
    d = csr(system, level)
    d.update(level=lname(level), n_vars=system.n_vars, x=planes(level, x), f=planes(level, ev.values),
             J=ctx.from_scalars([list(r) for r in ev.jacobian]),
             counts=np.asarray([ev.counter.eval_mults, ev.counter.grad_mults], np.int64))
    np.savez_compressed(os.path.join(OUT, f"eval_{name}.npz"), **d)
    print("eval", name, system.monomial_count(), "monomials")


def random_aug(level, m, n, seed, spread=0.0):
    """test_mgs.random_aug / cli._random_augmented style input."""
    ctx = varith.VecContext(level)
    rng = np.random.default_rng(seed)
    data = np.zeros(ctx.cshape + (m, n + 1))
    scale = 10.0 ** (-spread * np.arange(n + 1) / max(n, 1))
    lead = (0, 0) if level.cplx else (0,)
    data[lead] = rng.uniform(-1.0, 1.0, (m, n + 1)) * scale
    if level.cplx:
        data[1, 0] = rng.uniform(-1.0, 1.0, (m, n + 1)) * scale
    return mgs.AugmentedMatrix(ctx, data)


def busy(level, aug, seed):
    """Perturb every entry by a factor (1 + 1e-15 u) in working precision so
    the low components are populated (test_varith.py:14-21 style)."""
    ctx = aug.ctx
    rng = random.Random(seed)
    shape = aug.data.shape[len(ctx.cshape):]
    fac = [level.from_float(1.0 + rng.random() * 1e-14) for _ in range(int(np.prod(shape)))]
    f = ctx.from_scalars(fac).reshape(ctx.cshape + shape)
    return mgs.AugmentedMatrix(ctx, ctx.mul(aug.data, f))


def mgs_case(name, level, m, n, seed, spread=0.0, make_busy=True):
    aug = random_aug(level, m, n, seed, spread)
    if make_busy and level.base != "d":
        aug = busy(level, aug, seed + 100)
    d = dict(level=lname(level), aug=aug.data)
    try:
        res = mgs.least_squares_solve(aug)
        d.update(Q=res.factors.Q, R=res.factors.R, x=res.x, z=np.asarray(res.z))
    except mgs.MgsBreakdownError as e:
        d.update(breakdown=np.asarray([e.k, e.rkk, e.threshold]))
    np.savez_compressed(os.path.join(OUT, f"mgs_{name}.npz"), **d)
    print("mgs", name)


def vec_case(level):
    rng = random.Random(7)

    def scalars(k, s):
        r = random.Random(s)
        out = []
        for _ in range(k):
            x = level.from_float(r.uniform(-2.0, 2.0), r.uniform(-2.0, 2.0) if level.cplx else 0.0)
            out.append(x * level.from_float(1.0 + r.random() * 1e-14))
        return out
    ctx = varith.VecContext(level)
    a, b = scalars(64, 1), scalars(64, 2)
    va, vb = ctx.from_scalars(a), ctx.from_scalars(b)
    d = dict(level=lname(level), a=va, b=vb, add=ctx.add(va, vb), sub=ctx.sub(va, vb), mul=ctx.mul(va, vb),
             div=ctx.div(va, vb), abs2=ctx.abs2(va))
    d["sqrt"] = ctx.sqrt_real(d["abs2"])
    for n in (1, 2, 3, 5, 7, 8, 33, 100, 257):
        vals = scalars(n, 1000 + n)
        arr = ctx.from_scalars(vals)
        d[f"tree_in_{n}"] = arr
        d[f"tree_out_{n}"] = ctx.tree_sum(arr, axis=0)
    del rng
    np.savez_compressed(os.path.join(OUT, f"vec_{lname(level)}.npz"), **d)
    print("vec", lname(level))


def newton_cases():
    # C1 config (BASELINE.json configs[0]): F(32, 32, 8, cd, seed=1), x = random_point(32, 2)
    cd = xprec.precision_level("d", True)
    sys_ = random_sparse(32, 32, 8, cd, seed=1)
    x = bench.random_point(32, 2, cd)
    cfg = newton.NewtonConfig(level=cd, max_iters=1)
    prep = evaldiff.PreparedSystem(sys_)
    x1, entry, counter, _ = newton.newton_step(prep, x, cfg)
    ev = evaldiff.evaluate_system(prep, x)
    d = csr(sys_, cd)
    d.update(level="cd", n_vars=32, x=planes(cd, x), x_next=planes(cd, x1), f=planes(cd, ev.values),
             trace=np.asarray(entry.to_json()))
    np.savez_compressed(os.path.join(OUT, "newton_c1.npz"), **d)
    print("newton c1")

    # homotopy runs with full JSON traces (newton.py:106-159)
    cdd = xprec.precision_level("dd", True)
    cqd = xprec.precision_level("qd", True)
    for name, level, base_sys, zseed, t_val, iters in [
            ("homotopy_cdd", cdd, random_sparse(12, 6, 3, cdd, seed=5), 9, 0.99, 8),
            ("homotopy_cqd", cqd, random_sparse(8, 5, 3, cqd, seed=6), 11, 0.99, 8),
            ("homotopy_cd", cd, random_sparse(16, 8, 4, cd, seed=7), 13, 0.99, 8),
            ("cyclic8_cdd", cdd, bench.cyclic_n_roots(8, cdd), 33, 0.99, 7)]:
        z = bench.random_unit_point(base_sys.n_vars, zseed, level)
        shifted = newton.homotopy_start_system(base_sys, z, level.from_float(t_val))
        trace = newton.run_newton(shifted, z, newton.NewtonConfig(level=level, max_iters=iters))
        d = csr(base_sys, level)
        s2 = csr(shifted, level)
        d.update({f"shifted_{k}": v for k, v in s2.items()})
        d.update(level=lname(level), n_vars=base_sys.n_vars, z=planes(level, z),
                 t=planes(level, [level.from_float(t_val)]), trace=np.asarray(trace.to_json_lines()),
                 x_final=planes(level, trace.x), converged=np.asarray(trace.converged))
        np.savez_compressed(os.path.join(OUT, f"newton_{name}.npz"), **d)
        print("newton", name, len(trace.entries), trace.converged)

    # Chandrasekhar H-equation, real dd and real qd (test_newton.py:18-53)
    for name, level, n, iters in [("chandra_dd", xprec.precision_level("dd", False), 8, 10),
                                  ("chandra_qd", xprec.precision_level("qd", False), 7, 9),
                                  ("chandra_cdd", cdd, 6, 10)]:
        sys_ = bench.chandrasekhar_system(n, level)
        x0 = bench.chandrasekhar_start(n, level)
        trace = newton.run_newton(sys_, x0, newton.NewtonConfig(level=level, max_iters=iters))
        d = csr(sys_, level)
        d.update(level=lname(level), n_vars=n, x0=planes(level, x0), trace=np.asarray(trace.to_json_lines()),
                 x_final=planes(level, trace.x), converged=np.asarray(trace.converged))
        np.savez_compressed(os.path.join(OUT, f"newton_{name}.npz"), **d)
        print("newton", name, len(trace.entries), trace.converged)


def main():
    for level in LEVELS.values():
        vec_case(level)
    # evaluation: every level on a small random system; mixed supports with
    # constants, single-variable bypass, common factors and folded trees
    for lv_name, level in LEVELS.items():
        sys_ = random_sparse(16, 8, 5, level, seed=3)
        eval_case(f"f16_{lv_name}", sys_, bench.random_point(16, 4, level), level)
        mixed = random_sparse(20, 12, 9, level, seed=11, maxexp=3, kmin=1, const_every=3)
        eval_case(f"mixed_{lv_name}", mixed, bench.random_point(20, 12, level), level)
    cdd = LEVELS["cdd"]
    eval_case("cyclic5_cdd", bench.cyclic_n_roots(5, cdd), bench.random_point(5, 3, cdd), cdd)
    eval_case("cyclic40_cdd", bench.cyclic_n_roots(40, cdd), bench.random_point(40, 8, cdd), cdd)
    eval_case("chandra6_rdd", bench.chandrasekhar_system(6, LEVELS["rdd"]),
              bench.random_point(6, 1, LEVELS["rdd"]), LEVELS["rdd"])
    eval_case("wide_cqd", random_sparse(64, 3, 37, LEVELS["cqd"], seed=21, maxexp=2, m=6),
              bench.random_point(64, 22, LEVELS["cqd"]), LEVELS["cqd"])
    eval_case("k32_cd", random_sparse(64, 16, 32, LEVELS["cd"], seed=23), bench.random_point(64, 24, LEVELS["cd"]),
              LEVELS["cd"])
    eval_case("k32_cqd", random_sparse(40, 6, 32, LEVELS["cqd"], seed=25), bench.random_point(40, 26, LEVELS["cqd"]),
              LEVELS["cqd"])
    # MGS: all levels, square / overdetermined / graded / odd sizes
    for lv_name, level in LEVELS.items():
        mgs_case(f"24x13_{lv_name}", level, 24, 13, seed=5)
        mgs_case(f"40x17_{lv_name}", level, 40, 17, seed=9)
    mgs_case("33x33_cqd", LEVELS["cqd"], 33, 33, seed=14)
    mgs_case("96x64_cdd", LEVELS["cdd"], 96, 64, seed=15)
    mgs_case("300x40_cd", LEVELS["cd"], 300, 40, seed=16)
    mgs_case("graded_rdd", LEVELS["rdd"], 16, 8, seed=13, spread=10.0)
    # rank deficiency: column 2 = column 0 + column 1 (test_mgs.py:111-122)
    level = LEVELS["rdd"]
    ctx = varith.VecContext(level)
    data = np.zeros(ctx.cshape + (8, 5))
    cols = np.random.default_rng(3).uniform(-1, 1, (8, 5))
    cols[:, 2] = cols[:, 0] + cols[:, 1]
    data[0] = cols
    try:
        mgs.mgs_qr(mgs.AugmentedMatrix(ctx, data))
        raise SystemExit("expected breakdown")
    except mgs.MgsBreakdownError as e:
        np.savez_compressed(os.path.join(OUT, "mgs_breakdown_rdd.npz"), level="rdd", aug=data,
                            breakdown=np.asarray([e.k, e.rkk, e.threshold]))
        print("mgs breakdown", e.k)
    newton_cases()
    with open(os.path.join(OUT, "MANIFEST.json"), "w") as fh:
        json.dump(sorted(f for f in os.listdir(OUT) if f.endswith(".npz")), fh, indent=1)


if __name__ == "__main__":
    main()
