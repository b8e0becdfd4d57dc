"""Host-side logic and the C ABI surface (CPU only: no kernel launches)."""

import ctypes
import os
import re
from fractions import Fraction

import numpy as np
import pytest

from conftest import ROOT, golden

HEADER = os.path.join(ROOT, "include", "polynewt_b200.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char \*)\s*(pn_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_1402_2626_b200 import _lib
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"
    assert lib.pn_version() >= 100


def test_no_device_is_reported_not_faked():
    from paper_1402_2626_b200 import _lib
    n = _lib.device_count()
    assert n >= 0
    if n == 0:
        with pytest.raises(RuntimeError):
            _lib.require_gpu()


def test_error_codes_map_to_reference_exceptions():
    from paper_1402_2626_b200 import _lib
    from paper_1402_2626_b200.mgs import MgsBreakdownError, SingularMatrixError
    info = _lib.NumInfo(k=3, index=5, rkk=1e-40, threshold=1e-30)
    with pytest.raises(MgsBreakdownError) as e:
        _lib.check(_lib.PN_E_BREAKDOWN, info)
    assert e.value.k == 3
    with pytest.raises(SingularMatrixError) as e:
        _lib.check(_lib.PN_E_SINGULAR, info)
    assert e.value.index == 5
    with pytest.raises(ValueError):
        _lib.check(_lib.PN_E_ARG)


def test_argument_validation_without_gpu():
    """pn_system_create validates supports like Monomial/PolySystem before
    touching the device."""
    from paper_1402_2626_b200 import _lib
    lib = _lib.load()
    h = ctypes.c_void_p()
    pp = np.array([0, 1], np.int32)
    mp = np.array([0, 2], np.int32)
    vi = np.array([3, 1], np.int32)  # not increasing
    ex = np.array([1, 1], np.int32)
    co = np.ones((2, 1, 1))
    rc = lib.pn_system_create(1, 1, 1, 4, 1, 2, _lib.ptr(pp), _lib.ptr(mp), _lib.ptr(vi), _lib.ptr(ex),
                              _lib.ptr(co), 0, ctypes.byref(h))
    assert rc == _lib.PN_E_ARG
    assert "strictly increasing" in _lib.last_error()
    vi = np.array([1, 9], np.int32)  # out of range
    rc = lib.pn_system_create(1, 1, 1, 4, 1, 2, _lib.ptr(pp), _lib.ptr(mp), _lib.ptr(vi), _lib.ptr(ex),
                              _lib.ptr(co), 0, ctypes.byref(h))
    assert rc == _lib.PN_E_ARG and "out of range" in _lib.last_error()


def test_generator_is_deterministic_and_valid():
    from paper_1402_2626_b200.generators import random_sparse_system
    from paper_1402_2626_b200.xprec import precision_level
    level = precision_level("dd", True)
    a = random_sparse_system(64, 16, 8, level, seed=3, maxexp=3)
    b = random_sparse_system(64, 16, 8, level, seed=3, maxexp=3)
    assert np.array_equal(a.var_idx, b.var_idx) and np.array_equal(a.coeffs, b.coeffs)
    assert a.monomials == 64 * 16 and a.support == 64 * 16 * 8
    k = np.diff(a.mon_ptr)
    assert np.all(k == 8)
    for c in range(0, a.monomials, 37):
        v = a.var_idx[a.mon_ptr[c]:a.mon_ptr[c + 1]]
        assert np.all(np.diff(v) > 0) and v.min() >= 0 and v.max() < 64
    assert a.exps.min() >= 1 and a.exps.max() <= 3
    mag = np.abs(a.coeffs[:, 0])
    assert mag.min() >= 0.5 and mag.max() < 2.0
    assert np.all(a.coeffs[:, 1] == 0.0)


@pytest.mark.parametrize("n,T,k,maxexp,m,kmin,lv", [
    (64, 16, 8, 3, None, None, "cdd"), (1024, 64, 32, 3, None, 1, "cqd"), (50, 7, 5, 2, 80, 0, "rd"),
    (1024, 8, 32, 1, 1536, None, "cqd")])
def test_oracle_generator_matches_product_generator(n, T, k, maxexp, m, kmin, lv):
    """bench.py's reference arm builds F(n,T,k) with the oracle's own
    generator (no product library); it must give the product's arrays,
    including the C2 "mixed" variant (kmin < k)."""
    import oracle
    from conftest import level_from_name, oracle_level
    from paper_1402_2626_b200.generators import random_sparse_system
    p = random_sparse_system(n, T, k, level_from_name(lv), seed=5, maxexp=maxexp, m=m, kmin=kmin)
    c = oracle.random_sparse_csr(n, T, k, oracle_level(lv), seed=5, maxexp=maxexp, m=m, kmin=kmin)
    for a, b in [(p.poly_ptr, c.poly_ptr), (p.mon_ptr, c.mon_ptr), (p.var_idx, c.var_idx), (p.exps, c.exps),
                 (p.coeffs, c.coeffs)]:
        assert np.array_equal(a, b)
    ks = np.diff(c.mon_ptr)
    lo = k if kmin is None else kmin
    assert ks.min() >= lo and ks.max() <= k
    if kmin is not None and T * (m or n) > 1000:
        assert ks.min() == lo and ks.max() == k  # the whole range is drawn
    assert c.exps.min() >= 1 and c.exps.max() <= maxexp


def test_canonical_sparse_key_equals_dense_key():
    # the sparse key orders like the dense exponent vector
    from paper_1402_2626_b200.polyrep import Monomial
    rng = np.random.default_rng(0)
    mons = []
    for _ in range(300):
        k = int(rng.integers(0, 5))
        vs = sorted(rng.choice(12, size=k, replace=False).tolist())
        mons.append(Monomial(1.0, tuple((v, int(rng.integers(1, 3))) for v in vs)))
    dense = sorted(range(300), key=lambda i: mons[i].exponent_key(12))
    sparse = sorted(range(300), key=lambda i: mons[i].sparse_key())
    assert dense == sparse


def test_monomial_validation():
    from paper_1402_2626_b200.polyrep import Monomial, PolySystem
    from paper_1402_2626_b200.xprec import precision_level
    dd = precision_level("dd", False)
    with pytest.raises(ValueError):
        Monomial(dd.zero(), ((0, 1),))
    with pytest.raises(ValueError):
        Monomial(dd.one(), ((1, 1), (0, 1)))
    with pytest.raises(ValueError):
        Monomial(dd.one(), ((0, 0),))
    with pytest.raises(ValueError):
        PolySystem(2, [[Monomial(dd.one(), ((2, 1),))]])


def test_precision_level_and_scalars():
    from paper_1402_2626_b200.xprec import (DoubleDouble, QuadDouble, precision_level, render_decimal)
    cqd = precision_level("qd", True)
    assert cqd.cshape == (2, 4) and cqd.es == 8 and cqd.eps == 2.0 ** -209
    x = cqd.from_float(1.5, -2.0)
    assert cqd.to_components(x) == [1.5, 0, 0, 0, -2.0, 0, 0, 0]
    assert cqd.from_components(cqd.to_components(x)) == x
    third = precision_level("dd", False).from_fraction(Fraction(1, 3))
    assert third.comps[0] == 1 / 3 and third.comps[1] != 0.0
    assert render_decimal(third).startswith("3.333333333333333333333333333333")
    assert float(QuadDouble(1.0, 2.0 ** -60)) == 1.0
    assert DoubleDouble(-0.0).comps == (0.0, 0.0)
    planes = cqd.to_planes([x, -x])
    assert planes.shape == (2, 4, 2)
    assert cqd.from_planes(planes) == [x, -x]


def test_reference_scalars_are_accepted_by_packing():
    """Coefficients may be the reference's own objects (duck typing)."""
    from paper_1402_2626_b200.polyrep import Monomial, PackedSystem, PolySystem
    from paper_1402_2626_b200.xprec import precision_level

    class RefDD:  # stand-in with the reference's attribute layout
        def __init__(self, hi, lo=0.0):
            self.comps = (hi, lo)

    class RefComplex:
        def __init__(self, re, im):
            self.re, self.im = re, im

    cdd = precision_level("dd", True)
    sys_ = PolySystem(3, [[Monomial(RefComplex(RefDD(1.0), RefDD(2.0)), ((0, 1), (2, 2)))]])
    p = PackedSystem.from_system(sys_, cdd)
    assert p.coeffs.shape == (2, 2, 1)
    assert p.coeffs[0, 0, 0] == 1.0 and p.coeffs[1, 0, 0] == 2.0
    assert p.var_idx.tolist() == [0, 2] and p.exps.tolist() == [1, 2]


def test_golden_fixture_manifest():
    import json
    names = json.load(open(os.path.join(ROOT, "tests", "golden", "MANIFEST.json")))
    assert len(names) >= 40
    g = golden("newton_c1")
    assert int(g["n_vars"]) == 32 and g["poly_ptr"][-1] == 32 * 32


def test_with_constant_terms_host_logic():
    """batch._with_constant_terms: every polynomial gets exactly one constant
    term (a placeholder 1 where it had none), the other monomials keep their
    order, and base_const points at the original constants."""
    from paper_1402_2626_b200.batch import _with_constant_terms
    from paper_1402_2626_b200.polyrep import PackedSystem
    from paper_1402_2626_b200.xprec import precision_level
    rng = np.random.default_rng(5)
    for trial in range(20):
        level = precision_level(["d", "dd", "qd"][trial % 3], trial % 2 == 0)
        m, n = int(rng.integers(1, 8)), 6
        pp, mp, vi, had = [0], [0], [], []
        for _ in range(m):
            terms = [sorted(rng.choice(n, int(rng.integers(1, 4)), replace=False).tolist())
                     for _ in range(int(rng.integers(0, 6)))]
            hasc = bool(rng.random() < 0.5)
            if hasc:
                terms.insert(int(rng.integers(0, len(terms) + 1)), [])
            had.append(hasc)
            for vs in terms:
                vi += vs
                mp.append(len(vi))
            pp.append(len(mp) - 1)
        M = len(mp) - 1
        coeffs = rng.uniform(-1, 1, level.cshape + (M,))
        p = PackedSystem(level, n, np.array(pp, np.int32), np.array(mp, np.int32), np.array(vi, np.int32),
                         np.ones(len(vi), np.int32), coeffs)
        q, base = _with_constant_terms(p)
        ks_q = np.diff(q.mon_ptr)
        for i in range(m):
            lo, hi = q.poly_ptr[i], q.poly_ptr[i + 1]
            assert int((ks_q[lo:hi] == 0).sum()) == 1
            assert (base[i] >= 0) == had[i]
            if had[i]:
                assert np.diff(p.mon_ptr)[base[i]] == 0
        assert np.array_equal(q.var_idx, p.var_idx)
        kept = ks_q[ks_q > 0]
        assert np.array_equal(kept, np.diff(p.mon_ptr)[np.diff(p.mon_ptr) > 0])


def test_cyclic_packed_equals_object_builder():
    """The numpy CSR builder of cyclic n-roots (67 M support entries at
    n = 512) equals PackedSystem.from_system of the Monomial builder."""
    import numpy as np
    from paper_1402_2626_b200.generators import cyclic_n_roots, cyclic_packed
    from paper_1402_2626_b200.polyrep import PackedSystem
    from paper_1402_2626_b200.xprec import precision_level
    for base, cplx in (("dd", True), ("qd", False), ("d", True)):
        level = precision_level(base, cplx)
        for n in (2, 3, 8, 17):
            a = cyclic_packed(n, level)
            b = PackedSystem.from_system(cyclic_n_roots(n, level), level)
            for x, y in ((a.poly_ptr, b.poly_ptr), (a.mon_ptr, b.mon_ptr), (a.var_idx, b.var_idx),
                         (a.exps, b.exps), (a.coeffs, b.coeffs)):
                assert np.array_equal(x, y)
            assert np.array_equal(np.signbit(a.coeffs), np.signbit(b.coeffs))


def test_point_planes_refuses_wrong_shape_and_dtype():
    """The C ABI reads exactly cshape * n doubles from the point pointer, so
    the Python boundary refuses any other shape."""
    import numpy as np
    import pytest
    from paper_1402_2626_b200.evaldiff import point_planes
    from paper_1402_2626_b200.xprec import precision_level
    cdd = precision_level("dd", True)
    ok = point_planes(np.zeros((2, 2, 5)), cdd, 5)
    assert ok.shape == (2, 2, 5) and ok.dtype == np.float64
    assert point_planes(np.zeros((2, 2, 3, 5)), cdd, 5, 3).shape == (2, 2, 3, 5)
    for bad in (np.zeros((2, 1, 5)), np.zeros((2, 2, 4)), np.zeros((2, 5)), np.zeros((2, 2, 2, 5))):
        with pytest.raises(ValueError):
            point_planes(bad, cdd, 5)
    # float32 input is converted, not reinterpreted
    assert point_planes(np.ones((2, 2, 5), np.float32), cdd, 5).dtype == np.float64
