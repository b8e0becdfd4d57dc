"""k_mgs_small (one CTA, m <= 32; the default for such systems): Q, R, x and
z bit-identical to the oracle's MGS least squares (mgs.py:145-305) for ragged
row counts, square and tall shapes, and the breakdown report on a dependent
column (mgs.py:176-193)."""

import numpy as np
import pytest

import oracle
from conftest import level_from_name, oracle_level, same

pytestmark = pytest.mark.gpu


def _aug(L, m, n, seed):
    rng = np.random.default_rng(seed)
    aug = rng.uniform(-1, 1, L.cshape + (m, n + 1))
    aug.reshape(L.es, -1)[[i for i in range(L.es) if i % L.nc != 0]] *= 1e-17
    return np.ascontiguousarray(aug)


@pytest.mark.parametrize("lv", ["cd", "cdd", "cqd", "rd", "rdd", "rqd"])
@pytest.mark.parametrize("m,n", [(1, 1), (5, 3), (17, 17), (32, 32), (32, 9), (24, 13), (31, 30)])
def test_small_least_squares_vs_oracle(gpu, lv, m, n):
    from paper_1402_2626_b200.mgs import AugmentedMatrix, least_squares_solve
    from paper_1402_2626_b200.varith import VecContext
    L = oracle_level(lv)
    aug = _aug(L, m, n, 100 * m + n)
    res = least_squares_solve(AugmentedMatrix(VecContext(level_from_name(lv)), aug))
    x, z, Q, R = oracle.least_squares(L, aug, nthreads=4)
    assert same(res.factors.R, R)
    assert same(res.factors.Q, Q)
    assert same(res.x, x)
    assert res.z == z


@pytest.mark.parametrize("lv", ["cdd", "rqd", "cd"])
def test_small_breakdown_vs_oracle(gpu, lv):
    from paper_1402_2626_b200.mgs import AugmentedMatrix, MgsBreakdownError, mgs_qr
    from paper_1402_2626_b200.varith import VecContext
    L = oracle_level(lv)
    aug = _aug(L, 30, 20, 7)
    aug[..., 14] = aug[..., 2] * 0.5  # exact multiple of column 2
    aug = np.ascontiguousarray(aug)
    with pytest.raises(oracle.Breakdown) as want:
        oracle.mgs_qr(L, aug, nthreads=4)
    with pytest.raises(MgsBreakdownError) as got:
        mgs_qr(AugmentedMatrix(VecContext(level_from_name(lv)), aug))
    assert (got.value.k, got.value.rkk, got.value.threshold) == (want.value.k, want.value.rkk, want.value.threshold)
