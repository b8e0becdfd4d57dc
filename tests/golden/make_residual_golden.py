"""Golden values of the reference's residual_check (mgs.py:311-357) on the
committed MGS goldens, written to residuals.json, plus the reference's own
criterion-5 factorisation (100 x 64 complex qd, test_acceptance.py:129-180).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_residual_golden.py

The qd levels go through 320-bit mpfr in the reference; gmpy2 is not
installed here, so tests/golden/shim/gmpy2.py supplies it over mpmath.
"""

from __future__ import annotations

import glob
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from polynewt import mgs, xprec  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(OUT, "shim"))


def main():
    vals = {}
    for path in sorted(glob.glob(os.path.join(OUT, "mgs_*.npz"))):
        name = os.path.basename(path)[:-4]
        with np.load(path) as z:
            g = {k: z[k] for k in z.files}
        lv = str(g["level"])
        if "Q" not in g:
            continue
        level = xprec.precision_level(lv[1:], lv[0] == "c")
        n = g["Q"].shape[-1]
        a = g["aug"][..., :, :n]
        vals[name] = mgs.residual_check(a, g["Q"], g["R"][..., :n, :n], level)
    # criterion 5's printed case: random_aug(cqd, 100, 64, seed=1164)
    from polynewt.varith import VecContext
    level = xprec.precision_level("qd", True)
    ctx = VecContext(level)
    rng = np.random.default_rng(1164)
    data = np.zeros(ctx.cshape + (100, 65))
    data[0, 0] = rng.uniform(-1.0, 1.0, (100, 65))
    data[1, 0] = rng.uniform(-1.0, 1.0, (100, 65))
    f = mgs.mgs_qr(mgs.AugmentedMatrix(ctx, data))
    vals["criterion5_cqd_100x64"] = mgs.residual_check(data[..., :, :64], f.Q, f.r_square, level)
    with open(os.path.join(OUT, "residuals.json"), "w") as f:
        json.dump(vals, f, indent=1, sort_keys=True)
    print(json.dumps(vals, indent=1))


if __name__ == "__main__":
    main()
