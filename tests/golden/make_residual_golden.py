"""Golden values of the reference's residual_check (mgs.py:311-357) on the
committed MGS goldens of the d and dd levels, written to residuals.json.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_residual_golden.py

The qd levels are skipped: the reference checks them in 320-bit mpfr
(gmpy2), which the GPU path does not offer.
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


def main():
    vals = {}
    for path in sorted(glob.glob(os.path.join(OUT, "mgs_*.npz"))):
        name = os.path.basename(path)[:-4]
        with np.load(path) as z:
            g = {k: z[k] for k in z.files}
        lv = str(g["level"])
        if lv[1:] == "qd" or "Q" not in g:
            continue
        level = xprec.precision_level(lv[1:], lv[0] == "c")
        n = g["Q"].shape[-1]
        a = g["aug"][..., :, :n]
        vals[name] = mgs.residual_check(a, g["Q"], g["R"][..., :n, :n], level)
    with open(os.path.join(OUT, "residuals.json"), "w") as f:
        json.dump(vals, f, indent=1, sort_keys=True)
    print(json.dumps(vals, indent=1))


if __name__ == "__main__":
    main()
