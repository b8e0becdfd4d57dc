"""Golden vectors for the system text format (polyrep.py:140-304): the
reference's serialize_system output for systems at all six precision levels,
its parse_system result (exponents + coefficient components) for those texts
and for hand-formatted inputs, and the exact SystemParseError text and
position for malformed inputs.

    python tests/golden/make_text_golden.py      # writes text_format.json
"""

from __future__ import annotations

import json
import os
import random
import sys

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from polynewt import polyrep, xprec  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
LEVELS = [("d", False), ("dd", False), ("qd", False), ("d", True), ("dd", True), ("qd", True)]


def name(level):
    return ("c" if level.cplx else "r") + level.base


def decimal(rng):
    digits = "".join(rng.choice("0123456789") for _ in range(rng.randint(1, 40)))
    return f"{rng.choice(['', '-'])}{digits[0]}.{digits[1:] or '0'}e{rng.randint(-30, 30)}"


def coefficient(rng, level):
    kind = rng.randrange(3)
    if kind == 0:
        re_, im_ = rng.uniform(-2, 2), rng.uniform(-2, 2)
        return level.from_float(re_, im_) if level.cplx else level.from_float(re_)
    if kind == 1 or not level.cplx:
        return level.parse(decimal(rng).lstrip("-")) if rng.random() < 0.5 else -level.parse(decimal(rng).lstrip("-"))
    return level.parse(f"({decimal(rng)},{decimal(rng)})")


def random_system(level, seed, m=5, n=7):
    rng = random.Random(seed)
    polys = []
    for _ in range(m):
        poly = []
        for _ in range(rng.randint(1, 6)):
            vs = sorted(rng.sample(range(n), rng.randint(0, 4)))
            poly.append(polyrep.Monomial(coefficient(rng, level), tuple((v, rng.randint(1, 3)) for v in vs)))
        polys.append(poly)
    return polyrep.PolySystem(n, polys)


def dump(system, level):
    return [[[list(map(list, mon.exponents)), level.to_components(mon.coeff)] for mon in poly]
            for poly in system.polys]


HAND = [  # (level, text)
    ("cdd", "2 3\n x0*x1 + 2*x2^3 - (1.5,-2e-3)*x0^2 ;\n-x1*x1 + .5 − 3;\n"),
    ("rqd", "1 2\n0.1*x0 + 1_000*x1^1 - 7;"),
    ("rd", "2 2\nx0;x1*2.5e-3*x0;\n\n"),
    ("cqd", "1 4\n(0.3333333333333333333333333333333333333333333333333333333333333333,1e-70)*x3 + x2^2*x1 - x0;"),
    ("rdd", "1 3\n+x0 - x1 + 3.25*x2^4;"),
    ("cd", "1 1\n(1,2);"),
]

BAD = [  # (level, text) -- every SystemParseError branch
    ("rd", "1\nx0;"), ("rd", "a b\nx0;"), ("rd", "1 2\nx0 + ;"), ("rd", "1 2\n;"), ("rd", "1 2\nx0 x1;"),
    ("rd", "1 2\nx0 + + x1;"), ("rd", "1 2\nx0 + x1"), ("rd", "1 2\nx5;"), ("rd", "1 2\nx0^;"), ("rd", "1 2\nx0^0;"),
    ("rd", "1 2\n2*3*x0;"), ("rd", "1 2\n(1,2)*x0;"), ("rd", "1 2\n1.2.3*x0;"), ("rd", "1 2\nx0;\nx1;"),
    ("rd", "1 2\n0*x0;"), ("rd", "1 2\n*x0;"), ("rd", "1 2\nx0*;"), ("cdd", "1 2\n(1,)*x0;"), ("cdd", "1 2\n(1 2);"),
    ("rd", "2 2\nx0;\n  x1 +\n   y;"), ("rd", "1 2\n3-x0;"), ("rd", "1 1\nx0 −;"), ("rd", ""), ("rd", "1 2 3\nx0;"),
]


def main():
    out = {"systems": [], "hand": [], "bad": []}
    for i, (base, cplx) in enumerate(LEVELS):
        level = xprec.precision_level(base, cplx)
        for seed in (10 * i + 1, 10 * i + 2):
            sysm = random_system(level, seed)
            text = polyrep.serialize_system(sysm, level)
            back = polyrep.parse_system(text, level)
            out["systems"].append({"level": name(level), "input": dump(sysm, level), "text": text,
                                   "parsed": dump(back, level)})
    for lv, text in HAND:
        level = xprec.precision_level(lv[1:], lv[0] == "c")
        sysm = polyrep.parse_system(text, level)
        out["hand"].append({"level": lv, "text": text, "n_vars": sysm.n_vars, "parsed": dump(sysm, level),
                            "serialized": polyrep.serialize_system(sysm, level)})
    for lv, text in BAD:
        level = xprec.precision_level(lv[1:], lv[0] == "c")
        try:
            polyrep.parse_system(text, level)
            err = None
        except polyrep.SystemParseError as e:
            err = {"message": str(e), "line": e.line, "col": e.col}
        except ValueError as e:  # header errors before the scanner exists
            err = {"message": str(e), "type": type(e).__name__}
        out["bad"].append({"level": lv, "text": text, "error": err})
    with open(os.path.join(OUT, "text_format.json"), "w") as f:
        json.dump(out, f, indent=0)
    print(len(out["systems"]), len(out["hand"]), len(out["bad"]))


if __name__ == "__main__":
    main()
