"""Golden outputs of the reference's CLI building blocks for tests/test_cli.py,
produced by running the REFERENCE (polynewt) in this container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_cli_golden.py

* `gen`: serialize_system of the benchmark systems (what `polynewt gen`
  prints, cli.py:247-258), for cyclic and Chandrasekhar at several levels;
* `newton`: the JSON-lines trace of `polynewt newton --benchmark
  chandrasekhar --n 12 --iters 6 --tol 0` (cli.py:150-186: run_newton from
  the all-ones start), whose summary record differs only in timings.

(The reference CLI module itself imports matplotlib, absent here, so the
same calls are made directly.)
"""

import json
import os
import sys
from fractions import Fraction

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from polynewt import bench, newton  # noqa: E402
from polynewt.polyrep import serialize_system  # noqa: E402
from polynewt.xprec import precision_level  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cli.json")


def main():
    gen = {}
    for base, cplx in (("dd", True), ("qd", False), ("d", True), ("qd", True)):
        lv = precision_level(base, cplx)
        name = ("c" if cplx else "r") + base
        gen[f"cyclic 5 {name}"] = serialize_system(bench.cyclic_n_roots(5, lv), lv)
        gen[f"chandrasekhar 6 {name}"] = serialize_system(bench.chandrasekhar_system(6, lv, Fraction(33, 64)), lv)
    lv = precision_level("dd", True)
    system = bench.chandrasekhar_system(12, lv, Fraction(33, 64))
    trace = newton.run_newton(system, [lv.one() for _ in range(12)],
                              newton.NewtonConfig(level=lv, max_iters=6, tol=0.0))
    out = {"gen": gen, "newton_chandrasekhar_12_cdd": trace.to_json_lines(),
           "newton_summary": {"converged": trace.converged, "iterations": len(trace.entries),
                              "final_f_norm": trace.entries[-1].f_norm,
                              "final_dx_norm": trace.entries[-1].dx_norm,
                              "eval_mults": trace.counter.eval_mults, "grad_mults": trace.counter.grad_mults,
                              "precision": lv.name}}
    with open(OUT, "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
