"""System text format (polyrep.py:140-304) against the reference's own
outputs (tests/golden/text_format.json, made by make_text_golden.py):
serialize_system must write the reference's text byte for byte, parse_system
must recover the same monomials (exponents and every coefficient component),
and malformed inputs must raise SystemParseError with the reference's message,
line and column.  Host-only (no GPU)."""

import json
import os

import pytest

from conftest import GOLDEN, level_from_name

with open(os.path.join(GOLDEN, "text_format.json")) as _f:
    G = json.load(_f)


def _system(case, key, n_vars):
    from paper_1402_2626_b200.polyrep import Monomial, PolySystem
    level = level_from_name(case["level"])
    polys = [[Monomial(level.from_components(c), tuple(tuple(e) for e in ex)) for ex, c in poly]
             for poly in case[key]]
    return PolySystem(n_vars, polys)


def _dump(system, level):
    return [[[list(map(list, mon.exponents)), level.to_components(mon.coeff)] for mon in poly]
            for poly in system.polys]


def _exact(dump):
    """Components as repr strings: -0.0 and 0.0 must not compare equal."""
    return [[[ex, [repr(float(c)) for c in comps]] for ex, comps in poly] for poly in dump]


@pytest.mark.parametrize("i", range(len(G["systems"])))
def test_serialize_matches_reference(i):
    from paper_1402_2626_b200.polyrep import serialize_system
    case = G["systems"][i]
    level = level_from_name(case["level"])
    n_vars = int(case["text"].split()[1])
    assert serialize_system(_system(case, "input", n_vars), level) == case["text"]


@pytest.mark.parametrize("i", range(len(G["systems"])))
def test_parse_matches_reference(i):
    from paper_1402_2626_b200.polyrep import parse_system
    case = G["systems"][i]
    level = level_from_name(case["level"])
    assert _exact(_dump(parse_system(case["text"], level), level)) == _exact(case["parsed"])


@pytest.mark.parametrize("i", range(len(G["hand"])))
def test_hand_formatted_inputs(i):
    from paper_1402_2626_b200.polyrep import parse_system, serialize_system
    case = G["hand"][i]
    level = level_from_name(case["level"])
    sysm = parse_system(case["text"], level)
    assert sysm.n_vars == case["n_vars"]
    assert _exact(_dump(sysm, level)) == _exact(case["parsed"])
    assert serialize_system(sysm, level) == case["serialized"]


@pytest.mark.parametrize("i", range(len(G["bad"])))
def test_malformed_inputs(i):
    from paper_1402_2626_b200.polyrep import SystemParseError, parse_system
    case = G["bad"][i]
    level = level_from_name(case["level"])
    with pytest.raises(SystemParseError) as e:
        parse_system(case["text"], level)
    assert str(e.value) == case["error"]["message"]
    assert (e.value.line, e.value.col) == (case["error"]["line"], case["error"]["col"])


def test_round_trip_through_the_device_pack():
    """parse -> PackedSystem -> to_system keeps every monomial and the
    canonical order, so it serialises to the same text as the parsed system
    (not always the input: "-0.0" parses to +0.0 in the reference too)."""
    from paper_1402_2626_b200.polyrep import PackedSystem, parse_system, serialize_system
    for case in G["systems"]:
        level = level_from_name(case["level"])
        sysm = parse_system(case["text"], level)
        back = PackedSystem.from_system(sysm, level).to_system()
        assert serialize_system(back, level) == serialize_system(sysm, level)
        assert _exact(_dump(back, level)) == _exact(_dump(sysm.canonicalized(), level))


@pytest.mark.gpu
@pytest.mark.parametrize("i", [1, 5, 9, 11])
def test_parsed_system_evaluates_like_the_oracle(gpu, i):
    """Text -> parse_system -> device evaluation == the oracle on the same
    packed system (the ingestion path feeds the GPU kernels unchanged)."""
    import numpy as np

    import oracle
    from conftest import oracle_level, same
    from paper_1402_2626_b200.evaldiff import PreparedSystem, evaluate_system
    from paper_1402_2626_b200.polyrep import PackedSystem, parse_system
    case = G["systems"][i]
    level = level_from_name(case["level"])
    p = PackedSystem.from_system(parse_system(case["text"], level), level)
    rng = np.random.default_rng(i)
    x = np.ascontiguousarray(rng.uniform(0.5, 2.0, level.cshape + (p.n_vars,)))
    ev = evaluate_system(PreparedSystem(p), x)
    f, J, _ = oracle.evaluate(oracle_level(case["level"]), oracle.CSR.from_packed(p), x, nthreads=4)
    assert same(ev.f, f)
    assert same(ev.J, J)
