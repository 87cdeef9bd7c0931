"""MATPOWER numeric-subset parser / writer (pflow/case_io.py:85-260 restated)."""

from pathlib import Path

import numpy as np
import pytest

from _util import SINGLE, case_of, load
from paper_2011_11880_b200 import case as C

REF_CASES = Path("/root/reference/pkg/src/pflow/cases")


def same(a: C.RawCase, b: C.RawCase) -> bool:
    return all(np.array_equal(getattr(a, k), getattr(b, k)) for k in C._COLUMNS) and \
        a.base_mva == b.base_mva


@pytest.mark.parametrize("name", SINGLE)
def test_write_parse_roundtrip(name):
    c = case_of(load(name))
    back = C.parse_case(C.write_case(c), name=name)
    assert same(c, back)


@pytest.mark.skipif(not REF_CASES.exists(), reason="reference fixtures not present")
@pytest.mark.parametrize("name", ["case2", "case5_shift", "case14"])
def test_parse_bundled_fixtures_like_reference(name):
    """The golden arrays came from pflow's own parser."""
    assert same(C.parse_case_file(REF_CASES / f"{name}.m"), case_of(load(name)))


def test_parse_errors_have_line_numbers():
    ok = "mpc.baseMVA = 100;\nmpc.bus = [\n 1 3 0 0 0 0 1 1 0 230;\n];\n" \
         "mpc.gen = [\n 1 0 0 0 0 1 100 1;\n];\nmpc.branch = [\n];\n"
    c = C.parse_case(ok)
    assert c.n_bus == 1 and c.n_gen == 1 and c.n_branch == 0
    with pytest.raises(C.CaseFormatError, match="missing required matrix 'gen'"):
        C.parse_case("mpc.baseMVA = 100;\nmpc.bus = [\n 1 3 0 0 0 0 1 1 0 230;\n];\n"
                     "mpc.branch = [\n];\n")
    with pytest.raises(C.CaseFormatError) as e:
        C.parse_case(ok.replace(" 1 3 0 0 0 0 1 1 0 230;", " 1 3 0 x 0 0 1 1 0 230;"))
    assert e.value.line == 3 and "non-numeric" in str(e.value)
    with pytest.raises(C.CaseFormatError, match="columns"):
        C.parse_case(ok.replace(" 1 3 0 0 0 0 1 1 0 230;", " 1 3 0;"))
    with pytest.raises(C.CaseFormatError, match="duplicate bus id 1"):
        C.parse_case(ok.replace(" 1 3 0 0 0 0 1 1 0 230;",
                                " 1 3 0 0 0 0 1 1 0 230;\n 1 1 0 0 0 0 1 1 0 230;"))
    with pytest.raises(C.CaseFormatError, match="never closed"):
        C.parse_case("mpc.baseMVA = 100;\nmpc.bus = [\n 1 3 0 0 0 0 1 1 0 230;\n")
    with pytest.raises(C.CaseFormatError, match="baseMVA"):
        C.parse_case(ok.replace("mpc.baseMVA = 100;", "mpc.baseMVA = abc;"))


def test_zero_tap_becomes_one():
    txt = ("mpc.baseMVA = 100;\nmpc.bus = [\n 1 3 0 0 0 0 1 1 0 230;\n 2 1 0 0 0 0 1 1 0 230;\n];\n"
           "mpc.gen = [\n 1 0 0 0 0 1 100 1;\n];\n"
           "mpc.branch = [\n 1 2 0.01 0.1 0 0 0 0 0 0 1;\n 1 2 0.01 0.1 0 0 0 0 0.95 2 1;\n];\n")
    c = C.parse_case(txt)
    assert c.ratio.tolist() == [1.0, 0.95] and c.angle.tolist() == [0.0, 2.0]


def test_parser_matches_pflow_on_mutated_cases():
    """Differential check against pflow's own parser (case_io.parse_case):
    400 randomly damaged copies of case14 (lines dropped, duplicated,
    truncated; stray tokens, missing ';' or ']', trailing comments) give
    the same arrays, or the same error message and line, in both."""
    import random

    from oracle.live import import_pflow

    pflow, why = import_pflow()
    if pflow is None:
        pytest.skip(why)
    from pflow import case_io as R

    src = REF_CASES / "case14.m" if REF_CASES.exists() else None
    if src is None:
        pytest.skip("reference fixtures not present")
    base = src.read_text().splitlines()
    rng = random.Random(7)

    def damaged():
        lines = list(base)
        for _ in range(rng.randint(0, 3)):
            i = rng.randrange(len(lines))
            op = rng.randint(0, 7)
            if op == 0:
                lines.pop(i)
            elif op == 1:
                lines.insert(i, lines[rng.randrange(len(lines))])
            elif op == 2:
                lines[i] = lines[i].replace(";", "", 1)
            elif op == 3:
                lines[i] = lines[i].replace(" ", " x ", 1)
            elif op == 4:
                lines[i] = lines[i].replace("]", "", 1)
            elif op == 5:
                lines[i] += " % comment = [ ;"
            elif op == 6:
                lines[i] = lines[i].replace("=", " = ", 1)
            else:
                toks = lines[i].split()
                if len(toks) > 3:
                    lines[i] = " ".join(toks[:rng.randint(1, len(toks))]) + ";"
        return "\n".join(lines) + "\n"

    n_err = 0
    for _ in range(400):
        text = damaged()
        try:
            ref, ref_err = R.parse_case(text, name="x"), None
        except R.CaseFormatError as e:
            ref, ref_err = None, str(e)
        try:
            got, got_err = C.parse_case(text, name="x"), None
        except C.CaseFormatError as e:
            got, got_err = None, str(e)
        assert ref_err == got_err
        if ref_err is None:
            assert same(C.from_rows(ref), got)
        n_err += ref_err is not None
    assert 20 < n_err < 380    # both branches exercised
