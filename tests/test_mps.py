"""MPS ingestion (paper_2601_07628_b200/mps.py) against fixtures produced by
the reference parser (tests/golden/make_mps_golden.py): parsed arrays bitwise,
written text identical, parse errors on the same line with the same message."""

import gzip

import numpy as np
import pytest

from conftest import load_json, load_npz
from paper_2601_07628_b200.mps import MpsParseError, parse_mps, write_mps

META = load_json("mps.json")
Z = load_npz("mps.npz")


def _check(p, name):
    m = META["cases"][name]
    A = p.matrix
    assert [A.num_rows, A.num_cols] == m["shape"]
    for k, v in (("ptr", A.row_offsets), ("col", A.col_indices), ("val", A.values), ("c", p.objective),
                 ("vlo", p.var_lower), ("vhi", p.var_upper), ("clo", p.con_lower), ("chi", p.con_upper)):
        np.testing.assert_array_equal(v, Z[f"{name}_{k}"], err_msg=f"{name}.{k}")
    assert (p.name, p.maximize, p.objective_constant) == (m["name"], m["maximize"], m["constant"])
    assert p.row_names == m["row_names"] and p.col_names == m["col_names"]


@pytest.mark.parametrize("name", sorted(META["cases"]))
def test_parse_matches_reference(name):
    text = META["cases"][name]["text"]
    _check(parse_mps(text), name)
    _check(parse_mps(gzip.compress(text.encode())), name)          # gzip detected by magic bytes


@pytest.mark.parametrize("name", sorted(META["cases"]))
def test_write_matches_reference_and_round_trips(name):
    p = parse_mps(META["cases"][name]["text"])
    text = write_mps(p)
    assert text == META["cases"][name]["written"]
    q = parse_mps(text)
    for a, b in ((p.matrix.values, q.matrix.values), (p.objective, q.objective), (p.con_lower, q.con_lower),
                 (p.con_upper, q.con_upper), (p.var_lower, q.var_lower), (p.var_upper, q.var_upper)):
        np.testing.assert_array_equal(a, b)
    assert (p.maximize, p.objective_constant) == (q.maximize, q.objective_constant)


@pytest.mark.parametrize("name", sorted(META["errors"]))
def test_errors_match_reference(name):
    e = META["errors"][name]
    with pytest.raises(MpsParseError) as info:
        parse_mps(e["text"])
    assert info.value.line_no == e["line"]
    assert str(info.value) == e["message"]
    assert isinstance(info.value, ValueError)
