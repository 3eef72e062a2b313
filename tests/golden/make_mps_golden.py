"""Golden fixtures for MPS ingestion, produced by the REFERENCE parser
(`gridlp.lp_model.parse_mps` / `write_mps`, lp_model.py:229-580) on a set of
MPS texts that exercise its rules (fixed/free format, MARKER lines, RANGES
on E/L/G rows, negative UP bounds, FR/MI/PL/BV, OBJSENSE MAX, objective RHS,
duplicate entries, extra N rows, comments) plus the reference's own toy
instance (tests/data/toy3x2.mps) and its documented parse errors.

Run here (the reference does not exist on the GPU box):
    python tests/golden/make_mps_golden.py
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
import make_golden  # noqa: E402,F401  (installs the import stubs and sys.path)
from gridlp.lp_model import MpsParseError, parse_mps, write_mps  # noqa: E402

CASES = {
    "toy3x2": Path("/root/reference/pkg/tests/data/toy3x2.mps").read_text(),
    "ranges_bounds": """NAME RB
ROWS
 N obj
 E e1
 L l1
 G g1
 E e2
 N free1
COLUMNS
    x obj 1.5 e1 1
    x l1 2 g1 -1
    MARKER 'MARKER' 'INTORG'
    y obj -3 e1 1
    y l1 1 e2 4
    MARKER 'MARKER' 'INTEND'
    z free1 1 g1 2
    z e2 -1 g1 0.5
RHS
    rhs obj 7 e1 2
    rhs l1 10 g1 -4
    rhs e2 3
RANGES
    rng e1 5 l1 3
    rng g1 -2 e2 -6
BOUNDS
 UP bnd x 4
 UP bnd y -2
 LO bnd z -1
 UP bnd z 8
 MI bnd w
ENDATA
""",
    "max_free": """NAME MAXP
OBJSENSE
    MAX
ROWS
 N profit
 L cap
 G need
COLUMNS
    a profit 3 cap 1
    a need 1
    b profit 2 cap 1
    c profit 1 need 1
    d profit 0.5 cap 2
RHS
    rhs profit -11 cap 4 need 1
BOUNDS
 FR bnd a
 BV bnd b
 PL bnd c
 FX bnd d 0.25
 LI bnd e 2
 UI bnd e 9
ENDATA
""",
    "free_format_sense_line": """NAME
OBJSENSE MAXIMIZE
ROWS
 N o
 E r1
COLUMNS
 x1 o 1 r1 1
 x2 o 1 r1 1
 x1 r1 2
RHS
 rhs r1 1
ENDATA
""",
}

ERRORS = {
    "bad_number": "NAME X\nROWS\n N o\n E r\nCOLUMNS\n x o abc\nENDATA\n",
    "undeclared_row": "NAME X\nROWS\n N o\n E r\nCOLUMNS\n x q 1\nENDATA\n",
    "out_of_order": "NAME X\nROWS\n N o\nRHS\n r 1\nCOLUMNS\n x o 1\nENDATA\n",
    "no_rows": "NAME X\nCOLUMNS\n x o 1\nENDATA\n",
    "bad_bounds": "NAME X\nROWS\n N o\nCOLUMNS\n x o 1\nBOUNDS\n LO b x 5\n UP b x 1\nENDATA\n",
    "unknown_row_type": "NAME X\nROWS\n Q o\nENDATA\n",
    "duplicate_row": "NAME X\nROWS\n N o\n E r\n L r\nENDATA\n",
    "rhs_two_tokens": "NAME X\nROWS\n N o\n E r\nCOLUMNS\n x r 1\nRHS\n r 1\nENDATA\n",
    "range_on_free": "NAME X\nROWS\n N o\n N f\nCOLUMNS\n x f 1\nRANGES\n r f 1\nENDATA\n",
}


def main():
    arrays, meta = {}, {"cases": {}, "errors": {}}
    for name, text in CASES.items():
        p = parse_mps(text)
        A = p.matrix
        for k, v in (("ptr", A.row_offsets), ("col", A.col_indices), ("val", A.values), ("c", p.objective),
                     ("vlo", p.var_lower), ("vhi", p.var_upper), ("clo", p.con_lower), ("chi", p.con_upper)):
            arrays[f"{name}_{k}"] = np.asarray(v)
        meta["cases"][name] = {"text": text, "shape": [A.num_rows, A.num_cols], "name": p.name,
                               "maximize": p.maximize, "constant": p.objective_constant,
                               "row_names": p.row_names, "col_names": p.col_names,
                               "written": write_mps(p)}
    for name, text in ERRORS.items():
        try:
            parse_mps(text)
            meta["errors"][name] = {"text": text, "line": "no error"}
        except MpsParseError as e:
            meta["errors"][name] = {"text": text, "line": getattr(e, "line_no", None), "message": str(e)}
    np.savez_compressed(HERE / "mps.npz", **arrays)
    (HERE / "mps.json").write_text(json.dumps(meta, indent=1) + "\n")
    print(f"wrote {len(CASES)} cases, {len(ERRORS)} error cases")


if __name__ == "__main__":
    main()
