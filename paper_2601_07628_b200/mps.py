"""MPS ingestion and output: the reference's
`parse_mps` / `load_mps` / `write_mps` contract (lp_model.py:229-580), so
real instances reach the B200 solve unchanged.

Host-side text processing (plumbing, not the hot path). Semantics follow the
reference: fixed- or free-format; sections in the standard order
(OBJSENSE, ROWS, COLUMNS, RHS, RANGES, BOUNDS, ENDATA); the first N row is the
objective and later N rows are free constraints; integer MARKER lines are
skipped (LP relaxation); duplicate matrix entries are summed; an RHS on the
objective row is the negated objective constant; RANGES follow the classic
table (E: sign of R picks the side, L: lo = hi - |R|, G: hi = lo + |R|); an
UP bound below zero frees a column whose lower bound is still the default;
maximisation negates c and the constant (internal sense is minimise). Errors
raise `MpsParseError` (a ValueError) with the line number.
"""

from __future__ import annotations

import gzip
import io

import numpy as np

from .problem import LpProblem, SparseMatrix

INF = float("inf")
SECTIONS = ("OBJSENSE", "ROWS", "COLUMNS", "RHS", "RANGES", "BOUNDS")
ROW_BOUNDS = {"E": (0.0, 0.0), "L": (-INF, 0.0), "G": (0.0, INF), "N": (-INF, INF)}


class MpsParseError(ValueError):
    """lp_model.py:30-37."""

    def __init__(self, message: str, line_no: int | None = None):
        self.line_no = line_no
        super().__init__(f"line {line_no}: {message}" if line_no is not None else message)


def _num(tok: str, line_no: int) -> float:
    try:
        return float(tok)
    except ValueError:
        raise MpsParseError(f"expected a number, got {tok!r}", line_no) from None


class _Reader:
    def __init__(self):
        self.name = ""
        self.maximize = False
        self.section = None
        self.history = []
        self.obj_row = None
        self.rows = {}            # name -> index
        self.row_kind = []
        self.row_names = []
        self.cols = {}
        self.col_names = []
        self.ti, self.tj, self.tv = [], [], []
        self.c = {}
        self.rhs = {}
        self.obj_rhs = 0.0
        self.ranges = {}
        self.lo, self.hi = {}, {}
        self.lo_set = set()

    # ---------------------------------------------------------------- helpers
    def col(self, tok: str) -> int:
        j = self.cols.get(tok)
        if j is None:
            j = self.cols[tok] = len(self.col_names)
            self.col_names.append(tok)
        return j

    def pairs(self, toks, start, line_no):
        for k in range(start, len(toks), 2):
            yield toks[k], _num(toks[k + 1], line_no)

    def row_of(self, rname, line_no):
        i = self.rows.get(rname)
        if i is None:
            raise MpsParseError(f"undeclared row {rname!r}", line_no)
        return i

    # ---------------------------------------------------------------- headers
    def header(self, toks, line_no):
        head = toks[0].upper()
        if head == "NAME":
            self.name = toks[1] if len(toks) > 1 else ""
            self.section = "NAME"
            return False
        if head == "ENDATA":
            return True
        if head not in SECTIONS:
            raise MpsParseError(f"unrecognized section header {toks[0]!r}", line_no)
        if self.history and self.history[-1] in SECTIONS and SECTIONS.index(head) < SECTIONS.index(self.history[-1]):
            raise MpsParseError(f"section {head} out of order after {self.history[-1]}", line_no)
        self.history.append(head)
        self.section = head
        if head == "OBJSENSE" and len(toks) > 1:
            self.maximize = toks[1].upper().startswith("MAX")
            self.section = "OBJSENSE_DONE"
        return False

    # ----------------------------------------------------------------- bodies
    def objsense(self, toks, line_no):
        self.maximize = toks[0].upper().startswith("MAX")
        self.section = "OBJSENSE_DONE"

    def rows_line(self, toks, line_no):
        if len(toks) < 2:
            raise MpsParseError("ROWS entry needs a type and a name", line_no)
        kind, rname = toks[0].upper(), toks[1]
        if kind not in ROW_BOUNDS:
            raise MpsParseError(f"unknown row type {toks[0]!r}", line_no)
        if rname in self.rows or rname == self.obj_row:
            raise MpsParseError(f"duplicate row name {rname!r}", line_no)
        if kind == "N" and self.obj_row is None:
            self.obj_row = rname
            return
        self.rows[rname] = len(self.row_names)
        self.row_names.append(rname)
        self.row_kind.append(kind)

    def columns_line(self, toks, line_no):
        if len(toks) >= 3 and toks[1].upper() == "'MARKER'":
            return
        if len(toks) < 3 or len(toks) % 2 == 0:
            raise MpsParseError("COLUMNS entry needs (row, value) pairs", line_no)
        j = self.col(toks[0])
        for rname, v in self.pairs(toks, 1, line_no):
            if rname == self.obj_row:
                self.c[j] = self.c.get(j, 0.0) + v
            else:
                self.ti.append(self.row_of(rname, line_no))
                self.tj.append(j)
                self.tv.append(v)

    def rhs_line(self, toks, line_no):
        if len(toks) < 3:
            raise MpsParseError("RHS entry needs (row, value) pairs", line_no)
        for rname, v in self.pairs(toks, len(toks) % 2, line_no):
            if rname == self.obj_row:
                self.obj_rhs = v
            else:
                self.rhs[self.row_of(rname, line_no)] = v

    def ranges_line(self, toks, line_no):
        if len(toks) < 3:
            raise MpsParseError("RANGES entry needs (row, value) pairs", line_no)
        for rname, v in self.pairs(toks, len(toks) % 2, line_no):
            i = self.row_of(rname, line_no)
            if self.row_kind[i] == "N":
                raise MpsParseError(f"RANGES entry on free row {rname!r}", line_no)
            self.ranges[i] = v

    def bounds_line(self, toks, line_no):
        code = toks[0].upper()
        if code in ("UP", "LO", "FX", "LI", "UI"):
            if len(toks) not in (3, 4):
                raise MpsParseError(f"malformed {code} bound", line_no)
            j, v = self.col(toks[-2]), _num(toks[-1], line_no)
        elif code in ("FR", "MI", "PL", "BV"):
            if len(toks) < 2:
                raise MpsParseError(f"malformed {code} bound", line_no)
            j, v = self.col(toks[-1]), 0.0
        else:
            raise MpsParseError(f"unknown bound code {toks[0]!r}", line_no)
        if code in ("LO", "LI"):
            self.lo[j] = v
            self.lo_set.add(j)
        elif code in ("UP", "UI"):
            self.hi[j] = v
            if v < 0 and j not in self.lo_set:
                self.lo[j] = -INF
        elif code == "FX":
            self.lo[j] = self.hi[j] = v
            self.lo_set.add(j)
        elif code == "FR":
            self.lo[j], self.hi[j] = -INF, INF
            self.lo_set.add(j)
        elif code == "MI":
            self.lo[j] = -INF
            self.lo_set.add(j)
        elif code == "PL":
            self.hi[j] = INF
        else:  # BV
            self.lo[j], self.hi[j] = 0.0, 1.0
            self.lo_set.add(j)

    HANDLERS = {"OBJSENSE": objsense, "ROWS": rows_line, "COLUMNS": columns_line, "RHS": rhs_line,
                "RANGES": ranges_line, "BOUNDS": bounds_line}

    # ----------------------------------------------------------------- driver
    def feed(self, lines):
        for line_no, raw in enumerate(lines, start=1):
            stripped = raw.strip()
            if not stripped or stripped.startswith("*"):
                continue
            toks = raw.split()
            if raw[0] not in " \t":
                if self.header(toks, line_no):
                    break
                continue
            handler = self.HANDLERS.get(self.section)
            if handler is None:
                raise MpsParseError("data line outside any section", line_no)
            handler(self, toks, line_no)
        if "ROWS" not in self.history:
            raise MpsParseError("missing ROWS section")

    def problem(self) -> LpProblem:
        m, n = len(self.row_names), len(self.col_names)
        A = SparseMatrix.from_coo(m, n, self.ti, self.tj, self.tv)
        clo, chi = np.empty(m), np.empty(m)
        for i, kind in enumerate(self.row_kind):
            b = self.rhs.get(i, 0.0)
            lo, hi = ROW_BOUNDS[kind]
            lo, hi = (lo + b if lo == 0.0 else lo), (hi + b if hi == 0.0 else hi)
            if i in self.ranges:
                r = self.ranges[i]
                if kind == "E":
                    lo, hi = (b, b + r) if r >= 0 else (b + r, b)
                elif kind == "L":
                    lo = hi - abs(r)
                elif kind == "G":
                    hi = lo + abs(r)
            clo[i], chi[i] = lo, hi
        c = np.zeros(n)
        for j, v in self.c.items():
            c[j] = v
        vlo, vhi = np.zeros(n), np.full(n, INF)
        for j, v in self.lo.items():
            vlo[j] = v
        for j, v in self.hi.items():
            vhi[j] = v
        bad = np.flatnonzero(vlo > vhi)
        if len(bad):
            raise MpsParseError(f"bounds for column {self.col_names[bad[0]]!r} are inconsistent (lower > upper)")
        const = -self.obj_rhs
        if self.maximize:
            c, const = -c, -const
        return LpProblem(A, c, vlo, vhi, clo, chi, objective_constant=const, maximize=self.maximize,
                         name=self.name, row_names=list(self.row_names), col_names=list(self.col_names))


def parse_mps(source) -> LpProblem:
    """str, bytes (gzip detected by magic bytes) or a file object."""
    if hasattr(source, "read"):
        source = source.read()
    if isinstance(source, bytes):
        if source[:2] == b"\x1f\x8b":
            source = gzip.decompress(source)
        source = source.decode("utf-8", errors="replace")
    r = _Reader()
    r.feed(source.splitlines())
    return r.problem()


def load_mps(path) -> LpProblem:
    with open(path, "rb") as fh:
        return parse_mps(fh.read())


def _g(v: float) -> str:
    return f"{v:.17g}"


def write_mps(problem, name: str = "") -> str:
    """Free-format MPS with normalised names R<i> / C<j>; %.17g values, so a
    re-parse reproduces the problem exactly (lp_model.py:504-580)."""
    A = problem.matrix
    m, n = int(A.num_rows), int(A.num_cols)
    sign = -1.0 if problem.maximize else 1.0
    c = sign * np.asarray(problem.objective, np.float64)
    const = sign * float(problem.objective_constant)
    lc, uc = np.asarray(problem.con_lower), np.asarray(problem.con_upper)
    lv, uv = np.asarray(problem.var_lower), np.asarray(problem.var_upper)
    kinds = np.where(lc == uc, "E", np.where((lc == -INF) & (uc == INF), "N",
                                             np.where(lc == -INF, "L", "G")))
    out = io.StringIO()
    out.write(f"NAME {name or problem.name or 'GRIDLP'}\n")
    if problem.maximize:
        out.write("OBJSENSE\n    MAX\n")
    out.write("ROWS\n N  OBJ\n")
    out.writelines(f" {k}  R{i}\n" for i, k in enumerate(kinds))
    out.write("COLUMNS\n")
    off = np.asarray(A.row_offsets, np.int64)
    rows = np.repeat(np.arange(m), np.diff(off))
    cols = np.asarray(A.col_indices, np.int64)
    order = np.lexsort((rows, cols))               # column-major, rows ascending
    cstart = np.searchsorted(cols[order], np.arange(n + 1))
    vals = np.asarray(A.values, np.float64)
    for j in range(n):
        if c[j] != 0.0:
            out.write(f"    C{j}  OBJ  {_g(c[j])}\n")
        for k in order[cstart[j]:cstart[j + 1]]:
            out.write(f"    C{j}  R{rows[k]}  {_g(vals[k])}\n")
    out.write("RHS\n")
    if const != 0.0:
        out.write(f"    RHS  OBJ  {_g(-const)}\n")
    for i, k in enumerate(kinds):
        if k == "N":
            continue
        b = lc[i] if k in ("E", "G") else uc[i]
        if b != 0.0:
            out.write(f"    RHS  R{i}  {_g(b)}\n")
    ranged = [i for i, k in enumerate(kinds) if k == "G" and uc[i] != INF]
    if ranged:
        out.write("RANGES\n")
        out.writelines(f"    RNG  R{i}  {_g(uc[i] - lc[i])}\n" for i in ranged)
    bounds = []
    for j in range(n):
        lo, hi = lv[j], uv[j]
        if lo == 0.0 and hi == INF:
            continue
        if lo == -INF and hi == INF:
            bounds.append(f" FR BND  C{j}\n")
        elif lo == hi:
            bounds.append(f" FX BND  C{j}  {_g(lo)}\n")
        else:
            if lo == -INF:
                bounds.append(f" MI BND  C{j}\n")
            elif lo != 0.0:
                bounds.append(f" LO BND  C{j}  {_g(lo)}\n")
            if hi != INF:
                bounds.append(f" UP BND  C{j}  {_g(hi)}\n")
    if bounds:
        out.write("BOUNDS\n")
        out.writelines(bounds)
    out.write("ENDATA\n")
    return out.getvalue()
