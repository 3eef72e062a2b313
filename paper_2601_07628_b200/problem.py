"""Input contract of `solve`: the LP data model.

Mirrors the reference types so a reference user can hand either ours or
theirs to `solve` (duck-typed: any object with `.matrix.row_offsets /
.col_indices / .values / .num_rows / .num_cols` and the five bound/cost
vectors works):

    minimize c'x + const  s.t.  con_lower <= A x <= con_upper,
                                 var_lower <=  x  <= var_upper

Reference: SparseMatrix and LpProblem (/root/reference/pkg/src/gridlp/
lp_model.py:40-200), objective_value / reported_objective (:203-215).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

INF = float("inf")


class SparseMatrix:
    """CSR with int64 offsets/indices and float64 values.

    Same invariants as the reference (lp_model.py:62-88): offsets start at 0,
    end at nnz and never decrease; columns strictly increase inside a row and
    stay in range; values are finite.
    """

    __slots__ = ("num_rows", "num_cols", "row_offsets", "col_indices", "values")

    def __init__(self, num_rows, num_cols, row_offsets, col_indices, values, check=True):
        self.num_rows = int(num_rows)
        self.num_cols = int(num_cols)
        self.row_offsets = np.ascontiguousarray(row_offsets, dtype=np.int64)
        self.col_indices = np.ascontiguousarray(col_indices, dtype=np.int64)
        self.values = np.ascontiguousarray(values, dtype=np.float64)
        if check:
            self.validate()

    def validate(self):
        m, n = self.num_rows, self.num_cols
        off, col, val = self.row_offsets, self.col_indices, self.values
        if off.shape != (m + 1,):
            raise ValueError(f"row_offsets has length {off.shape[0]}, expected {m + 1}")
        if off[0] != 0 or off[-1] != len(val):
            raise ValueError("row_offsets must start at 0 and end at nnz")
        if np.any(off[1:] < off[:-1]):
            raise ValueError("row_offsets must be non-decreasing")
        if len(col) != len(val):
            raise ValueError("col_indices and values length mismatch")
        if len(col):
            if col.min() < 0 or col.max() >= n:
                raise ValueError("column index out of range")
            inner = np.ones(len(col) - 1, dtype=bool)
            starts = off[1:-1]
            starts = starts[(starts > 0) & (starts < len(col))]
            inner[starts - 1] = False
            if np.any((col[1:] <= col[:-1]) & inner):
                raise ValueError("column indices must be strictly increasing within a row")
            if not np.all(np.isfinite(val)):
                raise ValueError("stored matrix values must be finite")

    @property
    def nnz(self) -> int:
        return int(len(self.values))

    @property
    def shape(self) -> tuple[int, int]:
        return (self.num_rows, self.num_cols)

    def row_nnz(self) -> np.ndarray:
        return np.diff(self.row_offsets)

    def col_nnz(self) -> np.ndarray:
        return np.bincount(self.col_indices, minlength=self.num_cols).astype(np.int64)

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.num_rows, self.num_cols))
        rows = np.repeat(np.arange(self.num_rows), self.row_nnz())
        d[rows, self.col_indices] = self.values
        return d

    @classmethod
    def from_coo(cls, num_rows, num_cols, rows, cols, vals) -> "SparseMatrix":
        """Triplets -> CSR; duplicates summed in input order
        (lp_model.py:121-141)."""
        r = np.asarray(rows, dtype=np.int64)
        c = np.asarray(cols, dtype=np.int64)
        v = np.asarray(vals, dtype=np.float64)
        key = r * max(int(num_cols), 1) + c
        order = np.argsort(key, kind="stable")
        key, r, c, v = key[order], r[order], c[order], v[order]
        if len(key):
            new = np.concatenate([[True], key[1:] != key[:-1]])
            if not new.all():
                v = np.bincount(np.cumsum(new) - 1, weights=v)
                r, c = r[new], c[new]
        off = np.concatenate([[0], np.cumsum(np.bincount(r, minlength=int(num_rows)))])
        return cls(num_rows, num_cols, off, c, v)

    @classmethod
    def from_dense(cls, dense) -> "SparseMatrix":
        d = np.asarray(dense, dtype=np.float64)
        r, c = np.nonzero(d)
        return cls.from_coo(d.shape[0], d.shape[1], r, c, d[r, c])

    def __repr__(self):
        return f"SparseMatrix({self.num_rows}x{self.num_cols}, nnz={self.nnz})"


@dataclass
class LpProblem:
    """One LP instance (lp_model.py:153-200)."""

    matrix: SparseMatrix
    objective: np.ndarray
    var_lower: np.ndarray
    var_upper: np.ndarray
    con_lower: np.ndarray
    con_upper: np.ndarray
    objective_constant: float = 0.0
    maximize: bool = False
    name: str = ""
    row_names: list = field(default_factory=list, repr=False)
    col_names: list = field(default_factory=list, repr=False)

    def __post_init__(self):
        m, n = self.matrix.num_rows, self.matrix.num_cols
        for attr, size in (("objective", n), ("var_lower", n), ("var_upper", n),
                           ("con_lower", m), ("con_upper", m)):
            arr = np.ascontiguousarray(getattr(self, attr), dtype=np.float64)
            if arr.shape != (size,):
                raise ValueError(f"{attr} has length {arr.shape[0]}, expected {size}")
            setattr(self, attr, arr)
        bad = self.var_lower > self.var_upper
        if bad.any():
            raise ValueError(f"variable {int(np.argmax(bad))}: lower bound exceeds upper bound")
        bad = self.con_lower > self.con_upper
        if bad.any():
            raise ValueError(f"constraint {int(np.argmax(bad))}: lower bound exceeds upper bound")
        if not np.all(np.isfinite(self.objective)):
            raise ValueError("objective coefficients must be finite")

    @property
    def num_constraints(self) -> int:
        return self.matrix.num_rows

    @property
    def num_variables(self) -> int:
        return self.matrix.num_cols


def objective_value(problem, x) -> float:
    """c'x + constant, internal (minimisation) sense (lp_model.py:203-210)."""
    x = np.asarray(x, dtype=np.float64)
    if x.shape != (problem.matrix.num_cols,):
        raise ValueError(f"x has length {x.shape[0]}, expected {problem.matrix.num_cols}")
    return float(np.dot(problem.objective, x) + problem.objective_constant)


def reported_objective(problem, internal_value: float) -> float:
    """Objective in the declared sense (lp_model.py:213-215)."""
    return -internal_value if getattr(problem, "maximize", False) else internal_value
