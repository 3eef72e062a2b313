"""Shared test helpers: golden-fixture loading and the gpu marker."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = Path(__file__).resolve().parent / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


class _Mat:
    """Duck-typed reference SparseMatrix (lp_model.py:40-150)."""

    def __init__(self, m, n, ptr, col, val):
        self.num_rows, self.num_cols = int(m), int(n)
        self.row_offsets = np.asarray(ptr, dtype=np.int64)
        self.col_indices = np.asarray(col, dtype=np.int64)
        self.values = np.asarray(val, dtype=np.float64)

    @property
    def nnz(self):
        return len(self.values)

    @property
    def shape(self):
        return (self.num_rows, self.num_cols)


class _Prob:
    """Duck-typed reference LpProblem (lp_model.py:153-200)."""

    def __init__(self, **kw):
        self.__dict__.update(kw)

    @property
    def num_constraints(self):
        return self.matrix.num_rows

    @property
    def num_variables(self):
        return self.matrix.num_cols


def golden_problem(z, prefix=""):
    g = lambda k: z[prefix + k]  # noqa: E731
    return _Prob(
        matrix=_Mat(g("m"), g("n"), g("row_offsets"), g("col_indices"), g("values")),
        objective=np.asarray(g("objective"), np.float64),
        var_lower=np.asarray(g("var_lower"), np.float64),
        var_upper=np.asarray(g("var_upper"), np.float64),
        con_lower=np.asarray(g("con_lower"), np.float64),
        con_upper=np.asarray(g("con_upper"), np.float64),
        objective_constant=float(g("objective_constant")),
        maximize=bool(g("maximize")),
        name=prefix,
    )


_cache = {}


def load_npz(name):
    if name not in _cache:
        _cache[name] = np.load(GOLDEN / name)
    return _cache[name]


def load_json(name):
    if name not in _cache:
        _cache[name] = json.loads((GOLDEN / name).read_text())
    return _cache[name]


@pytest.fixture(scope="session")
def golden_solves():
    return load_npz("solves.npz"), load_json("solves.json")


@pytest.fixture(scope="session")
def golden_cfg1():
    return load_npz("cfg1.npz")
