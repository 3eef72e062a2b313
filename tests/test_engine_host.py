"""Engine HOST logic vs the reference's golden outputs, on CPU.

The engine (grid plans, ascending reductions, KKT/restart/PID decisions,
collective ledger, result assembly) is driven with the CPU test double of
the device ops (tests/host_ops.py), whose arithmetic mirrors the
reference's numpy expressions — so the whole solve must match the reference
BIT FOR BIT, counters included. The device kernels themselves are checked
in the gpu-marked tests."""

import math

import numpy as np
import pytest
import torch

from conftest import golden_problem, load_json, load_npz
from host_ops import host_factory
from paper_2601_07628_b200.api import SolverConfig, _solve

CPU = torch.device("cpu")


def host_solve(problem, **cfg):
    if cfg.get("grid") is not None:
        cfg["grid"] = tuple(cfg["grid"])
    return _solve(problem, SolverConfig(**cfg), ops_factory=host_factory, device=CPU)


def _same(a, b):
    return a == b or (isinstance(a, float) and isinstance(b, float) and math.isnan(a) and math.isnan(b))


def test_cfg1_bitwise(golden_cfg1):
    z = golden_cfg1
    r = host_solve(golden_problem(z), tolerance=1e-4, seed=0)
    assert (r.status, r.iterations, r.restarts) == ("optimal", int(z["iterations"]), int(z["restarts"]))
    np.testing.assert_array_equal(r.x, z["x"])
    np.testing.assert_array_equal(r.y, z["y"])
    assert r.objective == float(z["result_objective"])


@pytest.mark.parametrize("chunk", range(6))
def test_solve_cases_bitwise(golden_solves, chunk):
    z, meta = golden_solves
    cases = [m for m in meta if "result" in m]
    for m in cases[chunk::6]:
        exp = m["result"]
        r = host_solve(golden_problem(z, m["problem"] + "_"), **dict(m["cfg"]))
        t = m["id"]
        assert r.status == exp["status"], m["id"]
        assert r.iterations == exp["iterations"], m["id"]
        assert r.restarts == exp["restarts"], m["id"]
        if "time_limit_seconds" not in m["cfg"]:
            np.testing.assert_array_equal(r.x, z[f"S{t}_x"])
            np.testing.assert_array_equal(r.y, z[f"S{t}_y"])
            for k, v in exp["kkt"].items():
                assert _same(r.report.as_dict()[k], v), (m["id"], k)
            assert _same(r.objective, exp["objective"])
        assert r.counters == exp["counters"], m["id"]
        assert r.layout == exp["layout"], m["id"]
        assert r.to_json_dict().keys() == exp.keys()


def test_trace_matches_reference_trace(golden_cfg1):
    z = golden_cfg1

    class Keep(list):
        keep = set(int(t) for t in z["fx_trace_iters"])

    tr = Keep()
    from paper_2601_07628_b200.api import _solve as s
    s(golden_problem(z), SolverConfig(tolerance=1e-300, seed=0, eta=0.05, restarts=False,
                                      max_iterations=512),
      trace=tr, force_1x1=True, ops_factory=host_factory, device=CPU)
    assert [t for t, _, _ in tr] == [int(t) for t in z["fx_trace_iters"]]
    for k, (_, x, y) in enumerate(tr):
        np.testing.assert_array_equal(x, z["fx_trace_x"][k])
        np.testing.assert_array_equal(y, z["fx_trace_y"][k])
