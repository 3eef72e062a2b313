"""Bounds-checked runs of the hot path (the stand-in for compute-sanitizer
memcheck, which this GPU pool has closed): the library is rebuilt with
-DGRIDLP_CHECKED (native.build(checked=True)) so every kernel verifies its
gather indices, SELL lane extents, long-row ranges and written rows and traps
on a violation, and the sanitizer workload (tools/sanitizer_case.py: every
kernel family, both grids, the persistent and cluster launches) runs on it
in a subprocess; results are compared with the product build. A corrupted
column index must trap, proving the checks are live. The reference analogue
is its lockstep checker (comm.py:87-91, :309-320)."""

import os
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = Path(__file__).resolve().parents[1]

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2601_07628_b200 import native  # noqa: E402


@pytest.fixture(scope="module")
def checked_lib():
    return native.build(checked=True)


def _run(code_or_script, lib, timeout=900):
    env = dict(os.environ, PYTHONPATH=str(ROOT))
    if lib is not None:
        env["GRIDLP_LIB"] = str(lib)
    args = [sys.executable, str(code_or_script)] if str(code_or_script).endswith(".py") else \
        [sys.executable, "-c", code_or_script]
    r = subprocess.run(args, capture_output=True, text=True, timeout=timeout, env=env, cwd=str(ROOT))
    return r.returncode, r.stdout + r.stderr


def test_workload_clean_under_bounds_checks(checked_lib):
    rc, out = _run(ROOT / "tools" / "sanitizer_case.py", checked_lib)
    assert rc == 0 and "SANITIZER_CASE_DONE" in out, out[-3000:]
    assert "GRIDLP_CHECK failed" not in out, out[-3000:]
    rc2, ref = _run(ROOT / "tools" / "sanitizer_case.py", None)
    assert rc2 == 0, ref[-3000:]
    # the checked build computes the same solves (checks never change a value)
    lines = lambda t: [ln for ln in t.splitlines() if ": " in ln and "it=" in ln]  # noqa: E731
    assert lines(out) == lines(ref) and lines(out)


CORRUPT = r"""
import numpy as np, torch
from paper_2601_07628_b200 import native
from paper_2601_07628_b200.blocks import DeviceCsr, HostCsr
from paper_2601_07628_b200.ops import CudaOps, Fused
assert native.load()._lib.gridlp_build_flags() == 1
dev = torch.device("cuda", 0)
m, n = 64, 100
ptr = np.arange(0, 3 * m + 1, 3)
col = np.tile(np.array([1, 5, 9]), m)
h = HostCsr(m, n, ptr, col, np.ones(3 * m))
A = DeviceCsr(h, dev)
A.dev["cols"][5] = n + 1000          # a gather past the end of x
ops = CudaOps(dev, 1024, 4)
out = torch.empty(m, dtype=torch.float64, device=dev)
ops.store(Fused(A, torch.ones(n, dtype=torch.float64, device=dev)), out)
torch.cuda.synchronize()
print("NO_TRAP")
"""


def test_corrupted_index_traps(checked_lib):
    rc, out = _run(CORRUPT, checked_lib, timeout=300)
    assert "GRIDLP_CHECK failed: SELL gather index" in out, out[-3000:]
    assert rc != 0 and "NO_TRAP" not in out
