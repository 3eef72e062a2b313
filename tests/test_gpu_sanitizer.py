"""compute-sanitizer over the hot path's kernels (tools/sanitizer_case.py):
memcheck (out-of-bounds / misaligned device accesses), racecheck (shared
memory hazards: the long-row kernel's product buffer and add chain, block
reductions), synccheck (barrier misuse). The cross-CTA protocols (heavy-row
arrival counters, chained products) run inside the checked workload. The
reference analogue is its lockstep checker (comm.py:87-91, :309-320)."""

import os
import shutil
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = Path(__file__).resolve().parents[1]
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")
@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_clean(tool):
    if not Path(SAN).exists():  # pragma: no cover
        pytest.skip("compute-sanitizer not installed")
    cmd = [SAN, "--tool", tool, "--error-exitcode", "99", "--print-limit", "20",
           "--kernel-name", "regex=sell32|heavy_chunk|long_row|rows_kernel|reduce_kernel|terms_reduce|step_advance|epoch_advance|persistent|cluster",
           sys.executable, str(ROOT / "tools" / "sanitizer_case.py")]
    env = dict(os.environ, PYTHONPATH=str(ROOT))
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, env=env)
    out = r.stdout + r.stderr
    if "compute-sanitizer is closed" in out:
        # this GPU pool disabled the tool; tests/test_gpu_bounds.py runs the
        # same workload on the bounds-checked build instead
        pytest.skip("compute-sanitizer is closed on this GPU pool")
    assert "SANITIZER_CASE_DONE" in out, out[-3000:]
    assert r.returncode == 0, out[-3000:]
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards" in out, out[-3000:]
