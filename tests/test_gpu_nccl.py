"""The comm_backend="nccl" engine path on a real GPU.

The round's GPU boxes have one B200, so the NCCL grid runs as a world of one
rank: the per-pass scalar all_gather and the final x/y all_gather go through
NCCL on device tensors, and the engine takes its non-graph launch path
(eager kernels between collectives). The result must equal the virtual-grid
solve bit for bit — same kernels, same order. Grids with >1 rank per axis
are covered on CPU with gloo (tests/test_dist_gloo.py)."""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture
def nccl_world1():
    import torch.distributed as dist

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    torch.cuda.set_device(0)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        yield dist
    finally:
        dist.destroy_process_group()


def test_nccl_world1_matches_virtual_grid_bitwise(nccl_world1):
    from paper_2601_07628_b200 import GeneratorSpec, SolverConfig, generate, solve

    p = generate(GeneratorSpec(kind="uniform_random", num_rows=400, num_cols=700, nnz_target=5000,
                               inequality_fraction=0.3, seed=3))
    a = solve(p, SolverConfig(tolerance=1e-6, seed=3, comm_backend="nccl"))
    b = solve(p, SolverConfig(tolerance=1e-6, seed=3))
    assert a.status == b.status == "optimal"
    assert (a.iterations, a.restarts) == (b.iterations, b.restarts)
    np.testing.assert_array_equal(a.x, b.x)
    np.testing.assert_array_equal(a.y, b.y)
    assert a.report == b.report
    assert a.counters == b.counters


def test_nccl_graph_capture_option_matches(nccl_world1):
    """EngineOptions.graph_nccl captures the NCCL executor's iterations in a
    CUDA graph (collectives included); on a world of one it must reproduce
    the eager NCCL path bit for bit."""
    from paper_2601_07628_b200 import GeneratorSpec, SolverConfig, generate
    from paper_2601_07628_b200.api import _solve

    p = generate(GeneratorSpec(kind="uniform_random", num_rows=400, num_cols=700, nnz_target=5000,
                               inequality_fraction=0.3, seed=5))
    cfg = SolverConfig(tolerance=1e-6, seed=5, comm_backend="nccl")
    a = _solve(p, cfg, engine_overrides={"graph_nccl": True})
    b = _solve(p, cfg)
    assert (a.status, a.iterations, a.restarts) == (b.status, b.iterations, b.restarts)
    np.testing.assert_array_equal(a.x, b.x)
    np.testing.assert_array_equal(a.y, b.y)
