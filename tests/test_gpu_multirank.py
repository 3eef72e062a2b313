"""The multi-rank executor (comm_backend="nccl": one grid block per process)
with the REAL device path, on the round's single GPU.

NCCL refuses two ranks on one GPU, but torch.distributed's gloo backend runs
all_reduce / all_gather on CUDA tensors, so four processes sharing cuda:0
exercise everything the 8-GPU run does except NCCL itself: per-rank blocks
built on the device, partial products and the fused epilogues from the
sm_100a library, axis collectives on device vectors, the once-per-pass
scalar table and the final x / y gather. Every axis sum runs in ascending
member order (the sharded exchange in the main loop, ordered all-gather sums
elsewhere), so every grid shape reproduces the single-process virtual grid
bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASE = dict(kind="uniform_random", num_rows=700, num_cols=1100, nnz_target=9000, inequality_fraction=0.3, seed=6)
# peer exchanges between processes that share ONE GPU wait for the driver's
# time slicing at every exchange, so those cases run a bounded iteration count
PEER_CASE = dict(kind="uniform_random", num_rows=300, num_cols=400, nnz_target=3000, inequality_fraction=0.3, seed=6)
PEER_CFG = dict(tolerance=1e-12, seed=6, max_iterations=192)


def _worker(rank, world, port, grid, backend, q):
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        from paper_2601_07628_b200 import GeneratorSpec, SolverConfig, generate, solve

        if backend == "peer":
            p, cfg = generate(GeneratorSpec(**PEER_CASE)), dict(PEER_CFG)
        else:
            p, cfg = generate(GeneratorSpec(**CASE)), dict(tolerance=1e-5, seed=6)
        r = solve(p, SolverConfig(**cfg, n_procs=world, grid=grid, comm_backend=backend))
        q.put((rank, r.status, r.iterations, r.restarts, r.x, r.y, r.report.as_dict(), r.counters, r.layout))
        dist.barrier()          # members keep their IPC-shared buffers alive until everyone is done
    finally:
        dist.destroy_process_group()


def _run(grid, backend="nccl"):
    import torch.multiprocessing as mp

    world = grid[0] * grid[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, grid, backend, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return sorted(out, key=lambda t: t[0])


# every axis sum is in ascending member order (sharded exchange in the main
# loop, ordered all-gather sums elsewhere): bitwise for every grid shape
@pytest.mark.parametrize("grid,bitwise", [((2, 2), True), ((1, 4), True), ((3, 1), True)])
def test_multirank_device_path_matches_virtual_grid(grid, bitwise):
    from paper_2601_07628_b200 import GeneratorSpec, SolverConfig, generate, solve

    os.environ.setdefault("OMP_NUM_THREADS", "1")
    p = generate(GeneratorSpec(**CASE))
    want = solve(p, SolverConfig(tolerance=1e-5, seed=6, n_procs=grid[0] * grid[1], grid=grid))
    res = _run(grid)
    for rank, status, iters, restarts, x, y, kkt, counters, layout in res:
        assert (status, iters, restarts) == (want.status, want.iterations, want.restarts), rank
        assert layout == want.layout
        if bitwise:
            np.testing.assert_array_equal(x, want.x)
            np.testing.assert_array_equal(y, want.y)
            assert kkt == want.report.as_dict()
            assert counters == want.counters
        else:
            np.testing.assert_allclose(x, want.x, rtol=1e-9, atol=1e-9)
            np.testing.assert_allclose(y, want.y, rtol=1e-9, atol=1e-9)
        # every rank returns the same solution (replicated, never broadcast)
        np.testing.assert_array_equal(x, res[0][4])
        np.testing.assert_array_equal(y, res[0][5])


@pytest.mark.parametrize("grid", [(2, 2), (1, 4), (3, 1), (2, 3)])
def test_peer_exchange_is_bitwise_the_virtual_grid(grid):
    """comm_backend="peer": products write their partial rows into the group
    members' receive buffers (CUDA IPC, here between processes sharing the
    GPU; NVLink P2P across GPUs) and the epilogue adds the slots in ascending
    order after a device-side arrival counter — so unlike a ring allreduce
    the result is the virtual grid's (= the reference's) bit for bit for
    every group size; iterations run inside CUDA graphs."""
    from paper_2601_07628_b200 import GeneratorSpec, SolverConfig, generate, solve

    p = generate(GeneratorSpec(**PEER_CASE))
    want = solve(p, SolverConfig(**PEER_CFG, n_procs=grid[0] * grid[1], grid=grid))
    for rank, status, iters, restarts, x, y, kkt, counters, layout in _run(grid, "peer"):
        assert (status, iters, restarts) == (want.status, want.iterations, want.restarts), rank
        np.testing.assert_array_equal(x, want.x)
        np.testing.assert_array_equal(y, want.y)
        assert kkt == want.report.as_dict()
        assert counters == want.counters


def _band_worker(rank, world, port, grid, q):
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        from paper_2601_07628_b200 import SolverConfig, solve
        from paper_2601_07628_b200.synth import BandProblem, PlantedBands, PlantedSpec

        spec = PlantedSpec(1500, 2000, 6, seed=13)
        prob = BandProblem(PlantedBands(spec, torch.device("cuda", 0), chunk_draws=6 * 400))
        r = solve(prob, SolverConfig(tolerance=1e-6, seed=13, n_procs=world, grid=grid, permutation="none",
                                     partitioning="uniform", comm_backend="nccl", max_iterations=200_000))
        q.put((rank, r.status, r.iterations, r.objective, r.layout["total_nnz"]))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_band_problem_sharded_over_processes_reaches_planted_optimum():
    """The oversized-LP path end to end over 4 processes: each rank generates
    only its own grid block and band vectors on the device (no global matrix
    anywhere), the grid solves over the multi-rank executor, and every rank
    reports the analytic optimum c·x*."""
    import torch.multiprocessing as mp

    from paper_2601_07628_b200.synth import PlantedSpec, generate_planted

    star = generate_planted(PlantedSpec(1500, 2000, 6, seed=13), torch.device("cuda", 0)).optimal_objective()
    grid, world = (2, 2), 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_band_worker, args=(r, world, port, grid, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert len({(s, it, obj) for _, s, it, obj, _ in out}) == 1      # replicated decisions
    _, status, _, obj, nnz = out[0]
    assert status == "optimal" and nnz > 0
    assert abs(obj - star) <= 1e-4 * (1.0 + abs(star))
