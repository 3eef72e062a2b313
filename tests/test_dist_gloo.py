"""Multi-process grid (comm_backend="nccl" code path) on CPU with gloo.

One process per grid block, exactly as on GPUs under torchrun: NcclGrid
builds the per-column (R axis) and per-row (C axis) groups, reduces block
partials with allreduce, all-gathers the pass scalars and assembles x / y
from devices (0, j) / (i, 0). The device ops are the CPU test double
(tests/host_ops.py). With two ranks per reduction group an allreduce is a
single IEEE addition, so the result must equal the reference's simulated
grid BIT FOR BIT (golden fixtures), counters included."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import golden_problem, load_json, load_npz


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case_ids, out_q):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        from host_ops import host_factory
        from paper_2601_07628_b200.api import SolverConfig, _solve

        z = load_npz("solves.npz")
        meta = {m["id"]: m for m in load_json("solves.json")}
        for cid in case_ids:
            m = meta[cid]
            cfg = dict(m["cfg"])
            cfg["grid"] = tuple(cfg["grid"])
            r = _solve(golden_problem(z, m["problem"] + "_"), SolverConfig(**cfg, comm_backend="nccl"),
                       ops_factory=host_factory, device=torch.device("cpu"))
            out_q.put((rank, cid, r.status, r.iterations, r.restarts, r.x, r.y, r.counters,
                       r.report.as_dict()))
    finally:
        dist.destroy_process_group()


def _run(world, case_ids):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case_ids, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world * len(case_ids))]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def _cases(grid, limit):
    meta = load_json("solves.json")
    return [m["id"] for m in meta if "result" in m and m["cfg"].get("grid") == list(grid)][:limit]


@pytest.mark.parametrize("grid,limit", [((1, 2), 3), ((2, 1), 3), ((2, 2), 3)])
def test_grid_over_processes_matches_reference_bitwise(grid, limit):
    import sys
    from pathlib import Path

    here = str(Path(__file__).resolve().parent)
    if here not in sys.path:
        sys.path.insert(0, here)
    os.environ["PYTHONPATH"] = os.pathsep.join([here, str(Path(here).parent), os.environ.get("PYTHONPATH", "")])
    ids = _cases(grid, limit)
    assert ids
    z = load_npz("solves.npz")
    meta = {m["id"]: m for m in load_json("solves.json")}
    for rank, cid, status, iters, restarts, x, y, counters, kkt in _run(grid[0] * grid[1], ids):
        exp = meta[cid]["result"]
        assert (status, iters, restarts) == (exp["status"], exp["iterations"], exp["restarts"]), (rank, cid)
        np.testing.assert_array_equal(x, z[f"S{cid}_x"])
        np.testing.assert_array_equal(y, z[f"S{cid}_y"])
        assert counters == exp["counters"]
        assert kkt == exp["kkt"]


def _worker_grid3(rank, world, port, grid, out_q):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        from host_ops import host_factory
        from paper_2601_07628_b200 import GeneratorSpec, generate
        from paper_2601_07628_b200.api import SolverConfig, _solve

        p = generate(GeneratorSpec(kind="uniform_random", num_rows=37, num_cols=53, nnz_target=400,
                                   inequality_fraction=0.3, seed=3))
        r = _solve(p, SolverConfig(tolerance=1e-7, seed=3, n_procs=world, grid=grid, comm_backend="nccl"),
                   ops_factory=host_factory, device=torch.device("cpu"))
        out_q.put((rank, r.status, r.iterations, r.restarts, r.x, r.y))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("grid", [(1, 3), (3, 1)])
def test_three_member_axis_sums_match_the_oracle_bitwise(grid):
    """Axis groups of 3 (lengths not divisible by 3: the sharded exchange pads
    to 3·ceil(len/3)): the multi-process grid equals the CPU oracle's
    lockstep grid (ascending-order sums, oracle/pdhg_oracle.py) bit for bit."""
    import sys
    from pathlib import Path

    from oracle import pdhg_oracle
    from paper_2601_07628_b200 import GeneratorSpec, generate

    here = str(Path(__file__).resolve().parent)
    if here not in sys.path:
        sys.path.insert(0, here)
    os.environ["PYTHONPATH"] = os.pathsep.join([here, str(Path(here).parent), os.environ.get("PYTHONPATH", "")])
    p = generate(GeneratorSpec(kind="uniform_random", num_rows=37, num_cols=53, nnz_target=400,
                               inequality_fraction=0.3, seed=3))
    want = pdhg_oracle.oracle_solve(p, tolerance=1e-7, seed=3, n_procs=3, grid=grid)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_grid3, args=(r, 3, port, grid, q)) for r in range(3)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=600) for _ in range(3)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, status, iters, restarts, x, y in res:
        assert (status, iters, restarts) == (want.status, want.iterations, want.restarts), rank
        np.testing.assert_array_equal(x, want.x)
        np.testing.assert_array_equal(y, want.y)
