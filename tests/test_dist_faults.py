"""Collective fault semantics of the multi-process executor (NcclGrid; gloo
on CPU, world size 2), mirroring the reference's threads backend:
a rank that stops issuing collectives surfaces as CollectiveTimeout after
collective_timeout_seconds (comm.py:49, :125-132), ranks on different
collective sequences raise CollectiveMismatch (the lockstep check,
comm.py:87-91, :309-320), and diverged replicated decisions raise
RuntimeError (solver_driver.py:242-244)."""

import os
import socket
import time

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, port, scenario, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=2)
    from paper_2601_07628_b200.comm import CollectiveMismatch, CollectiveTimeout, NcclGrid

    out = "ok"
    try:
        g = NcclGrid(1, 2, torch.device("cpu"), timeout=3.0)
        tab = g.table({g.coord: np.array([float(rank), 2.0])})
        assert tab[(0, 0)][0] == 0.0 and tab[(0, 1)][0] == 1.0
        if scenario == "timeout":
            if rank == 0:
                t0 = time.monotonic()
                try:
                    g.table({g.coord: np.array([1.0, 2.0])})
                    out = "no error"
                except CollectiveTimeout:
                    out = f"timeout after {time.monotonic() - t0:.1f}s"
            else:
                time.sleep(8.0)          # never joins the second table
        elif scenario == "mismatch":
            if rank == 1:
                g._seq += 3              # this rank skipped ahead in its collective sequence
            try:
                g.table({g.coord: np.array([1.0, 2.0])})
                out = "no error"
            except CollectiveMismatch as e:
                out = "mismatch " + str(e)[:40]
        elif scenario == "diverged":
            try:
                g.agree("optimal" if rank == 0 else "iteration_limit", "statuses")
                out = "no error"
            except RuntimeError as e:
                out = "diverged " + str(e)[:40]
    except Exception as e:  # pragma: no cover - reported to the parent
        out = f"error {type(e).__name__}: {e}"
    q.put((rank, out))
    if scenario != "timeout":
        dist.destroy_process_group()


def _run(scenario):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, scenario, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        if p.is_alive():  # pragma: no cover
            p.kill()
    return res


def test_timeout_raises_collective_timeout():
    os.environ.setdefault("PYTHONPATH", os.pathsep.join([os.getcwd()]))
    res = _run("timeout")
    assert res[0].startswith("timeout after"), res
    secs = float(res[0].split()[2].rstrip("s"))
    assert 2.0 <= secs <= 8.0, res


def test_sequence_mismatch_raises_collective_mismatch():
    res = _run("mismatch")
    assert res[0].startswith("mismatch") and res[1].startswith("mismatch"), res


def test_diverged_statuses_raise():
    res = _run("diverged")
    assert res[0].startswith("diverged") and res[1].startswith("diverged"), res
