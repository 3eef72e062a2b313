"""Debug probe: peer exchange between processes sharing one GPU."""
import os, socket, sys, time
import numpy as np
import torch
import torch.multiprocessing as mp

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def worker(rank, world, port, grid, iters):
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    from paper_2601_07628_b200 import GeneratorSpec, SolverConfig, generate, solve
    p = generate(GeneratorSpec(kind="uniform_random", num_rows=300, num_cols=400, nnz_target=3000,
                               inequality_fraction=0.3, seed=6))
    base = dict(tolerance=1e-12, seed=6, n_procs=world, grid=grid, max_iterations=iters)
    t0 = time.time()
    r = solve(p, SolverConfig(**base, comm_backend="peer"))
    t1 = time.time()
    want = solve(p, SolverConfig(**base)) if rank == 0 else None
    if rank == 0:
        print("peer", r.status, r.iterations, f"{t1 - t0:.1f}s", "bitwise x", np.array_equal(r.x, want.x),
              "y", np.array_equal(r.y, want.y), "kkt", r.report == want.report, flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    grid = tuple(int(v) for v in sys.argv[1].split("x"))
    iters = int(sys.argv[2])
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    mp.spawn(worker, args=(grid[0] * grid[1], port, grid, iters), nprocs=grid[0] * grid[1])
