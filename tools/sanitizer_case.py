"""Small workload for compute-sanitizer (tests/test_gpu_sanitizer.py): every
kernel family of the hot path — SELL lanes (both variants), warp-per-row
long rows (shared-memory add chain), chunked heavy rows (the cross-CTA
arrival counter), fused KKT / probe reductions, chained products in a
captured graph, the 2x2 virtual grid's partial sums, power iteration, the
persistent cooperative launch and the thread-block-cluster launch (DSMEM
broadcasts, cluster barriers)."""

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2601_07628_b200 import LpProblem, SolverConfig, SparseMatrix, native, solve  # noqa: E402


def problem(seed=0, m=700, n=900):
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, 30, m)
    lens[[3, 100]] = [300, 2000]          # long exact rows (warp per row)
    lens[5] = 5000 if n > 5000 else n     # heavy (chunked) when n allows
    ptr = np.concatenate([[0], np.cumsum(lens)])
    col = np.concatenate([np.sort(rng.choice(n, k, replace=False)) for k in lens]).astype(np.int64)
    val = rng.standard_normal(len(col))
    x_hat = rng.uniform(1.0, 3.0, n)
    A = SparseMatrix(m, n, ptr, col, val)
    ax = np.array([val[ptr[i]:ptr[i + 1]] @ x_hat[col[ptr[i]:ptr[i + 1]]] for i in range(m)])
    return LpProblem(A, rng.standard_normal(n), np.zeros(n), np.full(n, 4.0), ax - 0.5, ax + 0.5)


def main():
    p = problem(0, 700, 6000)
    lib = native.load()
    for variant in (0, 1):
        lib.set_tuning("sell_variant", variant)
        for grid in ((1, 1), (2, 2)):
            r = solve(p, SolverConfig(tolerance=1e-6, max_iterations=192, seed=1, n_procs=grid[0] * grid[1],
                                      grid=grid))
            print(f"variant {variant} grid {grid}: {r.status} it={r.iterations} obj={r.objective:.10g}")
    from paper_2601_07628_b200.api import _solve

    r = _solve(p, SolverConfig(tolerance=1e-6, max_iterations=192, seed=1),
               engine_overrides={"persistent_max_nnz": 1 << 30})      # the persistent cooperative launch
    print(f"persistent: {r.status} it={r.iterations} obj={r.objective:.10g}")
    from paper_2601_07628_b200 import GeneratorSpec, generate

    q = generate(GeneratorSpec(kind="uniform_random", num_rows=600, num_cols=1000, nnz_target=6000,
                               inequality_fraction=0.3, seed=2))
    r = solve(q, SolverConfig(tolerance=1e-6, max_iterations=192, seed=2))   # all rows light: cluster launch
    print(f"cluster: {r.status} it={r.iterations} obj={r.objective:.10g}")
    r = _solve(q, SolverConfig(tolerance=1e-6, max_iterations=192, seed=2),
               engine_overrides={"device_loop": True})          # the device-side loop (WHILE graph)
    print(f"device loop: {r.status} it={r.iterations} obj={r.objective:.10g}")
    print("SANITIZER_CASE_DONE")


if __name__ == "__main__":
    main()
