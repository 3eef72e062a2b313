"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
package itself (`/root/reference/pkg/src/gridlp`, read-only, pure Python).

Run here (the reference does not exist on the GPU box):

    python tests/golden/make_golden.py            # small fixtures (seconds)
    python tests/golden/make_golden.py --cfg2     # + cfg2 summary (~15 min)

`import gridlp` needs two import-only stubs in this image: `greenlet`
(comm.py:30; only used by the cooperative multi-device executor, which we
never select — grids run with comm_backend="threads", bit-identical per
test_solver_driver.py:104-111) and `matplotlib` (figures.py:6-10, only
plotting). The stubs are installed into sys.modules by this script only.
"""

from __future__ import annotations

import argparse
import json
import logging
import sys
import types
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SRC = Path("/root/reference/pkg/src")


def _install_stubs():
    gl = types.ModuleType("greenlet")

    class _G:  # pragma: no cover - never executed
        def __init__(self, *a, **k):
            raise RuntimeError("greenlet stub: cooperative backend unavailable")

    gl.greenlet = _G
    gl.getcurrent = lambda: None
    sys.modules.setdefault("greenlet", gl)
    mpl = types.ModuleType("matplotlib")
    mpl.use = lambda *a, **k: None
    plt = types.ModuleType("matplotlib.pyplot")
    mpl.pyplot = plt
    sys.modules.setdefault("matplotlib", mpl)
    sys.modules.setdefault("matplotlib.pyplot", plt)
    sys.path.insert(0, str(REF_SRC))


_install_stubs()
import gridlp  # noqa: E402
from gridlp import (  # noqa: E402
    GeneratorSpec, GridTopology, LpProblem, SolverConfig, SparseMatrix,
    build_layout, generate, layout_summary, reference_solve, select_grid, solve,
)
from gridlp.sparse_kernels import spmv, transpose, estimate_spectral_norm_dense  # noqa: E402
from gridlp.partition import distribute  # noqa: E402

INF = float("inf")


def problem_arrays(p, prefix=""):
    A = p.matrix
    return {
        prefix + "m": np.int64(A.num_rows), prefix + "n": np.int64(A.num_cols),
        prefix + "row_offsets": A.row_offsets, prefix + "col_indices": A.col_indices,
        prefix + "values": A.values, prefix + "objective": p.objective,
        prefix + "var_lower": p.var_lower, prefix + "var_upper": p.var_upper,
        prefix + "con_lower": p.con_lower, prefix + "con_upper": p.con_upper,
        prefix + "objective_constant": np.float64(p.objective_constant),
        prefix + "maximize": np.bool_(p.maximize),
    }


def random_lp(seed, m=14, n=18, nnz=140, inequality_fraction=0.4):
    return generate(GeneratorSpec(kind="uniform_random", num_rows=m, num_cols=n,
                                  nnz_target=nnz, inequality_fraction=inequality_fraction,
                                  seed=seed))


class PassLog(logging.Handler):
    """Captures the raw arguments of the per-pass INFO line
    (solver_driver.py:184-190)."""

    def __init__(self):
        super().__init__(logging.INFO)
        self.rows = []

    def emit(self, record):
        it, rep, ss, epoch = None, None, None, None
        a = record.args
        # (iter, r_p, r_d, r_gap, obj_p, obj_d, omega, eta, epoch)
        self.rows.append([float(v) for v in a])


def solve_logged(problem, cfg):
    lg = logging.getLogger("gridlp.solver")
    h = PassLog()
    lg.addHandler(h)
    lg.setLevel(logging.INFO)
    try:
        res = solve(problem, cfg)
    finally:
        lg.removeHandler(h)
    return res, np.asarray(h.rows, dtype=np.float64).reshape(-1, 9)


class Checkpoints(list):
    """trace sink that keeps only selected iterations (solver_driver.py:387-388)."""

    def __init__(self, keep):
        super().__init__()
        self.keep = set(keep)

    def append(self, item):
        if item[0] in self.keep:
            super().append(item)


def result_dict(r):
    d = r.to_json_dict()
    return d


# ---------------------------------------------------------------------------

def gen_spmv():
    out = {}
    rng = np.random.default_rng(7)
    cases = [(40, 30, 500), (300, 200, 6000), (1, 5, 5), (5, 1, 3), (64, 64, 0)]
    for t, (m, n, nnz) in enumerate(cases):
        A = SparseMatrix.from_coo(
            m, n, rng.integers(0, m, nnz), rng.integers(0, n, nnz),
            rng.standard_normal(nnz) * 10.0 ** rng.integers(-8, 8, nnz),
        )
        x = rng.standard_normal(n) * 10.0 ** rng.integers(-3, 3, n)
        y = rng.standard_normal(m)
        At = transpose(A)
        out.update({f"c{t}_m": np.int64(m), f"c{t}_n": np.int64(n),
                    f"c{t}_ptr": A.row_offsets, f"c{t}_col": A.col_indices,
                    f"c{t}_val": A.values, f"c{t}_x": x, f"c{t}_y": y,
                    f"c{t}_ax": spmv(A, x), f"c{t}_aty": spmv(At, y),
                    f"c{t}_tptr": At.row_offsets, f"c{t}_tcol": At.col_indices,
                    f"c{t}_tval": At.values})
    out["ncases"] = np.int64(len(cases))
    np.savez_compressed(HERE / "spmv.npz", **out)


def gen_layouts():
    out = {}
    meta = []
    probs = {
        "u300": random_lp(3, m=300, n=500, nnz=4000),
        "u1000": random_lp(4, m=1000, n=700, nnz=9000),
        "tall": random_lp(5, m=900, n=90, nnz=3000),
    }
    for name, p in probs.items():
        out.update(problem_arrays(p, prefix=f"{name}_"))
    t = 0
    for name, p in probs.items():
        for grid in [(1, 1), (1, 2), (2, 1), (2, 2), (2, 4), (4, 2), None]:
            for perm in ("none", "full_random", "block_random"):
                for part in ("uniform", "nnz"):
                    for bs in (64, 7):
                        if perm != "block_random" and bs != 64:
                            continue
                        procs = 8 if grid is None else grid[0] * grid[1]
                        lay = build_layout(p, n_procs=procs, block_size=bs, seed=t % 5,
                                           permutation=perm, partitioning=part,
                                           grid=None if grid is None else GridTopology(*grid))
                        out[f"L{t}_row_perm"] = lay.perm.row_perm
                        out[f"L{t}_col_perm"] = lay.perm.col_perm
                        out[f"L{t}_row_cuts"] = lay.row_cuts
                        out[f"L{t}_col_cuts"] = lay.col_cuts
                        meta.append({"id": t, "problem": name, "grid": grid, "procs": procs,
                                     "permutation": perm, "partitioning": part,
                                     "block_size": bs, "seed": t % 5,
                                     "topology": [lay.topology.rows, lay.topology.cols],
                                     "summary": layout_summary(p, lay)})
                        t += 1
    # select_grid known answers over a sweep
    sg = []
    for m in (1, 2, 7, 100, 1000, 1500000):
        for n in (1, 3, 50, 1000, 126000000):
            for procs in (1, 2, 3, 4, 6, 8):
                g = select_grid(m, n, procs)
                sg.append([m, n, procs, g.rows, g.cols])
    out["select_grid"] = np.asarray(sg, dtype=np.int64)
    # permuted + distributed blocks for one case (block CSR pins)
    p = probs["u300"]
    lay = build_layout(p, n_procs=4, grid=GridTopology(2, 2), seed=1)
    blocks = distribute(p, lay)
    for (i, j), b in blocks.items():
        out[f"B{i}{j}_ptr"] = b.matrix.row_offsets
        out[f"B{i}{j}_col"] = b.matrix.col_indices
        out[f"B{i}{j}_val"] = b.matrix.values
        out[f"B{i}{j}_tptr"] = b.matrix_transpose.row_offsets
        out[f"B{i}{j}_tcol"] = b.matrix_transpose.col_indices
        out[f"B{i}{j}_tval"] = b.matrix_transpose.values
    out["B_row_perm"] = lay.perm.row_perm
    out["B_col_perm"] = lay.perm.col_perm
    out["B_row_cuts"] = lay.row_cuts
    out["B_col_cuts"] = lay.col_cuts
    np.savez_compressed(HERE / "layouts.npz", **out)
    (HERE / "layouts.json").write_text(json.dumps(meta, indent=0, sort_keys=True))


def gen_cfg1():
    spec = GeneratorSpec(kind="uniform_random", num_rows=2000, num_cols=4000,
                         nnz_target=20000, inequality_fraction=0.3, seed=0)
    p = generate(spec)
    keep = [1, 2, 3, 64, 65, 128, 640, 1024, 4096, 8192]
    tr = Checkpoints(keep)
    cfg = SolverConfig(tolerance=1e-4, seed=0)
    ref = reference_solve(p, cfg, trace=tr)
    res, log = solve_logged(p, cfg)
    assert np.array_equal(res.x, ref.x) and res.iterations == ref.iterations
    lay = build_layout(p, n_procs=1, grid=GridTopology(1, 1), seed=0)
    blk = distribute(p, lay)[(0, 0)]
    from gridlp.solver_driver import _norm_probe_vector
    est = estimate_spectral_norm_dense(blk.matrix, 30, _norm_probe_vector(4000, 0))
    out = problem_arrays(p)
    out.update({
        "x": ref.x, "y": ref.y, "iterations": np.int64(ref.iterations),
        "restarts": np.int64(ref.restarts), "result_objective": np.float64(ref.objective),
        "kkt": np.array([ref.report.r_primal, ref.report.r_dual, ref.report.r_gap,
                         ref.report.obj_primal, ref.report.obj_dual]),
        "estimate": np.float64(est), "passlog": log,
        "trace_iters": np.array([t[0] for t in tr], dtype=np.int64),
        "trace_x": np.stack([t[1] for t in tr]), "trace_y": np.stack([t[2] for t in tr]),
        "row_perm": lay.perm.row_perm, "col_perm": lay.perm.col_perm,
    })
    # fixed-eta, restart-free trajectory (bitwise target for the device path)
    tr2 = Checkpoints([1, 2, 7, 64, 300, 512])
    cfg2 = SolverConfig(tolerance=1e-300, seed=0, eta=0.05, restarts=False, max_iterations=512)
    ref2 = reference_solve(p, cfg2, trace=tr2)
    out.update({"fx_trace_iters": np.array([t[0] for t in tr2], dtype=np.int64),
                "fx_trace_x": np.stack([t[1] for t in tr2]),
                "fx_trace_y": np.stack([t[2] for t in tr2]),
                "fx_x": ref2.x, "fx_y": ref2.y,
                "fx_kkt": np.array([ref2.report.r_primal, ref2.report.r_dual, ref2.report.r_gap,
                                    ref2.report.obj_primal, ref2.report.obj_dual])})
    np.savez_compressed(HERE / "cfg1.npz", **out)


def kat_problems():
    """Known-answer problems from the reference tests."""
    P = {}
    P["lower_bounded"] = LpProblem(matrix=SparseMatrix.from_coo(1, 1, [0], [0], [1.0]),
                                   objective=np.array([1.0]), var_lower=np.array([0.0]),
                                   var_upper=np.array([10.0]), con_lower=np.array([1.0]),
                                   con_upper=np.array([INF]))
    P["packing"] = LpProblem(matrix=SparseMatrix.from_coo(1, 2, [0, 0], [0, 1], [1.0, 1.0]),
                             objective=np.array([-1.0, -1.0]), var_lower=np.zeros(2),
                             var_upper=np.ones(2), con_lower=np.array([-INF]),
                             con_upper=np.array([1.0]))
    P["zero_obj_box"] = LpProblem(matrix=SparseMatrix.from_coo(1, 2, [0, 0], [0, 1], [1.0, 1.0]),
                                  objective=np.zeros(2), var_lower=np.array([-1.0, -1.0]),
                                  var_upper=np.array([1.0, 1.0]), con_lower=np.array([-2.0]),
                                  con_upper=np.array([2.0]))
    # max sense: max 2x + y s.t. x + y <= 4, x <= 2 (box) -> 6 (test_solver_driver.py:159-175)
    P["max_sense"] = LpProblem(matrix=SparseMatrix.from_coo(1, 2, [0, 0], [0, 1], [1.0, 1.0]),
                               objective=-np.array([2.0, 1.0]), var_lower=np.zeros(2),
                               var_upper=np.array([2.0, 10.0]), con_lower=np.array([-INF]),
                               con_upper=np.array([4.0]), maximize=True)
    P["box_only"] = generate(GeneratorSpec(kind="box_lp_known_optimum", num_cols=9, seed=3))
    P["free_rows"] = LpProblem(matrix=SparseMatrix.from_coo(2, 2, [0, 1], [0, 1], [1.0, 2.0]),
                               objective=np.array([1.0, -1.0]), var_lower=np.array([-1.0, -1.0]),
                               var_upper=np.array([1.0, 1.0]), con_lower=np.array([-INF, -INF]),
                               con_upper=np.array([INF, INF]))
    P["block_diag"] = generate(GeneratorSpec(kind="block_diagonal", num_blocks=4, block_rows=6,
                                             block_cols=8, inequality_fraction=0.5, seed=2))
    P["staircase"] = generate(GeneratorSpec(kind="staircase", num_blocks=3, block_rows=5,
                                            block_cols=7, overlap=2, inequality_fraction=0.3,
                                            seed=4))
    P["empty_cols"] = LpProblem(matrix=SparseMatrix.from_coo(2, 4, [0, 1], [0, 2], [1.0, -1.0]),
                                objective=np.array([1.0, 0.0, -1.0, 2.0]),
                                var_lower=np.array([0.0, -1.0, 0.0, 0.0]),
                                var_upper=np.array([1.0, 1.0, 3.0, 5.0]),
                                con_lower=np.array([0.5, -2.0]), con_upper=np.array([0.5, -1.0]))
    # unbounded-ish: infinite var bounds -> can blow up -> numerical_failure or limit
    P["inf_var_bounds"] = LpProblem(matrix=SparseMatrix.from_coo(1, 2, [0, 0], [0, 1], [1.0, -1.0]),
                                    objective=np.array([-1.0, -1.0]),
                                    var_lower=np.array([0.0, 0.0]), var_upper=np.array([INF, INF]),
                                    con_lower=np.array([0.0]), con_upper=np.array([0.0]))
    return P


def gen_solves():
    out = {}
    meta = []
    t = 0
    # reference solve-level cases (small random LPs on the four grids)
    for seed in range(20):
        p = random_lp(seed, m=14, n=18, nnz=140)
        out.update(problem_arrays(p, prefix=f"P{seed}_"))
        for grid in [(1, 1), (1, 2), (2, 1), (2, 2)]:
            cfg = SolverConfig(tolerance=1e-8, n_procs=grid[0] * grid[1], grid=grid, seed=seed,
                               max_iterations=300_000, comm_backend="threads")
            r, log = solve_logged(p, cfg)
            out[f"S{t}_x"] = r.x
            out[f"S{t}_y"] = r.y
            out[f"S{t}_log"] = log
            meta.append({"id": t, "problem": f"P{seed}", "cfg": {"tolerance": 1e-8,
                         "n_procs": grid[0] * grid[1], "grid": list(grid), "seed": seed,
                         "max_iterations": 300_000}, "result": result_dict(r)})
            t += 1
    # ledger case (test_acceptance.py:106-138)
    p = random_lp(17, m=24, n=32, nnz=300)
    out.update(problem_arrays(p, prefix="P17L_"))
    lcfg = dict(tolerance=1e-300, max_iterations=640, kkt_interval=64, beta_sufficient=0.0,
                beta_necessary=0.0, beta_artificial=1e12, n_procs=4, grid=[2, 2], seed=17)
    r, log = solve_logged(p, SolverConfig(**{**lcfg, "grid": (2, 2)}, comm_backend="threads"))
    out[f"S{t}_x"], out[f"S{t}_y"], out[f"S{t}_log"] = r.x, r.y, log
    meta.append({"id": t, "problem": "P17L", "cfg": lcfg, "result": result_dict(r)})
    t += 1
    # known-answer problems, several configs
    for name, p in kat_problems().items():
        out.update(problem_arrays(p, prefix=f"{name}_"))
        for cfgd in ({"tolerance": 1e-6}, {"tolerance": 1e-9},
                     {"tolerance": 1e-6, "n_procs": 2},
                     {"tolerance": 1e-6, "max_iterations": 100},
                     {"tolerance": 1e-6, "max_iterations": 0},
                     {"tolerance": 1e-6, "halpern": False, "restarts": False},
                     {"tolerance": 1e-6, "gamma": 0.5, "kkt_interval": 16,
                      "max_iterations": 3000}):
            if name == "inf_var_bounds":
                cfgd = {**cfgd, "max_iterations": min(cfgd.get("max_iterations", 3000), 3000)}
            try:
                r, log = solve_logged(p, SolverConfig(**cfgd, comm_backend="threads"))
            except Exception as exc:  # record failures too
                meta.append({"id": t, "problem": name, "cfg": cfgd, "error": repr(exc)})
                t += 1
                continue
            out[f"S{t}_x"], out[f"S{t}_y"], out[f"S{t}_log"] = r.x, r.y, log
            meta.append({"id": t, "problem": name, "cfg": cfgd, "result": result_dict(r)})
            t += 1
    # failure / limit statuses (test_solver_driver.py:178-236)
    special = {
        "diverge": (LpProblem(matrix=SparseMatrix.from_coo(1, 1, [0], [0], [1.0]),
                              objective=np.array([0.0]), var_lower=np.array([-INF]),
                              var_upper=np.array([INF]), con_lower=np.array([1.0]),
                              con_upper=np.array([1.0])),
                    [{"tolerance": 1e-8, "eta": 10.0, "max_iterations": 5000, "kkt_interval": 64},
                     {"tolerance": 1e-8, "eta": 10.0, "max_iterations": 5000, "kkt_interval": 64,
                      "n_procs": 2}]),
        "varfree": (LpProblem(matrix=SparseMatrix.from_coo(2, 0, [], [], []),
                              objective=np.empty(0), var_lower=np.empty(0), var_upper=np.empty(0),
                              con_lower=np.array([-1.0, -INF]), con_upper=np.array([1.0, 5.0])),
                    [{"tolerance": 1e-9}, {"tolerance": 1e-9, "n_procs": 2}]),
        "Q10": (random_lp(10, m=12, n=16, nnz=90),
                [{"tolerance": 1e-12, "max_iterations": 96}]),
        "Q11": (random_lp(11, m=12, n=16, nnz=90),
                [{"tolerance": 1e-14, "time_limit_seconds": 0.0, "kkt_interval": 8,
                  "max_iterations": 10**9}]),
        "Q12": (random_lp(12, m=8, n=10, nnz=40), [{"tolerance": 1e-6, "n_procs": 2}]),
        "Q13": (random_lp(13, m=9, n=11, nnz=50), [{"tolerance": 1e-8, "n_procs": 4, "seed": 3}]),
        "Q14": (random_lp(14, m=8, n=10, nnz=40),
                [{"tolerance": 1e-300, "max_iterations": 128, "kkt_interval": 64}]),
        "box12": (generate(GeneratorSpec(kind="box_lp_known_optimum", num_cols=12, seed=4)),
                  [{"tolerance": 1e-9, "n_procs": 4}]),
        "Q5": (random_lp(5, m=10, n=14, nnz=70), [{"tolerance": 1e-7, "n_procs": 4, "seed": 2}]),
        "Q2F": (random_lp(2, m=14, n=18, nnz=140),
                [{"tolerance": 1e-8, "eta": 1e3, "max_iterations": 2000, "restarts": False},
                 {"tolerance": 1e-8, "n_procs": 8, "permutation": "full_random",
                  "partitioning": "uniform"},
                 {"tolerance": 1e-8, "n_procs": 3, "permutation": "none", "block_size": 3}]),
    }
    for name, (p, cfgs) in special.items():
        out.update(problem_arrays(p, prefix=f"{name}_"))
        for cfgd in cfgs:
            r, log = solve_logged(p, SolverConfig(**cfgd, comm_backend="threads"))
            out[f"S{t}_x"], out[f"S{t}_y"], out[f"S{t}_log"] = r.x, r.y, log
            meta.append({"id": t, "problem": name, "cfg": cfgd, "result": result_dict(r)})
            t += 1
    np.savez_compressed(HERE / "solves.npz", **out)
    (HERE / "solves.json").write_text(json.dumps(meta, indent=0, sort_keys=True))


def gen_cfg2():
    """cfg2 (1M x 2M, 20M nnz) oracle summary: per-pass log + final scalars."""
    import time
    spec = GeneratorSpec(kind="uniform_random", num_rows=1_000_000, num_cols=2_000_000,
                         nnz_target=20_000_000, inequality_fraction=0.3, seed=0)
    t0 = time.time()
    p = generate(spec)
    t1 = time.time()
    res, log = solve_logged(p, SolverConfig(tolerance=1e-4, seed=0))
    t2 = time.time()
    summary = {
        "spec": {"num_rows": 1_000_000, "num_cols": 2_000_000, "nnz_target": 20_000_000,
                 "inequality_fraction": 0.3, "seed": 0},
        "generate_seconds": t1 - t0, "solve_seconds": t2 - t1,
        "result": result_dict(res),
        "x_sum": float(np.sum(res.x)), "y_sum": float(np.sum(res.y)),
        "x_abs_sum": float(np.sum(np.abs(res.x))), "y_abs_sum": float(np.sum(np.abs(res.y))),
        "x_head": res.x[:16].tolist(), "y_head": res.y[:16].tolist(),
        "rhs_sum": float(np.sum(p.con_lower)), "c_sum": float(np.sum(p.objective)),
        "vals_sum": float(np.sum(p.matrix.values)),
        "col_checksum": int(np.sum(p.matrix.col_indices * (np.arange(p.matrix.nnz) % 1009))),
        "passlog": log.tolist(),
    }
    (HERE / "cfg2_summary.json").write_text(json.dumps(summary, indent=0, sort_keys=True))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg2", action="store_true")
    ap.add_argument("--only", default=None)
    a = ap.parse_args()
    steps = {"spmv": gen_spmv, "layouts": gen_layouts, "cfg1": gen_cfg1, "solves": gen_solves}
    for k, f in steps.items():
        if a.only and k != a.only:
            continue
        f()
        print("wrote", k, flush=True)
    if a.cfg2:
        gen_cfg2()
        print("wrote cfg2", flush=True)
