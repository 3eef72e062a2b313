"""Drop-in entry point: solve(problem, SolverConfig) -> SolveResult.

Same options, statuses, result fields and JSON payload as the reference
driver (/root/reference/pkg/src/gridlp/solver_driver.py:55-272,
pdhg_engine.py:48-126, docs/output.md). The compute runs on the B200 kernels;
there is no CPU path.

`comm_backend` selects the executor:
  "cuda" (default) — one process, one GPU; an R x C grid (n_procs / grid)
       keeps all R*C blocks in that GPU's HBM and reduces partial products
       in ascending device order (the reference's simulated grid semantics).
  "cooperative", "threads" — the reference's simulated-grid executors;
       accepted as aliases of "cuda" so reference call sites run unchanged.
  "nccl" — one process per GPU under torchrun, one grid block per rank,
       NCCL over NVLink between them (world size must equal rows*cols).
"""

from __future__ import annotations

import math
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np
import torch

from . import engine as eng
from .comm import CollectiveError, Ledger, NcclGrid, PeerGrid, VirtualGrid, WorkerError
from .blocks import upload_csr
from .layout import GridTopology, build_layout, layout_summary, unpermute_solution
from .ops import CudaOps
from .problem import reported_objective
from .scaling import MODES as SCALING_MODES
from .scaling import scale_problem

STEP_SIZE_SAFETY = 0.998
BACKENDS = ("cuda", "cooperative", "threads", "nccl", "peer")

STATUS_OPTIMAL = eng.OPTIMAL
STATUS_ITERATION_LIMIT = eng.ITERATION_LIMIT
STATUS_TIME_LIMIT = eng.TIME_LIMIT
STATUS_NUMERICAL_FAILURE = eng.NUMERICAL_FAILURE


@dataclass(frozen=True)
class StepSizes:
    """eta and primal weight omega; tau = eta/omega, sigma = eta*omega
    (pdhg_engine.py:48-67)."""

    eta: float
    omega: float

    def __post_init__(self):
        if not (self.eta > 0 and math.isfinite(self.eta)):
            raise ValueError("eta must be positive and finite")
        if not (self.omega > 0 and math.isfinite(self.omega)):
            raise ValueError("omega must be positive and finite")

    @property
    def tau(self) -> float:
        return self.eta / self.omega

    @property
    def sigma(self) -> float:
        return self.eta * self.omega


@dataclass(frozen=True)
class KktReport:
    """pdhg_engine.py:106-126."""

    r_primal: float
    r_dual: float
    r_gap: float
    obj_primal: float
    obj_dual: float

    @property
    def overall(self) -> float:
        return max(self.r_primal, self.r_dual, self.r_gap)

    def as_dict(self) -> dict:
        return {"r_primal": self.r_primal, "r_dual": self.r_dual, "r_gap": self.r_gap,
                "obj_primal": self.obj_primal, "obj_dual": self.obj_dual,
                "overall": self.overall}


@dataclass(frozen=True)
class SolverConfig:
    """solver_driver.py:55-101 (same fields, defaults and validation)."""

    tolerance: float = 1e-4
    max_iterations: int = 200_000
    time_limit_seconds: float | None = None
    kkt_interval: int = 64
    block_size: int = 64
    seed: int = 0
    n_procs: int = 1
    grid: tuple | None = None
    permutation: str = "block_random"
    partitioning: str = "nnz"
    gamma: float = 0.0
    halpern: bool = True
    restarts: bool = True
    beta_sufficient: float = 0.2
    beta_necessary: float = 0.8
    beta_artificial: float = 0.36
    pid_kp: float = 0.6
    pid_ki: float = 0.1
    pid_kd: float = 0.1
    omega_min: float = 1e-6
    omega_max: float = 1e6
    omega_initial: float | None = None
    eta: float | None = None
    power_iterations: int = 30
    collective_timeout_seconds: float = 120.0
    comm_backend: str = "cuda"
    # B200 extensions (not in the reference; defaults keep its behaviour):
    # on-device diagonal preconditioning (scaling.py) — "none", "ruiz",
    # "pock_chambolle" or "ruiz+pock_chambolle". With scaling the iteration,
    # the iteration and the restart tests run on the scaled LP; the KKT
    # report (termination, log, SolveResult.report) is evaluated on the
    # ORIGINAL LP at the unscaled iterate; x, y and the objective are
    # returned in the original space.
    scaling: str = "none"
    ruiz_iterations: int = 10

    def __post_init__(self):
        if self.tolerance <= 0:
            raise ValueError("tolerance must be positive")
        if self.kkt_interval < 1:
            raise ValueError("kkt_interval must be >= 1")
        if self.n_procs < 1:
            raise ValueError("n_procs must be >= 1")
        if self.max_iterations < 0:
            raise ValueError("max_iterations must be non-negative")
        if self.grid is not None:
            rows, cols = self.grid
            if rows < 1 or cols < 1:
                raise ValueError("grid dimensions must be positive")
            if rows * cols > self.n_procs:
                raise ValueError(f"grid {rows}x{cols} needs {rows * cols} devices but n_procs={self.n_procs}")
        if self.comm_backend not in BACKENDS:
            raise ValueError(f"unknown backend {self.comm_backend!r}; expected one of {BACKENDS}")
        if self.scaling not in SCALING_MODES:
            raise ValueError(f"unknown scaling {self.scaling!r}; expected one of {SCALING_MODES}")
        if self.ruiz_iterations < 0:
            raise ValueError("ruiz_iterations must be non-negative")

    def engine_options(self) -> eng.EngineOptions:
        return eng.EngineOptions(
            tolerance=self.tolerance, max_iterations=self.max_iterations,
            kkt_interval=self.kkt_interval, gamma=self.gamma, halpern=self.halpern,
            restarts=self.restarts, beta_sufficient=self.beta_sufficient,
            beta_necessary=self.beta_necessary, beta_artificial=self.beta_artificial,
            pid_kp=self.pid_kp, pid_ki=self.pid_ki, pid_kd=self.pid_kd,
            omega_min=self.omega_min, omega_max=self.omega_max,
            time_limit_seconds=self.time_limit_seconds)


@dataclass
class SolveResult:
    """solver_driver.py:123-146."""

    status: str
    x: np.ndarray
    y: np.ndarray
    report: KktReport
    objective: float
    iterations: int
    restarts: int
    wall_seconds: float
    counters: dict
    layout: dict
    timings: dict | None = None

    def to_json_dict(self) -> dict:
        return {"status": self.status, "objective": self.objective, "kkt": self.report.as_dict(),
                "iterations": self.iterations, "restarts": self.restarts,
                "counters": self.counters, "layout": self.layout}


def problem_scalars(problem):
    """(||c||, ||finite bounds||, constant) from the ORIGINAL order
    (solver_driver.py:149-158)."""
    lc = np.asarray(problem.con_lower, np.float64)
    uc = np.asarray(problem.con_upper, np.float64)
    finite_sq = float(np.sum(lc[np.isfinite(lc)] ** 2) + np.sum(uc[np.isfinite(uc)] ** 2))
    return (float(np.linalg.norm(np.asarray(problem.objective, np.float64))), math.sqrt(finite_sq),
            float(getattr(problem, "objective_constant", 0.0)))


_HOST_POOL = []
HOST_OVERLAP = True


class _Pair:
    def __init__(self, a, b):
        self.a, self.b = a, b

    def result(self):
        return self.a.result(), self.b.result()


class _Done:
    def __init__(self, value):
        self.value = value

    def result(self):
        return self.value


def _host_pool():
    if not _HOST_POOL:
        _HOST_POOL.append(ThreadPoolExecutor(3, thread_name_prefix="gridlp-host"))
    return _HOST_POOL[0]


def norm_probe_vector(n: int, seed: int) -> np.ndarray:
    """solver_driver.py:161-165."""
    return np.random.default_rng(np.random.SeedSequence(entropy=(seed, 0x5eed))).standard_normal(n)


def initial_omega(cfg: SolverConfig, cnorm: float, bnorm: float) -> float:
    """solver_driver.py:168-173."""
    if cfg.omega_initial is not None:
        return cfg.omega_initial
    if cnorm > 0.0 and bnorm > 0.0:
        return cnorm / bnorm
    return 1.0


def eta_from_estimate(cfg: SolverConfig, estimate: float) -> float:
    """solver_driver.py:176-181."""
    if cfg.eta is not None:
        return cfg.eta
    if estimate > 0.0:
        return STEP_SIZE_SAFETY / estimate
    return 1.0


def _log_pass(iteration, report, omega, eta, epoch_n):
    """Per-pass INFO line, same fields and order (solver_driver.py:184-190)."""
    eng.log.info(
        "iter=%d r_primal=%.6e r_dual=%.6e r_gap=%.6e obj_p=%.12e obj_d=%.12e "
        "omega=%.6e eta=%.6e epoch=%d",
        iteration, report.r_primal, report.r_dual, report.r_gap,
        report.obj_primal, report.obj_dual, omega, eta, epoch_n,
    )


def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the B200 PDHG path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def prepare(problem, cfg: SolverConfig, force_1x1=False, ops_factory=None, device=None,
            engine_overrides=None, scaled=None):
    """Layout + blocks in HBM + step sizes: everything before the main loop
    (solver_driver.py:199-227). Returns (engine, layout, eta, omega, timings)."""
    t_start = time.perf_counter()
    timings = {}
    banded = hasattr(problem, "bands")
    # host-only inputs of the step sizes (the reference's numpy RNG stream and
    # norms, which must stay bit-identical) are computed on a helper thread
    # while the layout and the device setup run; numpy drops the GIL in both
    # while the matrix goes up (it does not depend on the layout), the
    # layout's permutations follow on the same helper thread
    host_job = lambda: (problem_scalars(problem), norm_probe_vector(int(problem.matrix.num_cols), cfg.seed))  # noqa: E731
    if banded and (cfg.permutation != "none" or cfg.partitioning != "uniform"):
        raise ValueError("a band problem (blocks generated per device) needs permutation='none' and "
                         "partitioning='uniform'")
    grid = GridTopology(1, 1) if force_1x1 else (GridTopology(*cfg.grid) if cfg.grid is not None else None)
    layout_job = lambda: build_layout(problem, n_procs=1 if force_1x1 else cfg.n_procs,  # noqa: E731
                                      block_size=cfg.block_size, seed=cfg.seed, permutation=cfg.permutation,
                                      partitioning=cfg.partitioning, grid=grid)
    opts = cfg.engine_options()
    for k, v in (engine_overrides or {}).items():
        setattr(opts, k, v)
    preload = None
    if scaled is not None:
        # diagonally scaled LP: its CSR is already in HBM (scaling.py)
        if device is None:
            device = _device()
        preload = scaled.device_csr
        host_f = _host_pool().submit(host_job) if HOST_OVERLAP else _Done(host_job())
        layout = layout_job()
    elif (HOST_OVERLAP and not banded and opts.device_setup and torch.cuda.is_available()
            and (device is None or device.type == "cuda")):
        layout_f = _host_pool().submit(layout_job)
        scal_f = _host_pool().submit(problem_scalars, problem)
        probe_f = _host_pool().submit(norm_probe_vector, int(problem.matrix.num_cols), cfg.seed)
        host_f = _Pair(scal_f, probe_f)
        if device is None:
            device = _device()
        t0 = time.perf_counter()
        preload = upload_csr(problem.matrix, device)
        t1 = time.perf_counter()
        layout = layout_f.result()
        timings["setup_preload_s"] = t1 - t0
        timings["layout_wait_s"] = time.perf_counter() - t1
    else:
        host_f = None if banded else (_host_pool().submit(host_job) if HOST_OVERLAP else _Done(host_job()))
        layout = layout_job()
    timings["layout_s"] = time.perf_counter() - t_start
    R, C = layout.topology.rows, layout.topology.cols
    if device is None:
        device = _device()
    if cfg.comm_backend in ("nccl", "peer") and not force_1x1:
        comm = (PeerGrid if cfg.comm_backend == "peer" else NcclGrid)(R, C, device, cfg.collective_timeout_seconds)
        if comm.world != R * C:
            raise ValueError(f"{cfg.comm_backend} backend needs world size == grid devices ({R * C}), "
                             f"got {comm.world}")
    else:
        comm = VirtualGrid(R, C)
    with eng.nvtx_range("gridlp.setup_blocks"):
        engine = eng.PdhgEngine(problem, layout, opts, comm, ops_factory or CudaOps, device, 0.0, 0.0, 0.0,
                                preload=preload,
                                kkt_scale=None if scaled is None else (scaled.row_scale_device,
                                                                       scaled.col_scale_device))
    del preload
    timings.update(engine.timings)
    timings["layout_order"] = engine.choices.get("order")
    probe = None
    if not banded:
        t0 = time.perf_counter()
        (cnorm, bnorm, const), probe = host_f.result()
        engine.cnorm, engine.bnorm, engine.const = cnorm, bnorm, const
        if scaled is not None:
            # KKT is reported on the original LP: its norms normalise the
            # residuals; the scaled norms (above) set the initial primal weight
            engine.cnorm, engine.bnorm, _ = problem_scalars(scaled.original)
        timings["host_scalars_wait_s"] = time.perf_counter() - t0
    if banded:
        cnorm, bnorm = engine.band_scalars()
        engine.cnorm, engine.bnorm = cnorm, bnorm
    t0 = time.perf_counter()
    with eng.nvtx_range("gridlp.power_iteration"):
        estimate = engine.power_estimate(cfg.power_iterations, probe, cfg.seed)
    timings["power_s"] = time.perf_counter() - t0
    timings["estimate"] = estimate
    eta = eta_from_estimate(cfg, estimate)
    omega = initial_omega(cfg, cnorm, bnorm)
    StepSizes(eta, omega)  # validates like the reference
    return engine, layout, eta, omega, timings


def _solve(problem, cfg: SolverConfig, trace=None, force_1x1=False, ops_factory=None,
           device=None, engine_overrides=None) -> SolveResult:
    t_start = time.perf_counter()
    scaled = None
    if cfg.scaling != "none":
        if hasattr(problem, "bands"):
            raise ValueError("scaling is not supported for band problems (blocks generated per device)")
        scaled = scale_problem(problem, cfg.scaling, cfg.ruiz_iterations, device)
        scaled.original = problem
        original, problem = problem, scaled.problem
    engine, layout, eta, omega, timings = prepare(problem, cfg, force_1x1, ops_factory, device,
                                                  engine_overrides, scaled=scaled)
    if scaled is not None:
        timings["scaling_s"] = scaled.seconds
    comm = engine.comm
    setup_events = engine.ledger.snapshot()
    leader = (not comm.local) or comm.local[0] == (0, 0)
    try:
        out = engine.run(eta, omega, trace=trace, log_hook=_log_pass if leader else None)
    except CollectiveError:
        raise
    except Exception as exc:
        if comm.kind in ("nccl", "peer"):
            # a device worker failed (reference solver_driver.py:215, comm.py:219-221)
            raise WorkerError(f"device {comm.local} failed: {exc}") from exc
        raise
    if comm.kind in ("nccl", "peer"):
        comm.agree(out["status"], "statuses")       # solver_driver.py:242-244
    timings.update(engine.timings)
    xy = engine.solution_original()
    if xy is None:
        xs, ys = engine.solution_blocks()
        xy = unpermute_solution(layout, xs, ys)
    x, y = xy
    if scaled is not None:
        x, y = scaled.unscale(x, y)
        problem = original
    rep = out["report"]
    report = KktReport(rep.r_primal, rep.r_dual, rep.r_gap, rep.obj_primal, rep.obj_dual)
    final_events = engine.ledger.snapshot()
    setup = Ledger.expand(setup_events, layout)
    total = Ledger.expand(final_events, layout)
    counters = {"setup": setup, "total": total,
                "main_loop": Ledger.expand(Ledger.diff(final_events, setup_events), layout),
                "grid_total": Ledger.grid_total(total)}
    if force_1x1:
        counters = {}
    timings["h2d_bytes"] = engine.h2d_bytes
    timings["passes"] = engine.passes
    return SolveResult(
        status=out["status"], x=x, y=y, report=report,
        objective=reported_objective(problem, report.obj_primal),
        iterations=out["iterations"], restarts=out["restarts"],
        wall_seconds=time.perf_counter() - t_start, counters=counters,
        layout=layout_summary(problem, layout, engine.per_device_nnz),
        timings=timings,
    )


def warmup() -> None:
    """Optional, once per process before the first timed solve: loads the
    sm_100a kernels (CUDA loads each kernel lazily at its first launch), the
    device-setup kernels and allocator pools, the pinned staging buffers and
    the host helper threads, by solving a small LP. The first solve of a
    process otherwise pays ~0.4 s for these (profiles/r1/e2e_host.md)."""
    from .blocks import upload
    from .generators import GeneratorSpec, generate

    dev = _device()
    upload(np.zeros(1 << 18), np.float64, dev)        # > 1 MB: allocates the pinned staging pair
    p = generate(GeneratorSpec(kind="uniform_random", num_rows=3000, num_cols=5000, nnz_target=40000,
                               inequality_fraction=0.3, seed=0))
    _solve(p, SolverConfig(tolerance=1e-4, max_iterations=256))
    torch.cuda.synchronize(dev)


def solve(problem, cfg: SolverConfig | None = None) -> SolveResult:
    """Solve on the device grid; deterministic for fixed (problem, cfg, seed)
    (solver_driver.py:193-272)."""
    return _solve(problem, cfg or SolverConfig())


def reference_solve(problem, cfg: SolverConfig | None = None, trace=None) -> SolveResult:
    """Single-device twin (solver_driver.py:290-332): the same algorithm on
    a forced 1x1 grid. `trace` collects (iteration, x, y) in permuted order;
    a trace object with a `keep` set records only those iterations."""
    return _solve(problem, cfg or SolverConfig(), trace=trace, force_1x1=True)
