"""Benchmark: PDHG iterations/s (FP64) on the BASELINE configs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg2|cfg1]

Workload (BASELINE.json configs[1], "cfg2"): the reference generator's
uniform_random LP, m=1,000,000 rows, n=2,000,000 columns, 20,000,000
nonzeros, 30% ranged rows, seed 0 — generated here with the same numpy
Generator sequence (synthetic, random-init; no datasets offline).

One STEP = one KKT interval of the reference loop: 64 PDHG iterations
(fused A^T y + primal/Halpern, fused A x_bar + dual/Halpern; a replayed CUDA
graph) followed by one KKT + restart-probe pass with its host decision
(pdhg_engine.py:389-462). tolerance is set to 1e-300 for the timed region so
every step does the full work; restarts fire as the reference's rules say.

`value` = iterations/s over the K timed steps (device time, CUDA events,
max over ranks). `e2e` = the same metric through the public API
`solve(problem, SolverConfig(tolerance=1e-4))` from host arrays to the
optimal status (setup, H2D, power iteration, iterations, D2H included),
with time-to-tolerance beside it. `roofline` = the fused iteration's
algorithmic bytes over its measured duration against the
measured HBM copy peak.

`--impl reference` times the reference algorithm's CPU implementation (the
numpy/scipy oracle restating reference_solve; the reference package itself
is pure Python and is not shipped to the GPU box) on the host cores with
one thread per grid block, as the reference's threads executor runs.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    "cfg2": dict(kind="uniform_random", num_rows=1_000_000, num_cols=2_000_000, nnz_target=20_000_000,
                 inequality_fraction=0.3, seed=0),
    "cfg1": dict(kind="uniform_random", num_rows=2_000, num_cols=4_000, nnz_target=20_000,
                 inequality_fraction=0.3, seed=0),
    # device generators (paper_2601_07628_b200/synth.py)
    "cfg3": dict(gen="powerlaw", num_rows=10_000_000, num_cols=20_000_000, nnz_target=200_000_000,
                 inequality_fraction=0.3, seed=0),
    "cfg3s": dict(gen="powerlaw", num_rows=1_000_000, num_cols=2_000_000, nnz_target=20_000_000,
                  inequality_fraction=0.3, seed=0),
    "cfg4": dict(gen="mcf", num_nodes=2_000, num_arcs=128_000, num_commodities=1_300, seed=0),
    "cfg4s": dict(gen="mcf", num_nodes=500, num_arcs=32_000, num_commodities=200, seed=0),
    # planted-optimum LP generated block by block (synth.BandProblem): cfg5 is
    # ~8B nnz (A + A^T > 180 GB, needs >= 4 GPUs); cfg5s is a 1/20 one-GPU cut
    "cfg5": dict(gen="planted", num_rows=250_000_000, num_cols=400_000_000, draws_per_row=32, seed=0),
    "cfg5s": dict(gen="planted", num_rows=12_500_000, num_cols=20_000_000, draws_per_row=32, seed=0),
    # one grid block of cfg5 on a 2x2 grid (4 GPUs): 125M x 200M, ~2B nnz
    # (16 of each row's 32 draws fall in a column half) — the single-GPU
    # readiness run for the sharded oversized solve
    "cfg5q": dict(gen="planted", num_rows=125_000_000, num_cols=200_000_000, draws_per_row=16, seed=0),
}
WORKLOADS = {
    "uniform_random": "reference generator uniform_random LP",
    "powerlaw": "power-law (Chung-Lu, exponent 0.8, heavy-first) feasible LP, device generator",
    "mcf": "block-angular multi-commodity flow LP (planted flow), device generator",
    "planted": "uniform random LP with a planted optimum, generated block by block on each device",
}
METRIC = "PDHG iters/s & time-to-1e-4 KKT (FP64) at 1/2/4/8 B200; SpMV HBM GB/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clocks / throttle reasons sampled DURING the timed region: NVML
    (pynvml) polled every 5 ms on a helper thread, plus one sample at entry
    and one at exit, so even a sub-second timed region has samples;
    `nvidia-smi -lms` as the fallback when pynvml is missing."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, index: int):
        self.index = index
        self.samples = []          # (sm_mhz, max_mhz, reasons bitmask)
        self._stop = threading.Event()
        self._nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self._max = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self._nvml = None
        self.proc = None
        self.lines = []

    def _sample(self):
        p = self._nvml
        try:
            sm = float(p.nvmlDeviceGetClockInfo(self._h, p.NVML_CLOCK_SM))
            try:
                rs = int(p.nvmlDeviceGetCurrentClocksEventReasons(self._h))
            except AttributeError:
                rs = int(p.nvmlDeviceGetCurrentClocksThrottleReasons(self._h))
            self.samples.append((sm, self._max, rs))
        except Exception:
            pass

    def _poll(self):
        while not self._stop.wait(0.005):
            self._sample()

    def __enter__(self):
        if self._nvml is not None:
            self._sample()
            self._t = threading.Thread(target=self._poll, daemon=True)
            self._t.start()
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self._nvml is not None:
            self._stop.set()
            self._t.join(timeout=1)
            self._sample()
            return
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], [], set()
        if self._nvml is not None:
            for c, mx, rs in self.samples:
                sm.append(c)
                smax.append(mx)
                for name, attr in self.REASONS:
                    bit = getattr(self._nvml, attr, 0)
                    if bit and rs & bit:
                        reasons.add(name)
        else:
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for line in self.lines:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 6:
                    continue
                try:
                    sm.append(float(parts[0]))
                    smax.append(float(parts[1]))
                except ValueError:
                    continue
                for name, val in zip(names, parts[2:6]):
                    if val.lower() == "active":
                        reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvml" if self._nvml is not None else "nvidia-smi"}


def make_problem(name):
    from paper_2601_07628_b200 import GeneratorSpec, generate

    t0 = time.perf_counter()
    spec = dict(CONFIGS[name])
    gen = spec.pop("gen", None)
    if gen is None:
        p = generate(GeneratorSpec(**spec))
    elif gen == "planted":
        from paper_2601_07628_b200 import synth

        p = synth.BandProblem(synth.PlantedBands(synth.PlantedSpec(**spec)), name)
        log(f"[bench] {name}: band problem m={p.num_constraints} n={p.num_variables} (blocks generated per device)")
        return p
    else:
        import torch

        from paper_2601_07628_b200 import synth

        dl = (synth.generate_powerlaw(synth.PowerLawSpec(**spec)) if gen == "powerlaw"
              else synth.generate_mcf(synth.McfSpec(**spec)))
        torch.cuda.synchronize()
        log(f"[bench] device generation {time.perf_counter() - t0:.1f}s")
        p = dl.to_problem(name)
        del dl
        torch.cuda.empty_cache()
    log(f"[bench] generated {name}: m={p.num_constraints} n={p.num_variables} "
        f"nnz={p.matrix.nnz} in {time.perf_counter() - t0:.1f}s")
    return p


def measure_config(name: str, dev, steps: int = 3) -> dict:
    """Device µs per fused iteration and the HBM roofline fraction of another
    BASELINE config on this GPU (the same measurement as the main line, a
    few steps): recorded as an extra key so every driver bench run carries
    the power-law (cfg3) number next to the cfg2 headline."""
    import torch

    from paper_2601_07628_b200 import SolverConfig
    from paper_2601_07628_b200.api import prepare

    p = make_problem(name)
    cfg = SolverConfig(tolerance=1e-300, max_iterations=10**12, seed=0)
    engine, layout, eta, omega, tim = prepare(p, cfg, device=dev)
    engine.start(eta, omega)
    for _ in range(3):
        engine.step()
    torch.cuda.synchronize()
    engine.iteration_events = []
    for _ in range(steps):
        engine.step()
    torch.cuda.synchronize()
    ev = engine.iteration_events
    t_iter = sum(a.elapsed_time(b) for a, b, _ in ev) * 1e-3 / max(sum(n for _, _, n in ev), 1)
    b = iteration_bytes(engine)
    peak, _ = measured_peak()
    nnz = sum(v for v in engine.per_device_nnz if v >= 0)
    out = {"workload": f"{name}: {workload_name(name)}, m={p.num_constraints} n={p.num_variables} "
                       f"nnz={nnz}",
           "us_per_iteration": t_iter * 1e6, "iterations_per_s": 1.0 / t_iter,
           "bytes_per_iteration": b["iteration"], "achieved_GBs": b["iteration"] / t_iter / 1e9,
           "frac": b["iteration"] / t_iter / 1e9 / peak, "layout_choices": dict(engine.choices)}
    if name == "cfg3":
        # the pattern's own ceiling: Zipf(0.8) 8-byte gathers over the 160 MB x_bar
        # and the 80 MB y at the rates tools/microbench_l2.cu measured on this
        # B200 (profiles/r2/microbench_l2.jsonl), before any stream byte
        rates = {"x_bar_160MB": 203.2e9, "y_80MB": 308.5e9}
        floor = nnz / rates["x_bar_160MB"] + nnz / rates["y_80MB"]
        out["gather_bound"] = {"gathers_per_s": rates, "seconds_at_ceiling": floor, "frac": floor / t_iter,
                               "source": "profiles/r2/microbench_l2.jsonl"}
    del engine, p
    torch.cuda.empty_cache()
    return out


def cfg1_latency(dev, runs: int = 3) -> dict:
    """BASELINE configs[0] (the reference's own CPU-runnable case, 2k x 4k,
    20k nnz): time to 1e-4 through the public solve() from host arrays
    (median of `runs` complete solves after one warm solve) and the device
    µs per iteration of its main loop. This size is launch bound (two
    products of 20k nonzeros per iteration): CUDA graphs of 64 iterations
    with programmatic chaining between the products."""
    import torch

    from paper_2601_07628_b200 import GeneratorSpec, SolverConfig, generate, solve
    from paper_2601_07628_b200.api import prepare

    p = generate(GeneratorSpec(**CONFIGS["cfg1"]))
    cfg = SolverConfig(tolerance=1e-4, seed=0)
    solve(p, cfg)
    walls = []
    for _ in range(runs):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = solve(p, cfg)
        walls.append(time.perf_counter() - t0)
    engine, layout, eta, omega, tim = prepare(p, SolverConfig(tolerance=1e-300, max_iterations=10**12, seed=0),
                                              device=dev)
    engine.start(eta, omega)
    for _ in range(3):
        engine.step()
    torch.cuda.synchronize()
    engine.iteration_events = []
    for _ in range(20):
        engine.step()
    torch.cuda.synchronize()
    ev = engine.iteration_events
    t_iter = sum(a.elapsed_time(b) for a, b, _ in ev) * 1e-3 / max(sum(n for _, _, n in ev), 1)
    del engine
    return {"workload": "cfg1: reference generator uniform_random LP m=2000 n=4000 nnz=20000 ineq=0.3 seed=0",
            "time_to_tol_s": statistics.median(walls), "runs_s": walls, "status": res.status,
            "iterations": res.iterations, "restarts": res.restarts, "objective": res.objective,
            "us_per_iteration": t_iter * 1e6,
            "reference_cpu_time_to_tol_s": "2.09-2.55 (BASELINE.md section 4, reference CPU PDHG)"}


def kernel_tuning() -> dict:
    from paper_2601_07628_b200 import native

    lib = native.load()
    return {k: lib.get_tuning(k) for k in ("sell_variant", "chain_products", "wide_ctas")}


def workload_name(cfg: str) -> str:
    c = CONFIGS[cfg]
    return WORKLOADS[c.get("gen") or c["kind"]]


def iteration_bytes(engine) -> dict:
    """Algorithmic bytes of one fused iteration per device:
    K1 (A^T y + primal): 12 nnz + 4(n+1) + 8 m (y gathered once) + 40 n read
    (x, c, lo, hi, x_anchor) + 16 n written (x, x_bar);
    K2 (A x_bar + dual): 12 nnz + 4(m+1) + 8 n (x_bar once) + 32 m read
    (y, lo, hi, y_anchor) + 8 m written."""
    out = {"K1": 0, "K2": 0}
    for blk in engine.blocks.values():
        m, n, nnz = blk.A.num_rows, blk.A.num_cols, blk.A.nnz
        out["K1"] += 12 * nnz + 4 * (n + 1) + 8 * m + 56 * n
        out["K2"] += 12 * nnz + 4 * (m + 1) + 8 * n + 40 * m
    out["iteration"] = out["K1"] + out["K2"]
    # bytes the kernels actually have to move on this instance: with uniform
    # variable bounds (GRIDLP_F_UNIFORM_BOUNDS) K1 reads two scalars instead
    # of the two n-vectors lo, hi
    out["iteration_moved"] = out["iteration"] - sum(
        16 * c.n for c in engine.cols.values() if getattr(c, "uniform_bounds", False))
    # ... and with a compact value codec (DeviceCsr.val_codec: +-1 values in the
    # column's sign bit, or exact floats) 8 resp. 4 fewer bytes per nonzero
    saved = 0
    for blk in engine.blocks.values():
        for mat in (blk.A, blk.AT):
            for d in getattr(mat, "bands", [mat]):
                saved += (0, 4, 8)[getattr(d, "val_codec", 0)] * d.nnz
    out["iteration_moved"] -= saved
    out["value_bytes_saved"] = saved
    # L1->L2 requests: one 32-byte sector request per gathered element (random
    # columns: no two lanes of a warp share a 128-byte line) plus one request
    # per 128-byte line of every streamed array
    gathers = sum(2 * blk.A.nnz for blk in engine.blocks.values())
    vec_once = sum(8 * (blk.A.num_rows + blk.A.num_cols) for blk in engine.blocks.values())
    out["requests"] = gathers + (out["iteration"] - vec_once) // 128
    return out


# Random 8-byte gathers from an L2-resident vector on this B200: 255 G/s
# (tools/microbench.cu, profiles/r1/microbench_gather.log) — one L1->L2
# sector request per gather, the port ncu shows 77-81 % busy in K1/K2
# (profiles/r1/ncu_sell32_full.md).
GATHER_CEILING_PER_S = 255e9


def spmv_compare(problem, device, reps=20) -> dict:
    """SpMV-only HBM GB/s: y = A·x over the instance's own CSR,
    our product (gridlp_op_store, bit-identical to scipy) against cuSPARSE
    csrmv through torch.sparse (FP64, int32 indices) on the same matrix and
    vector; CUDA events on the launching stream, L2 not flushed (A is 240 MB,
    > L2). Bytes per product: 12 nnz + 4(rows+1) + 8 cols + 8 rows. Ours is
    timed in both of its layouts: the rows in the user's order ("ours_us")
    and in the engine's internal length-class order ("ours_sorted_us", the
    layout every solve uses; y comes out permuted, same values)."""
    import numpy as np
    import torch

    from paper_2601_07628_b200.blocks import DeviceCsr, HostCsr, length_order, permute_csr
    from paper_2601_07628_b200.ops import CudaOps, Fused

    M = problem.matrix
    m, n = int(M.num_rows), int(M.num_cols)
    h = HostCsr(m, n, np.asarray(M.row_offsets, np.int64), np.asarray(M.col_indices, np.int64),
                np.asarray(M.values, np.float64))
    from paper_2601_07628_b200.blocks import LIGHT_ROW_CANDIDATES

    lens = np.diff(h.ptr)
    # the engine's per-block light_row_max choice (layout_autotune.md): every
    # candidate that moves rows is timed, the fastest is "ours"
    cands = [c for k, c in enumerate(LIGHT_ROW_CANDIDATES)
             if k == 0 or bool(np.any((lens > LIGHT_ROW_CANDIDATES[k - 1]) & (lens <= c)))]
    A = DeviceCsr(h, device, light_row_max=cands[0])
    ops = CudaOps(device, A.slots() + 8, 1)
    x = torch.from_numpy(np.random.default_rng(0).standard_normal(n)).to(device)
    ours = torch.empty(m, dtype=torch.float64, device=device)
    T = torch.sparse_csr_tensor(torch.from_numpy(h.ptr.astype(np.int32)), torch.from_numpy(h.col.astype(np.int32)),
                                torch.from_numpy(h.val), size=(m, n)).to(device)
    xs = x.reshape(n, 1)

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        evs = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            evs.append((a, b))
        torch.cuda.synchronize()
        return sorted(a.elapsed_time(b) for a, b in evs)[reps // 2] * 1e-3

    t_ours = timed(lambda: ops.store(Fused(A, x), ours))
    per_light = {cands[0]: t_ours * 1e6}
    light = cands[0]
    for c in cands[1:]:
        Ac = DeviceCsr(h, device, light_row_max=c)
        opc = CudaOps(device, Ac.slots() + 8, 1)
        tc = timed(lambda: opc.store(Fused(Ac, x), ours))
        per_light[c] = tc * 1e6
        if tc < t_ours:
            A, ops, t_ours, light = Ac, opc, tc, c
    ops.store(Fused(A, x), ours)
    order = length_order(np.diff(h.ptr))
    As = DeviceCsr(permute_csr(h, order), device, light_row_max=light)
    ours_s = torch.empty(m, dtype=torch.float64, device=device)
    t_sorted = timed(lambda: ops.store(Fused(As, x), ours_s))
    same_sorted = bool(torch.equal(ours_s, ours[torch.from_numpy(order).to(device)]))
    lib = {}
    t_lib = timed(lambda: lib.__setitem__("y", torch.mm(T, xs)))
    same = bool(torch.equal(lib["y"].reshape(m), ours))
    direct = cusparse_direct(T, x, m, n, h.nnz, reps, ours)
    bytes_ = 12 * h.nnz + 4 * (m + 1) + 8 * n + 8 * m
    out = {"rows": m, "cols": n, "nnz": h.nnz, "bytes_per_product": bytes_,
           "ours_us": t_ours * 1e6, "ours_GBs": bytes_ / t_ours / 1e9,
           "ours_sorted_us": t_sorted * 1e6, "ours_sorted_GBs": bytes_ / t_sorted / 1e9,
           "sorted_equals_natural_bitwise": same_sorted, "speedup_sorted_vs_cusparse": t_lib / t_sorted,
           "cusparse_us": t_lib * 1e6, "cusparse_GBs": bytes_ / t_lib / 1e9,
           "speedup_vs_cusparse": t_lib / t_ours, "cusparse_bitwise_equal_ours": same,
           "median_of": reps, "light_row_max": light, "ours_us_by_light_row_max": per_light,
           "cusparse_spmv_direct": direct}
    if direct:
        best = min(v["us"] for v in direct.values())
        out["speedup_vs_cusparse_spmv_best_alg"] = best / (t_ours * 1e6)
        out["speedup_sorted_vs_cusparse_spmv_best_alg"] = best / (t_sorted * 1e6)
    del A, As, ops, T
    torch.cuda.empty_cache()
    return out


def cusparse_direct(T, x, m, n, nnz, reps, ours):
    """cusparseSpMV called directly (tools/cusparse_ref.cu) with
    CUSPARSE_SPMV_CSR_ALG1 and ALG2 on the same CSR and vector: median µs of
    `reps`, and whether its y equals ours bit for bit."""
    import ctypes

    import torch

    so = ROOT / "tools" / "_lib" / "libcusparse_ref.so"
    if not so.exists():
        return None
    lib = ctypes.CDLL(str(so))
    f = lib.cusparse_ref_spmv
    f.argtypes = [ctypes.c_int64] * 3 + [ctypes.c_void_p] * 5 + [ctypes.c_int, ctypes.c_int,
                                                                ctypes.POINTER(ctypes.c_float), ctypes.c_void_p]
    f.restype = ctypes.c_int
    ptr, col, val = T.crow_indices(), T.col_indices(), T.values()
    res = {}
    for alg in (1, 2):
        y = torch.empty(m, dtype=torch.float64, device=x.device)
        ms = ctypes.c_float(0.0)
        rc = f(m, n, nnz, ptr.data_ptr(), col.data_ptr(), val.data_ptr(), x.data_ptr(), y.data_ptr(), alg, reps,
               ctypes.byref(ms), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        if rc == 0:
            bytes_ = 12 * nnz + 4 * (m + 1) + 8 * n + 8 * m
            res[f"CSR_ALG{alg}"] = {"us": ms.value * 1e3, "GBs": bytes_ / (ms.value * 1e-3) / 1e9,
                                    "bitwise_equal_ours": bool(torch.equal(y, ours))}
        else:
            res[f"CSR_ALG{alg}"] = {"error": rc}
    return res


def kernel_times(engine, reps=20):
    """Per-launch device time of the two fused kernels, eager launches with
    CUDA events on the launching stream (outside the graph)."""
    import torch

    ops = engine.ops
    cols, rows = engine.cols, engine.rows
    t = {"K1": [], "K2": []}
    for _ in range(reps):
        for j, col in cols.items():
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ops.primal(engine._run_plan(engine.plan_primal[j]), col, 0, engine.opts.halpern)
            e1.record()
            t["K1"].append((e0, e1))
        for i, row in rows.items():
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ops.dual(engine._run_plan(engine.plan_dual[i]), row, 0, engine.opts.halpern)
            e1.record()
            t["K2"].append((e0, e1))
    torch.cuda.synchronize()
    return {k: float(np.mean([a.elapsed_time(b) for a, b in v])) * 1e-3 for k, v in t.items()}


def run_reference(args, rank, world):
    """CPU arm: the reference algorithm on the host cores."""
    from oracle import pdhg_oracle

    if rank != 0:
        return
    try:
        from threadpoolctl import threadpool_limits
    except ImportError:  # pragma: no cover
        threadpool_limits = None
    from paper_2601_07628_b200 import select_grid

    p = make_problem(args.config)
    threads = max(1, min(os.cpu_count() or 1, 32))      # every host core the box has (capped at 32 blocks)
    g = select_grid(p.num_constraints, p.num_variables, threads)
    sample = args.ref_sample_iters
    ctx = threadpool_limits(1) if threadpool_limits else None
    total_iters, total_s, setup = 0, 0.0, None
    try:
        for s in range(args.warmup + args.steps):
            r = pdhg_oracle.iteration_rate(p, sample, grid=(g.rows, g.cols), threads=g.rows * g.cols)
            setup = r["setup_seconds"]
            if s >= args.warmup:
                total_iters += r["iterations"]
                total_s += r["seconds"]
    finally:
        if ctx is not None:
            ctx.unregister() if hasattr(ctx, "unregister") else None
    value = total_iters / total_s
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "iterations/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total_s / max(args.steps, 1), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: uniform_random LP m=1e6 n=2e6 nnz=2e7 ineq=0.3 seed=0"
                   if args.config == "cfg2" else f"{args.config}", "grid": [g.rows, g.cols]},
        "cpu_baseline": {"value": value, "unit": "iterations/s", "cores": g.rows * g.cols,
                         "kind": "port",
                         "sample": f"{sample} main-loop iterations per step on a {g.rows}x{g.cols} "
                                   f"block grid, one host thread per block for the block products and "
                                   f"the per-block epilogues (scipy csr_matvec and numpy release the "
                                   f"GIL), block build {setup:.1f}s untimed"},
        "e2e": {"value": value, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(problem, iters):
    from oracle import pdhg_oracle

    try:
        from threadpoolctl import threadpool_limits
        ctx = threadpool_limits(1)
    except ImportError:  # pragma: no cover
        ctx = None
    r = pdhg_oracle.iteration_rate(problem, iters, grid=(1, 1), threads=1)
    del ctx
    return {"value": r["iters_per_s"], "unit": "iterations/s", "cores": 1, "kind": "port",
            "sample": f"{iters} main-loop iterations of the reference algorithm (oracle/pdhg_oracle.py, "
                      f"numpy + scipy csr_matvec, 1 thread, 1x1 grid) on the same instance; "
                      f"{r['seconds']:.1f}s timed, block build {r['setup_seconds']:.1f}s untimed"}


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2601_07628_b200 import SolverConfig, select_grid, solve
    from paper_2601_07628_b200.api import prepare

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    p = make_problem(args.config)
    if world > 1 or args.force_nccl:
        g = select_grid(p.num_constraints, p.num_variables, world)
        base = dict(n_procs=world, grid=(g.rows, g.cols), comm_backend=args.comm)
    elif args.grid:
        R, C = (int(v) for v in args.grid.lower().split("x"))
        base = dict(n_procs=R * C, grid=(R, C))       # virtual grid: all blocks on this GPU
    else:
        base = dict(n_procs=1)
    if hasattr(p, "bands"):
        base.update(permutation="none", partitioning="uniform")
    if args.permutation:
        base["permutation"] = args.permutation
    if args.partitioning:
        base["partitioning"] = args.partitioning
    cfg = SolverConfig(tolerance=1e-300, max_iterations=10**12, seed=0, **base)
    t0 = time.perf_counter()
    over = {}
    if args.light_row_max is not None:
        over["light_row_max"] = args.light_row_max
    if args.no_graphs:
        over["use_graphs"] = False
    if args.natural_order:
        over["sorted_order"] = False
    if args.column_bands is not None:
        over["column_bands"] = args.column_bands
    if args.band_mb is not None:
        over["band_bytes"] = int(args.band_mb) << 20
    if args.no_first_touch:
        over["first_touch_cols"] = False
    if args.graph_nccl:
        over["graph_nccl"] = True
    if args.value_codec is not None:
        over["value_codec"] = args.value_codec
    if args.device_loop:
        over["device_loop"] = True
    engine, layout, eta, omega, tim = prepare(p, cfg, device=dev, engine_overrides=over)
    log(f"[bench] rank {rank}: setup {time.perf_counter() - t0:.1f}s {tim}")
    R, C = layout.topology.rows, layout.topology.cols
    pdn = [v for v in (engine.per_device_nnz or []) if v >= 0]
    nnz_total = int(sum(pdn))
    balance = (max(pdn) / (sum(pdn) / len(pdn))) if pdn and sum(pdn) else None
    engine.start(eta, omega)
    for _ in range(args.warmup):
        engine.step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # single-block grids: the timed steps run through the device-side loop
    # (the solve's own main loop: KKT intervals chained on the device, exactly
    # args.steps passes); the kernel-only time per iteration (roofline) is
    # then taken from a few host-driven intervals right after
    device_loop = engine._loop_ok() and not args.no_device_loop
    engine.iteration_events = None if device_loop else []
    launches0 = engine.ops.launches
    it0 = engine._s["total"]
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clocks:
        torch.cuda.synchronize()
        start.record()
        if device_loop:
            p0 = engine.passes
            while engine.passes - p0 < args.steps:
                engine.loop_budget = args.steps - (engine.passes - p0)
                engine.step(device_loop=True)
            engine.loop_budget = None
        else:
            for _ in range(args.steps):
                engine.step()
        stop.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    elapsed = start.elapsed_time(stop) * 1e-3
    iters = engine._s["total"] - it0
    launches = engine.ops.launches - launches0
    if device_loop:
        engine.iteration_events = []
        for _ in range(3):
            engine.step()
        torch.cuda.synchronize()
    ev = engine.iteration_events
    engine.iteration_events = None
    loop_s = sum(a.elapsed_time(b) for a, b, _ in ev) * 1e-3
    loop_iters = sum(n for _, _, n in ev)
    if world > 1:
        t = torch.tensor([elapsed, loop_s / max(loop_iters, 1)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed, t_iter = float(t[0]), float(t[1])
    else:
        t_iter = loop_s / max(loop_iters, 1)
    bytes_ = iteration_bytes(engine)
    peak, peak_src = measured_peak()
    ktimes = kernel_times(engine) if world == 1 else {}
    achieved = bytes_["iteration"] / t_iter / 1e9
    traffic = None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        tr = json.loads(tf.read_text()).get(args.config)
        traffic = tr["bytes_per_iteration"] if isinstance(tr, dict) else tr
    restarts = engine._s["epoch"]
    choices = {k: v for k, v in engine.choices.items()}
    del engine
    torch.cuda.empty_cache()
    spmv = spmv_compare(p, dev) if world == 1 and not args.no_spmv and not hasattr(p, "bands") else None
    extra = {}
    if world == 1 and args.config == "cfg2" and not args.no_extra:
        extra["cfg1_latency"] = cfg1_latency(dev)
        extra["cfg3"] = measure_config("cfg3", dev)

    # e2e through the public API, host arrays in, host arrays out
    e2e = None
    if not args.no_e2e:
        walls = []
        for _ in range(args.e2e_runs):           # each run is a complete solve from host arrays
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = solve(p, SolverConfig(tolerance=1e-4, seed=0, **base))
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
            if world > 1:
                t = torch.tensor([wall], dtype=torch.float64, device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                wall = float(t[0])
            walls.append(wall)
        wall = statistics.median(walls)
        passes = max(res.timings.get("passes", 1), 1)
        d2h = 8 * (p.num_variables + p.num_constraints)
        e2e = {"value": res.iterations / wall, "unit": "iterations/s",
               "h2d_bytes_per_step": int(res.timings.get("h2d_bytes", 0) / passes),
               "d2h_bytes_per_step": int(d2h / passes + 8 * 64 * 4),
               "time_to_tol_s": wall, "runs_s": walls, "status": res.status, "iterations": res.iterations,
               "restarts": res.restarts, "objective": res.objective,
               "kkt": res.report.as_dict(),
               "breakdown_s": {k: v for k, v in res.timings.items() if k.endswith("_s")}}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not hasattr(p, "bands"):
        cpu = cpu_baseline(p, args.cpu_sample_iters)
    if rank != 0:
        return
    value = iters / elapsed
    line = {
        "metric": METRIC, "value": value, "unit": "iterations/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{args.config}: {workload_name(args.config)}, m={p.num_constraints} "
                               f"n={p.num_variables} nnz={nnz_total}, spec {CONFIGS[args.config]}; step = 64 PDHG "
                               f"iterations + 1 KKT/restart pass",
                   "grid": [R, C], "permutation": cfg.permutation, "partitioning": cfg.partitioning,
                   "block_nnz_max_over_mean": balance,
                   "l2": "inputs larger than L2 (A + A^T = "
                   f"{24 * nnz_total / 1e6:.0f} MB of 126 MB L2 per iteration, streamed evict-first)",
                   "restarts_in_timed_region": restarts, "layout_choices": choices,
                   "main_loop": ("device (WHILE-graph of KKT intervals, gridlp_loop_graph_*; kernel time per "
                                 "iteration from 3 host-driven intervals after the timed region)"
                                 if device_loop else "host-driven KKT intervals"),
                   "kernel_tuning": kernel_tuning(),
                   "ranks_share_gpus": world > 1 and args.dist_backend == "gloo"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "fused PDHG iteration (K1 A^T y+primal/Halpern, K2 A x_bar+dual/Halpern)",
                     "bytes_per_launch": bytes_["iteration"], "seconds_per_launch": t_iter,
                     "peak_source": peak_src,
                     "frac_of_8TBs": achieved / 8000.0,
                     "bytes_per_launch_moved": bytes_["iteration_moved"],
                     "frac_moved": bytes_["iteration_moved"] / t_iter / 1e9 / peak,
                     "moved_note": "frac uses SURVEY 8d's byte model (24 nnz + 68 n + 52 m); frac_moved drops the "
                                   "16 B/column of lo/hi the primal kernel skips when every variable has the same "
                                   "bounds (GRIDLP_F_UNIFORM_BOUNDS, true for the reference generator's box)",
                     "request_bound": {
                         "requests_per_iteration": bytes_["requests"],
                         "ceiling_requests_per_s": GATHER_CEILING_PER_S,
                         "seconds_at_ceiling": bytes_["requests"] / GATHER_CEILING_PER_S,
                         "frac": bytes_["requests"] / GATHER_CEILING_PER_S / t_iter,
                         "note": "random FP64 gathers (2 nnz per iteration) cost one L1->L2 request each; "
                                 "ceiling measured by tools/microbench.cu"}},
        "kernels": {k: {"seconds": ktimes[k], "bytes": bytes_[k], "GB/s": bytes_[k] / ktimes[k] / 1e9}
                    for k in ktimes},
        "spmv": spmv,
        "extra_configs": extra or None,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` without torchrun: start N copies of this script
    with RANK / LOCAL_RANK / WORLD_SIZE / MASTER_* set (what torchrun
    exports), one per GPU; rank 0 prints the JSON line. With fewer GPUs than
    N the ranks share devices over gloo (an orchestration run: the line says
    ranks_share_gpus, and its time is not a scaling number)."""
    import socket
    import subprocess

    import torch

    ngpu = torch.cuda.device_count()
    share = ngpu < args.gpus
    if share:
        log(f"[bench] --gpus {args.gpus} on {ngpu} visible GPU(s): ranks share devices over gloo")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    procs = []
    for r in range(args.gpus):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(args.gpus),
                   LOCAL_WORLD_SIZE=str(args.gpus), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        if share:
            env["GRIDLP_SHARE_GPUS"] = "1"
        procs.append(subprocess.Popen([sys.executable, str(Path(__file__).resolve())] + sys.argv[1:], env=env))
    rcs = [p.wait() for p in procs]
    return max(rcs, key=abs)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=tuple(CONFIGS), default="cfg2")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-runs", type=int, default=5, help="complete solves timed for e2e (median reported)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-spmv", action="store_true", help="skip the SpMV-only comparison with cuSPARSE")
    ap.add_argument("--no-extra", action="store_true", help="skip the cfg1 latency / cfg3 extra keys")
    ap.add_argument("--light-row-max", type=int, default=None, help="EngineOptions.light_row_max override")
    ap.add_argument("--no-graphs", action="store_true", help="eager launches (the NCCL executor's path)")
    ap.add_argument("--no-device-loop", action="store_true",
                    help="time host-driven KKT intervals even where the device-side loop is on")
    ap.add_argument("--device-loop", action="store_true",
                    help="EngineOptions.device_loop=True (default: cluster-launched LPs only)")
    ap.add_argument("--natural-order", action="store_true", help="EngineOptions.sorted_order=False (layout order)")
    ap.add_argument("--column-bands", type=int, default=None, help="EngineOptions.column_bands (1 = off)")
    ap.add_argument("--band-mb", type=int, default=None, help="EngineOptions.band_bytes in MiB")
    ap.add_argument("--no-first-touch", action="store_true", help="EngineOptions.first_touch_cols=False")
    ap.add_argument("--graph-nccl", action="store_true", help="capture NCCL iterations in CUDA graphs (default now)")
    ap.add_argument("--value-codec", choices=("auto", "f64"), default=None,
                    help="EngineOptions.value_codec (lossless compact value storage; default auto)")
    ap.add_argument("--grid", default=None, help="RxC virtual grid on one GPU (load-balance study)")
    ap.add_argument("--permutation", default=None, help="SolverConfig.permutation override")
    ap.add_argument("--partitioning", default=None, help="SolverConfig.partitioning override")
    ap.add_argument("--dist-backend", choices=("nccl", "gloo"), default="nccl",
                    help="gloo lets several ranks share one GPU (orchestration check; timings are not NVLink)")
    ap.add_argument("--comm", choices=("nccl", "peer"), default="nccl",
                    help="multi-GPU vector sums: NCCL allreduce (default) or in-kernel peer-memory exchange")
    ap.add_argument("--force-nccl", action="store_true",
                    help="run the NCCL executor even at world size 1 (exercises the multi-GPU path on one GPU)")
    ap.add_argument("--tuning", action="append", default=[],
                    help="KEY=VALUE kernel knob (gridlp_set_tuning: sell_variant, chain_products)")
    ap.add_argument("--cpu-sample-iters", type=int, default=24)
    ap.add_argument("--ref-sample-iters", type=int, default=4)
    args = ap.parse_args()
    if args.warmup < 3:
        log("[bench] warmup raised to 3 (timing rules)")
        args.warmup = 3
    if "WORLD_SIZE" in os.environ:
        world_env = int(os.environ["WORLD_SIZE"])
        if world_env != args.gpus and not (args.gpus == 1 and world_env == 1):
            raise SystemExit(f"bench.py: WORLD_SIZE={world_env} but --gpus {args.gpus}: launch one rank per GPU")
    elif args.gpus > 1:
        # no launcher: spawn the N ranks ourselves (torchrun's environment)
        raise SystemExit(spawn_ranks(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if (args.impl == "ours" and world > 1 and args.dist_backend == "nccl"
            and os.environ.get("GRIDLP_SHARE_GPUS") == "1"):
        args.dist_backend = "gloo"
    if args.dist_backend == "gloo":
        # orchestration check on fewer GPUs than ranks: ranks share devices
        import torch

        local_rank %= max(torch.cuda.device_count(), 1)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    distributed = world > 1 or args.force_nccl
    if distributed:
        import torch
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        torch.cuda.set_device(local_rank)
        if args.dist_backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    if args.tuning:
        from paper_2601_07628_b200 import native

        for kv in args.tuning:
            k, v = kv.split("=", 1)
            native.load().set_tuning(k, int(v))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if distributed:
            import gc

            import torch.distributed as dist

            gc.collect()            # drop IPC-imported peer buffers before any producer exits
            dist.barrier()
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
