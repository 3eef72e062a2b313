"""Interleaved A/B of the device-side main loop (EngineOptions.device_loop)
on complete solves through the public path (api._solve with engine
overrides): cfg1 (tiny, cluster launch) and cfg2 (kernel-per-product chunks
with programmatic chaining), wall time to 1e-4, alternated run by run."""

import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2601_07628_b200 import GeneratorSpec, SolverConfig, generate  # noqa: E402
from paper_2601_07628_b200.api import _solve  # noqa: E402


def main():
    out = {}
    for name, reps in (("cfg1", 8), ("cfg2", 4)):
        p = generate(GeneratorSpec(**bench.CONFIGS[name])) if name == "cfg1" else bench.make_problem(name)
        cfg = SolverConfig(tolerance=1e-4, seed=0)
        res = {True: [], False: []}
        for v in (True, False):
            _solve(p, cfg, engine_overrides={"device_loop": v})     # warm
        for r in range(reps):
            for v in ((True, False) if r % 2 == 0 else (False, True)):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                s = _solve(p, cfg, engine_overrides={"device_loop": v})
                res[v].append(time.perf_counter() - t0)
                assert s.status == "optimal"
        out[name] = {("device_loop" if v else "host_loop"): {"median_s": statistics.median(x),
                                                             "all": [round(y, 4) for y in x]}
                     for v, x in res.items()}
        out[name]["iterations"] = s.iterations
    print(json.dumps(out))


if __name__ == "__main__":
    main()
