"""Host-side profile of one end-to-end solve (bench.py's e2e leg) under
cProfile: where the non-kernel part of time-to-tolerance goes.

    python tools/profile_e2e.py [--config cfg2] [--out gpurun_out/e2e_profile.txt]
"""

import argparse
import cProfile
import io
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2601_07628_b200 import SolverConfig, solve  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--out", default="gpurun_out/e2e_profile.txt")
    ap.add_argument("--sweep", action="store_true", help="with / without the host-scalar thread first")
    args = ap.parse_args()
    p = bench.make_problem(args.config)
    cfg = SolverConfig(tolerance=1e-4, seed=0)
    solve(p, cfg)                                   # warm: module load, allocator, graphs
    torch.cuda.synchronize()
    walls = []
    for _ in range(2):
        t0 = time.perf_counter()
        r = solve(p, cfg)
        torch.cuda.synchronize()
        walls.append(time.perf_counter() - t0)
    if args.sweep:
        from paper_2601_07628_b200 import api

        for overlap in (True, False):
            api.HOST_OVERLAP = overlap
            ws = []
            for _ in range(3):
                t0 = time.perf_counter()
                solve(p, cfg)
                torch.cuda.synchronize()
                ws.append(time.perf_counter() - t0)
            print(f"host overlap={overlap}: walls {[round(w, 4) for w in ws]}", flush=True)
        api.HOST_OVERLAP = True
    prof = cProfile.Profile()
    t0 = time.perf_counter()
    prof.enable()
    r = solve(p, cfg)
    torch.cuda.synchronize()
    prof.disable()
    wall = time.perf_counter() - t0
    s = io.StringIO()
    s.write(f"walls (unprofiled) {walls}  profiled {wall:.4f}s  status {r.status} it {r.iterations}\n")
    s.write("timings " + repr({k: round(v, 5) for k, v in r.timings.items() if k.endswith('_s')}) + "\n")
    st = pstats.Stats(prof, stream=s)
    st.sort_stats("cumulative").print_stats(45)
    st.sort_stats("tottime").print_stats(30)
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out, "w") as f:
        f.write(s.getvalue())
    print(s.getvalue()[:6000])


if __name__ == "__main__":
    main()
