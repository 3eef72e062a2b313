"""The bench's SpMV-only leg alone (cfg2 by default): ours vs torch.sparse vs
cusparseSpMV CSR_ALG1 / ALG2 — run under ncu to keep the library kernels'
names in a launch list (profiles/r2/launches_spmv_cusparse.csv).

    python tools/spmv_compare_only.py [--config cfg2] [--reps 3]
"""

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch

    p = bench.make_problem(args.config)
    out = bench.spmv_compare(p, torch.device("cuda", 0), reps=args.reps)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
