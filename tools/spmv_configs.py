"""SpMV-only comparison (ours vs cuSPARSE through torch.sparse, FP64) on the
device-generated §8f configs: bench.spmv_compare on each instance's own CSR.

    python tools/spmv_configs.py cfg3s cfg4s cfg3 cfg4 > gpurun_out/spmv_configs.jsonl
"""

import gc
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    for name in sys.argv[1:]:
        p = bench.make_problem(name)
        t0 = time.perf_counter()
        r = bench.spmv_compare(p, dev)
        r["config"] = name
        r["wall_s"] = time.perf_counter() - t0
        print(json.dumps(r), flush=True)
        del p
        gc.collect()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
