"""Summarise an `ncu --set full` capture (.ncu-rep) into a markdown table of
the counters DESIGN.md argues from, and optionally update
profiles/traffic.json (DRAM bytes per fused iteration, the bench's
`roofline.traffic`).

    python tools/ncu_summary.py gpurun_out/prof_sell32.ncu-rep profiles/r1/ncu_sell32_full.md \
        [--traffic-config cfg2]
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
from pathlib import Path

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__bytes_read.sum.per_second", "DRAM read rate"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory SOL %"),
    ("l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed", "L1->L2 request port busy %"),
    ("lts__t_tag_requests.avg.pct_of_peak_sustained_elapsed", "L2 tag lookups %"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 data-pipe wavefronts %"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "global load requests"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "global load sectors"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard /issue"),
    ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "stall lg_throttle /issue"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "stall mio_throttle /issue"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def raw(rep: Path):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep", type=Path)
    ap.add_argument("out", type=Path)
    ap.add_argument("--traffic-config", default=None)
    a = ap.parse_args()
    hdr, units, rows = raw(a.rep)
    col = {h: i for i, h in enumerate(hdr)}
    names = [r[col["Kernel Name"]] for r in rows]
    short = [n.split("(")[0].replace("void <unnamed>::", "").replace("<unnamed>::", "")[:60] for n in names]
    lines = [f"# ncu --set full summary: `{a.rep.name}`", "",
             "| metric | " + " | ".join(f"`{s}`" for s in short) + " |",
             "|---|" + "---|" * len(rows)]
    for key, label in METRICS:
        if key not in col:
            continue
        i = col[key]
        lines.append(f"| {label} ({units[i]}) | " + " | ".join(r[i] for r in rows) + " |")
    a.out.write_text("\n".join(lines) + "\n")
    print("\n".join(lines))
    if a.traffic_config:
        def to_bytes(i, r):
            u = units[i].lower()
            mult = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(u, 1)
            return float(r[i].replace(",", "")) * mult
        tot = sum(to_bytes(col["dram__bytes_read.sum"], r) + to_bytes(col["dram__bytes_write.sum"], r) for r in rows)
        tf = Path(__file__).resolve().parents[1] / "profiles" / "traffic.json"
        d = json.loads(tf.read_text()) if tf.exists() else {}
        d[a.traffic_config] = {"bytes_per_iteration": tot, "kernels": short, "source": str(a.out.name),
                               "note": "sum over the captured K1+K2 launches; ncu flushes L2 between "
                                       "replay passes, so the gathered vectors start cold"}
        tf.write_text(json.dumps(d, indent=1) + "\n")
        print(f"traffic {a.traffic_config}: {tot / 1e6:.1f} MB per iteration")


if __name__ == "__main__":
    main()
