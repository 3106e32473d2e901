"""Summarise ncu captures for profiles/ (run here, on the CPU box).

    python scripts/ncu_summary.py full  <report.ncu-rep>   > profiles/<round>_ncu_<what>.md
    python scripts/ncu_summary.py launches <launches.csv>  > profiles/<round>_launches.md
    python scripts/ncu_summary.py traffic <report.ncu-rep> [key]  -> updates profiles/ncu_traffic.json
"""

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg", "SM cycles"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smem load wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem load bank conflicts"),
    ("smsp__sass_inst_executed_op_shared_ld.sum", "LDS instructions"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1/smem data-pipe wavefronts % of peak"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall: wait (fixed latency)"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall: math pipe throttle"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall: short scoreboard (smem)"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall: long scoreboard (global)"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall: barrier"),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "stall: not selected"),
    ("smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio", "stall: dispatch"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_bytes.sum", "L2 bytes"),
]


def raw(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def full(rep: str):
    hdr, units, rows = raw(rep)
    idx = {h: i for i, h in enumerate(hdr)}
    print(f"# ncu --set full summary: `{Path(rep).name}`\n")
    names = [r[idx["Kernel Name"]] for r in rows]
    print("| metric | unit | " + " | ".join(f"#{i} {n.split('(')[0].split('::')[-1]}" for i, n in enumerate(names)) + " |")
    print("|---|---|" + "---|" * len(names))
    for key, label in METRICS:
        if key not in idx:
            continue
        i = idx[key]
        print(f"| {label} (`{key}`) | {units[i]} | " + " | ".join(r[i] for r in rows) + " |")


def launches(path: str):
    txt = Path(path).read_text().splitlines()
    start = next(i for i, l in enumerate(txt) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(txt[start:]))))
    per = defaultdict(lambda: [0, 0.0])
    dram = defaultdict(lambda: [0, 0.0])  # kernel -> [launches, read + write bytes]
    unit = ""
    for r in rows:
        name = r["Kernel Name"].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        metric = r.get("Metric Name", "gpu__time_duration.sum")
        v = float(r["Metric Value"].replace(",", ""))
        if metric == "gpu__time_duration.sum":
            unit = r.get("Metric Unit", "")
            per[name][0] += 1
            per[name][1] += v
        elif metric in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            dram[name][1] += v
            if metric == "dram__bytes_read.sum":
                dram[name][0] += 1
    total = sum(v for _, v in per.values())
    print(f"# launch list (`gpu__time_duration.sum`, cold-cache, serialised): `{Path(path).name}`\n")
    cols = "| kernel | launches | total (%s) | share |" % unit + (" DRAM bytes / launch |" if dram else "")
    print(cols)
    print("|---|---|---|---|" + ("---|" if dram else ""))
    for name, (n, v) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        extra = ""
        if dram:
            dn, db = dram.get(name, [0, 0.0])
            extra = f" {db / dn:,.0f} |" if dn else " — |"
        print(f"| {name} | {n} | {v:,.0f} | {v / total:.1%} |{extra}")


def traffic(rep: str, key: str = "energy_kernel_both"):
    hdr, units, rows = raw(rep)
    idx = {h: i for i, h in enumerate(hdr)}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    r = rows[0]
    b = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        b += float(r[idx[k]]) * scale[units[idx[k]]]
    p = Path(__file__).resolve().parents[1] / "profiles" / "ncu_traffic.json"
    d = json.loads(p.read_text()) if p.exists() else {}
    d[key] = b
    d["_source"] = f"{Path(rep).name}: dram__bytes_read.sum + dram__bytes_write.sum of the first captured launch"
    p.write_text(json.dumps(d, indent=2) + "\n")
    print(key, b)


if __name__ == "__main__":
    {"full": full, "launches": launches, "traffic": traffic}[sys.argv[1]](*sys.argv[2:])
