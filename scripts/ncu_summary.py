"""Summarise an ncu --set full report (.ncu-rep) into profiles/: key metrics,
DRAM traffic per launch, stall reasons, hottest source lines.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r01_encode4k.md
"""

import csv
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
    "launch__block_size", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
    "sm__warps_active.avg.per_cycle_active", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]
STALLS = ["barrier", "short_scoreboard", "long_scoreboard", "wait", "math_pipe_throttle",
          "no_instruction", "branch_resolving", "not_selected", "mio_throttle", "lg_throttle",
          "sleeping"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2:]


def lines(rep, top=20):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    res, tot, fname = [], 0, None
    for r in csv.reader(out.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No") or r[0] == "" or len(r) < 8:
            continue
        try:
            ie = int(r[7])
        except ValueError:
            continue
        res.append((ie, fname, r[0], r[1].strip()[:100]))
        tot += ie
    res.sort(reverse=True)
    return tot, res[:top]


def main(rep, out_path):
    h, units, rows = raw(rep)
    with open(out_path, "w") as f:
        for v in rows:
            name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
            f.write(f"## {name}\n\nsource report: `{rep}`\n\n| metric | value | unit |\n|---|---|---|\n")
            for k in KEYS:
                if k in h:
                    i = h.index(k)
                    f.write(f"| {k} | {v[i]} | {units[i]} |\n")
            f.write("\n| stall (per issue) | value |\n|---|---|\n")
            for s in STALLS:
                k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
                if k in h:
                    f.write(f"| {s} | {v[h.index(k)]} |\n")
        tot, top = lines(rep)
        f.write(f"\n### hottest source lines (share of {tot} executed warp instructions)\n\n")
        for ie, fn, ln, src in top:
            f.write(f"- {100 * ie / max(tot, 1):5.1f}%  `{fn}:{ln}`  `{src}`\n")
    print(out_path)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
