"""Markdown table of an ncu launch list (--metrics gpu__time_duration.sum --csv):
    python scripts/launch_table.py launches.csv  -> kernel, launches, mean us"""
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
acc = collections.OrderedDict()
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    v = v / 1000.0 if r[ui] in ("ns", "nsecond") else v * 1000.0 if r[ui] in ("ms", "msecond") else v
    name = r[ki].split("(")[0]
    acc.setdefault(name, []).append(v)
print("| kernel | launches | mean us |\n|---|---|---|")
for k, v in acc.items():
    print(f"| `{k}` | {len(v)} | {sum(v) / len(v):.1f} |")
