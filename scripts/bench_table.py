"""Markdown table of bench lines: python scripts/bench_table.py profiles/r02_bench_*.json"""
import json
import sys

print("| workload | encode µs (GB/s, frac) | decode µs (GB/s, frac) | `value` GB/s | e2e GB/s | CPU (threads) GB/s | CodedArray quantize / reconstruct frac |")
print("|---|---|---|---|---|---|---|")
for f in sys.argv[1:]:
    d = None
    for line in open(f):
        if line.startswith("{"):
            d = json.loads(line)
    if d is None or "kernels" not in d:
        continue
    k = d["kernels"]
    e, dc = k["encode"], k["decode"]
    cs = d.get("coded_stage") or {}
    q = cs.get("quantize", {}).get("frac")
    r = cs.get("reconstruct", {}).get("frac")
    cpu = d.get("cpu_baseline") or {}
    e2e = (d.get("e2e") or {}).get("value")
    name = d["config"]["workload"].split(":")[0]
    print(f"| {name} | {e['ms']*1e3:.0f} ({e['gbs']:.0f}, {e['frac']:.3f}) | {dc['ms']*1e3:.0f} ({dc['gbs']:.0f}, {dc['frac']:.3f}) "
          f"| {d['value']:.0f} | {e2e if e2e is None else round(e2e, 1)} | {cpu.get('value', 0):.2f} ({cpu.get('cores')}) "
          f"| {q if q is None else round(q, 2)} / {r if r is None else round(r, 2)} |")
