"""Top source lines by warp-stall samples (and their instruction share) for one kernel.
    python scripts/ncu_stalls.py REP KERNEL_REGEX [top]"""
import csv, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
hdr = None; fname = None; rows = []
for r in csv.reader(out.splitlines()):
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or r[0] == "Function Name" or r[2] != "-": continue
    try: ln = int(r[0])
    except ValueError: continue
    ss = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    ie = int(r[hdr.index("Instructions Executed")] or 0)
    rows.append((ss, ie, fname, ln, r[1].strip()[:100]))
ts = sum(x[0] for x in rows) or 1; ti = sum(x[1] for x in rows) or 1
rows.sort(reverse=True)
print(f"stall samples {ts}, warp instructions {ti}")
for ss, ie, f, ln, src in rows[:top]:
    print(f"{100*ss/ts:5.1f}% stall {100*ie/ti:5.1f}% inst  {f}:{ln}  {src}")
