"""Per-source-line instruction counts and stall samples of one kernel in an ncu report.
    python scripts/ncu_lines.py REP KERNEL_REGEX [top]"""
import csv, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
fname, res, tot, stot = None, [], 0, 0
hdr = None
for r in csv.reader(out.splitlines()):
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if r[0] == "Function Name" or hdr is None: continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    # cuda lines have an empty Address column
    if r[2] != "-": continue
    try:
        ie = int(r[hdr.index("Instructions Executed")] or 0); ss = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except (ValueError, IndexError):
        continue
    if ie == 0 and ss == 0: continue
    res.append((ie, ss, fname, ln, r[1].strip()[:110])); tot += ie; stot += ss
res.sort(reverse=True)
print(f"total warp instructions {tot}, stall samples {stot}")
for ie, ss, fn, ln, src in res[:top]:
    print(f"{100*ie/tot:5.1f}% inst {100*ss/max(stot,1):5.1f}% stall  {fn}:{ln}  {src}")
