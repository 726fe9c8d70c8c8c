"""Source lines ranked by shared-memory wavefronts (and the excess over ideal, i.e.
bank conflicts) for one kernel of an ncu report.
    python scripts/ncu_smem.py REP KERNEL_REGEX [top]"""
import csv, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
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
    g = lambda k: int(float(r[hdr.index(k)] or 0))
    rows.append((g("L1 Wavefronts Shared"), g("L1 Wavefronts Shared Excessive"), g("L1 Wavefronts Shared Ideal"),
                 fname, ln, r[1].strip()[:90]))
tw = sum(x[0] for x in rows) or 1; te = sum(x[1] for x in rows)
print(f"shared wavefronts {tw}, excessive {te} ({100 * te / tw:.1f}%)")
for w, e, i, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100 * w / tw:5.1f}% wf  excess {e:>11d} ({e / max(i, 1):4.2f}x ideal)  {f}:{ln}  {src}")
