"""Executed SASS instructions of one kernel split by issue pipe (alu / fma / xu /
lsu / other), per source line, from an ncu --import-source report.
    python scripts/ncu_pipes.py REP KERNEL_REGEX [top]"""
import csv, re, subprocess, sys
from collections import defaultdict
rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
ALU = {"IADD3", "LOP3", "SHF", "PRMT", "FMNMX", "ISETP", "FSETP", "SEL", "FSEL", "LEA", "IABS", "PLOP3",
       "P2R", "R2P", "VIADD", "IMNMX", "VIMNMX", "CS2R", "BMSK", "IADD", "MOV", "SGXT", "BREV", "VIADDMNMX", "LOP"}
FMA = {"FFMA", "FMUL", "FADD", "IMAD", "HFMA2", "IDP", "DFMA", "DMUL", "DADD", "IMUL"}
XU = {"FLO", "POPC", "MUFU", "I2F", "F2I", "FRND", "I2FP", "F2IP", "F2F", "I2I"}
LSU = {"LDS", "STS", "LDG", "STG", "LD", "ST", "ATOMS", "ATOMG", "ATOM", "RED", "SHFL", "LDSM", "REDUX", "VOTE",
       "LDC", "BAR", "SYNCS", "MEMBAR", "UBLKCP", "UTMALDG"}
def pipe(op):
    b = op.split(".")[0]
    if b.startswith("U") and b not in ("UBLKCP", "UTMALDG"): return "uniform"
    for name, s in (("alu", ALU), ("fma", FMA), ("xu", XU), ("lsu", LSU)):
        if b in s: return name
    return "other"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
hdr = None; fname = None; cur = None
per = defaultdict(lambda: defaultdict(int)); tot = defaultdict(int); src = {}
for r in csv.reader(out.splitlines()):
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or r[0] == "Function Name": continue
    if r[0]:                             # a source line: the SASS rows after it belong to it
        try: cur = (fname, int(r[0])); src[cur] = r[1].strip()[:80]
        except ValueError: cur = None
        continue
    if not r[2].startswith("0x"): continue
    v = r[hdr.index("Instructions Executed")]
    ie = int(v) if v.isdigit() else 0
    sass = r[3].strip()
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_.]+)", sass)
    if not m or cur is None: continue
    p = pipe(m.group(2))
    per[cur][p] += ie; tot[p] += ie
T = sum(tot.values()) or 1
print("total warp instructions", T, {k: f"{100 * v / T:.1f}%" for k, v in sorted(tot.items())})
for key, d in sorted(per.items(), key=lambda kv: -kv[1].get("alu", 0))[:top]:
    s = sum(d.values())
    print(f"alu {100 * d.get('alu', 0) / tot['alu']:5.1f}%  all {100 * s / T:5.1f}%  "
          f"(alu {d.get('alu',0)/1e6:7.1f}M fma {d.get('fma',0)/1e6:6.1f}M xu {d.get('xu',0)/1e6:5.1f}M lsu {d.get('lsu',0)/1e6:5.1f}M)  "
          f"{key[0]}:{key[1]}  {src.get(key, '')}")
