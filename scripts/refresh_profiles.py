"""Copy the evidence of one `scripts/gpu_round.sh` run from gpurun_out/ into
profiles/ (round prefix, default r02) and regenerate the derived summaries:
    python scripts/refresh_profiles.py [r02]
bench lines, reference arms, ncu --set full summaries of every stream-kernel
variant and of the CodedArray kernels, per-line pipe splits, the launch table,
GPU test / smoke / sanitizer logs (host frames dropped) and ncu_traffic.json."""
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
r = sys.argv[1] if len(sys.argv) > 1 else "r02"


def run(*cmd, out=None):
    res = subprocess.run([sys.executable, *cmd], capture_output=True, text=True, cwd=ROOT, timeout=900)
    if res.returncode != 0:
        raise SystemExit(res.stderr)
    if out:
        with open(out, "w") as f:
            f.write(res.stdout)


for w in ("c3", "c2", "c1", "c5", "c5rel", "c4"):
    shutil.copy(os.path.join(OUT, f"bench_{w}.json"), os.path.join(PROF, f"{r}_bench_{w}.json"))
for w in ("c3", "c2", "c4"):
    shutil.copy(os.path.join(OUT, f"bench_ref_{w}.json"), os.path.join(PROF, f"{r}_bench_reference_{w}.json"))
for w in ("c3", "c2", "c5", "c5rel"):
    run("scripts/ncu_summary.py", f"gpurun_out/prof_{w}_full.ncu-rep", f"profiles/{r}_ncu_{w}_stream.md")
run("scripts/ncu_summary.py", "gpurun_out/prof_c3_coded.ncu-rep", f"profiles/{r}_ncu_c3_coded.md")
for k, name in (("k_encode4k", "encode"), ("k_decode4k", "decode")):
    run("scripts/ncu_pipes.py", "gpurun_out/prof_c3_full.ncu-rep", k, "40", out=f"profiles/{r}_ncu_c3_{name}_pipes.txt")
shutil.copy(os.path.join(OUT, "launches_c3.csv"), os.path.join(PROF, f"{r}_launches_c3.csv"))
run("scripts/launch_table.py", f"profiles/{r}_launches_c3.csv", out=f"profiles/{r}_launches_c3.md")
for f in ("pytest_gpu", "smoke", "memcheck_gpu", "racecheck_gpu"):
    with open(os.path.join(OUT, f + ".log")) as src, open(os.path.join(PROF, f"{r}_{f}.log"), "w") as dst:
        dst.writelines(line for line in src if "Host Frame" not in line)


def dram(md):
    """DRAM bytes (read + write) per kernel kind from an ncu_summary.py report."""
    out, cur = {}, None
    for line in open(md):
        if line.startswith("## "):
            n = line[3:]
            cur = ("encode" if "encode4k" in n else "decode" if "decode4k" in n
                   else "quantize" if "quant" in n.lower() else "reconstruct" if "recon" in n.lower() else None)
        m = re.match(r"\| dram__bytes_(read|write)\.sum \| ([\d.]+) \| (\w+)", line)
        if m and cur:
            mul = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[m.group(3)]
            out[cur] = out.get(cur, 0) + round(float(m.group(2)) * mul)
    return out


path = os.path.join(PROF, "ncu_traffic.json")
traffic = json.load(open(path))
for w in ("c3", "c2", "c5", "c5rel"):
    d = dram(os.path.join(PROF, f"{r}_ncu_{w}_stream.md"))
    traffic.setdefault(w, {}).update({k: d[k] for k in ("encode", "decode")})
    traffic[w]["source"] = (f"profiles/{r}_ncu_{w}_stream.md (ncu --set full, dram__bytes_read.sum + "
                            "dram__bytes_write.sum per launch)")
traffic["c3"].update({k: v for k, v in dram(os.path.join(PROF, f"{r}_ncu_c3_coded.md")).items()
                      if k in ("quantize", "reconstruct")})
json.dump(traffic, open(path, "w"), indent=1)
print(json.dumps(traffic, indent=1))
