"""Executed warp instructions per tile, split by code region, for the two
stream kernels of one ncu --import-source report (the report's source lines
must match the regions below, i.e. the stream_fast.cu it was built from):
    python scripts/instr_budget.py REP SOURCE.cu TILES
TILES = tiles (encoder) / blocks (decoder) per launch; 8 warps per tile.
Regions are located by marker lines in SOURCE.cu, so they follow edits."""
import csv
import subprocess
import sys
from collections import defaultdict

rep, src, tiles = sys.argv[1], sys.argv[2], int(sys.argv[3])
lines = open(src).read().split("\n")


def at(marker, start=0):
    for i in range(start, len(lines)):
        if marker in lines[i]:
            return i + 1
    raise SystemExit("marker not found: " + marker)


enc0 = at("k_encode4k_sp(Enc4kArgs a, Consts<T> k0) {")
dec0 = at("k_decode4k_sp(DecodeCfg d, const uint8_t *__restrict__ region,")
ENC = [
    ("tile placement (place_tile)", at("void place_tile("), enc0 - 1),
    ("per-tile state: count loads and sums, FIFO, ring", enc0, at("auto row = [&](int r, auto full", enc0) - 1),
    ("general quantize row (partial tiles, slow rows)", at("auto row = [&](int r, auto full", enc0),
     at("auto fast_row = ", enc0) - 1),
    ("fast quantize row (binary32 ABS/NOA)", at("auto fast_row = ", enc0),
     at("// the earlier tiles' byte counts are loaded half way", enc0) - 1),
    ("quantize loop, tile head, slow-row redo", at("// the earlier tiles' byte counts are loaded half way", enc0),
     at("const uint4 lw = *reinterpret_cast", enc0) - 1),
    ("byte-count scan, barrier (AB), warp prefix", at("const uint4 lw = *reinterpret_cast", enc0),
     at("// ---- ring space for this tile's image", enc0) - 1),
    ("ring allocation, FIFO entry", at("// ---- ring space for this tile's image", enc0),
     at("// ---- this tile's image: bitmap words", enc0) - 1),
    ("emission (bitmap, quad / per-value runs, run joins, barrier C)", at("// ---- this tile's image: bitmap words", enc0),
     at("// the FIFO entry written above is visible after barrier (C)", enc0) - 1),
    ("FIFO pop, placement after C, next tile", at("// the FIFO entry written above is visible after barrier (C)", enc0),
     at("// images still waiting in the ring", enc0) - 1),
    ("ring drain, trigger counters", at("// images still waiting in the ring", enc0), dec0 - 200),
]
dr = at("auto rows = [&](auto DF, auto FB)", dec0)
DEC = [
    ("block head: table build, geometry, bulk copies", dec0, at("if (size_ok) {", dec0) - 1),
    ("terminator count, scan, run-start scatter", at("if (size_ok) {", dec0),
     at("bad = __syncthreads_or(bad);                           // (3)", dec0) - 1),
    ("parse setup, run starts", at("bad = __syncthreads_or(bad);                           // (3)", dec0),
     at("if (__all_sync(0xFFFFFFFFu, fast || !acth)) {", dr) - 1),
    ("fast 4-value half (window, table, reconstruct, store)", at("if (__all_sync(0xFFFFFFFFu, fast || !acth)) {", dr),
     at("} else if (acth) {", dr) - 1),
    ("general 4-value half (per-value parse)", at("} else if (acth) {", dr), at("auto rows64 = ", dr) - 1),
    ("binary64 rows, block tail", at("auto rows64 = ", dr), len(lines)),
]
# the window loads / table lookup of the fast half sit just before its vote: count
# them with the fast half
fast_pre = at("const uint32_t sh = pa << 3;", dr) if any("const uint32_t sh = pa << 3;" in l for l in lines) else None


def per_line(kre):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass", "-k",
                          "regex:" + kre], capture_output=True, text=True).stdout
    hdr = None; fname = None; cur = None; seen = set(); acc = defaultdict(int)
    for r in csv.reader(out.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]; continue
        if r[0] == "Line No":
            hdr = r; continue
        if hdr is None or r[0] == "Function Name":
            continue
        if r[0]:
            try:
                cur = (fname, int(r[0]))
            except ValueError:
                cur = None
            continue
        if not r[2].startswith("0x") or r[2] in seen:
            continue
        seen.add(r[2])   # each SASS address once (the CSV repeats rows)
        v = r[hdr.index("Instructions Executed")]
        acc[cur] += int(v) if v.isdigit() else 0
    return acc


def table(name, kre, regions):
    acc = per_line(kre)
    tot = sum(acc.values())
    reg = defaultdict(int)
    for (f, ln), n in ((k, v) for k, v in acc.items() if k):
        if f != "stream_fast.cu":
            reg["inlined headers (shuffles, votes, barriers, helpers)"] += n; continue
        if fast_pre and name == "decoder" and fast_pre - 3 <= ln < fast_pre + 12:
            reg["fast 4-value half (window, table, reconstruct, store)"] += n; continue
        for rn, a, b in regions:
            if a <= ln <= b:
                reg[rn] += n; break
        else:
            reg["other lines (warp scan, shared-load helpers, kernel prologue)"] += n
    print(f"\n### {name}: {tot / (tiles * 8):.0f} warp instructions per warp per tile\n")
    print("| region | per warp-tile | share |\n|---|---|---|")
    for rn, n in sorted(reg.items(), key=lambda x: -x[1]):
        print(f"| {rn} | {n / (tiles * 8):.0f} | {100 * n / tot:.1f} % |")


table("encoder", "k_encode4k", ENC)
table("decoder", "k_decode4k", DEC)
