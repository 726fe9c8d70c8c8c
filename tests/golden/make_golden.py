"""Generate the golden fixtures by running the REFERENCE implementation.

Run once in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py [--full-sweeps]

Everything written here is reference OUTPUT (digests, codes, tallies,
exception classes) on seeded inputs; no reference source is copied.  The
fixtures pin the oracle (tests/test_oracle.py) and the CUDA path
(tests/test_gpu_*.py) on machines where the reference is absent.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import gebq  # noqa: E402  (the reference, via PYTHONPATH)
import importlib  # noqa: E402
from gebq import _kernels, container, pipeline, quantizers  # noqa: E402

sweep = importlib.import_module("gebq.sweep")
verify = importlib.import_module("gebq.verify")
from gebq.quantizers import ABS, NOA, REL, QuantConfig  # noqa: E402

from paper_2407_15037_b200 import workloads  # noqa: E402  (input recipes only)

WORKERS = 8


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def cbits(v, width):
    if v is None:
        return None
    return int(np.float32(v).view(np.uint32)) if width == 32 else int(np.float64(v).view(np.uint64))


def derived_record(cfg: QuantConfig) -> dict:
    d = cfg.derived
    w = cfg.width
    return {k: cbits(getattr(d, k), w) for k in ("thr", "eb_eff", "eb2", "inv_eb2", "op_eps", "w")}


# ---------------------------------------------------------------------------

def gen_constants():
    grid = []
    for width in (32, 64):
        for eb in (1e-1, 1e-2, 1e-3, 1e-4, 1e-5, 1e-7, 1e-9, 0.5, 1.0, 3.0, 1e-30, 1e-300, 1e30):
            for mode in (ABS, REL):
                grid.append((mode, eb, width, None))
            for r in (1.0, 14.0, 1e10, 1e-10, 0.0, float("inf")):
                grid.append((NOA, eb, width, r))
    out = []
    for mode, eb, width, r in grid:
        cfg = QuantConfig(mode=mode, eb=eb, width=width, value_range=r)
        rec = {"mode": mode, "eb": eb, "width": width, "value_range": r}
        rec.update(derived_record(cfg))
        rec["header_bits"] = cfg.derived.header_bits
        out.append(rec)
    return out


def mixed_bits(width, n, seed):
    rng = np.random.default_rng(seed)
    if width == 32:
        bits = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
        specials = np.array([0, 1 << 31, 0x7F800000, 0xFF800000, 0x7FC00000, 1, 0x80000001,
                             0x7F7FFFFF, 0x7F7FFFA1, 0x7F7FFFA0, 0x00800000, 0x80800000,
                             0x4E7FFFFF, 0x4E800000, 0x3F800000, 0xBF800000], dtype=np.uint32)
    else:
        bits = rng.integers(0, 2**64, n, dtype=np.uint64)
        specials = np.array([0, 1 << 63, 0x7FF0000000000000, 0xFFF0000000000000,
                             0x7FF8000000000000, 1, 0x7FEFFFFFFFFFFFFF, 0x0010000000000000,
                             0x3FF0000000000000, 0xBFF0000000000000], dtype=np.uint64)
    return np.concatenate([specials, bits])


KERNEL_CASES = [
    (ABS, 1e-3, 32, None), (ABS, 0.5, 32, None), (ABS, 1e-7, 32, None),
    (REL, 1e-3, 32, None), (REL, 1.0, 32, None), (REL, 1e-2, 32, None), (REL, 1e-5, 32, None),
    (NOA, 1e-2, 32, 10.0), (NOA, 1e-3, 32, 1e-10),
    (ABS, 1e-3, 64, None), (ABS, 1e-9, 64, None), (REL, 1e-3, 64, None), (REL, 1e-1, 64, None),
    (NOA, 1e-4, 64, 14.0),
]


def gen_kernels():
    """Reference compress_coded on mixed corpora (+ a smooth slice) per case, safe and unsafe."""
    arrays = {}
    meta = []
    for ci, (mode, eb, width, vr) in enumerate(KERNEL_CASES):
        bits = mixed_bits(width, 2500, 1000 + ci)
        ft = np.float32 if width == 32 else np.float64
        # add a smooth slice so most values quantize (the bin/double-check paths)
        sm = (np.sin(np.linspace(0, 40, 1500)) * 5.0).astype(ft).view(bits.dtype)
        bits = np.concatenate([bits, sm])
        for unsafe in (False, True):
            cfg = QuantConfig(mode=mode, eb=eb, width=width, value_range=vr,
                              unsafe_no_double_check=unsafe)
            coded, cfg2, stats = pipeline.compress_coded(bits.view(ft), cfg, workers=1)
            key = f"c{ci}_{int(unsafe)}"
            if not unsafe:
                arrays[f"c{ci}_bits"] = bits
                arrays[key + "_recon"] = pipeline.decompress_to_array(
                    pipeline.compress(bits.view(ft), cfg, workers=1)[0], workers=1).view(bits.dtype)
            arrays[key + "_codes"] = coded.codes
            arrays[key + "_lossless"] = coded.lossless
            meta.append({"key": key, "mode": mode, "eb": eb, "width": width, "value_range": vr,
                         "unsafe": unsafe, "triggers": stats.triggers,
                         "derived": derived_record(cfg2)})
    return arrays, meta


def gen_reconstruct():
    """Adversarial raw (code, flag) pairs through reference reconstruct_* (incl. corrupt codes)."""
    arrays = {}
    meta = []
    rng = np.random.default_rng(77)
    cases = [(ABS, 32, np.float32(1.0)), (ABS, 32, np.float32(2e-3)), (ABS, 32, np.float32(3e38)),
             (REL, 32, np.float32(0.5)), (REL, 32, np.float32(1.0)),
             (REL, 32, np.float32(0.019920)), (REL, 32, np.float32(2.0)),
             (ABS, 64, np.float64(2e-3)), (ABS, 64, np.float64(1e300)),
             (REL, 64, np.float64(0.5)), (REL, 64, np.float64(1.0)),
             (REL, 64, np.float64(2.88e-3))]
    for ci, (mode, width, d) in enumerate(cases):
        n = 6000
        if width == 32:
            codes = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
            small = rng.integers(0, 4096, n // 2).astype(np.uint32)
            edge = np.array([0, 1, 2, 3, 514, 257 << 1, (0xFFFFFFFF), 0xFFFFFFFE, 1 << 31,
                             (1 << 31) - 1, 255, 254, 256, 253], dtype=np.uint32)
        else:
            codes = rng.integers(0, 2**64, n, dtype=np.uint64)
            small = rng.integers(0, 1 << 14, n // 2).astype(np.uint64)
            edge = np.array([0, 1, 2, 3, 2**64 - 1, 2**64 - 2, 1 << 63, (1 << 63) - 1, 4094,
                             4093, 4095, 4096, 2047 * 4], dtype=np.uint64)
        codes = np.concatenate([edge, small, codes])
        lossless = rng.random(len(codes)) < 0.2
        lossless[: len(edge) + len(small)] = False
        out = np.empty(len(codes), dtype=np.float32 if width == 32 else np.float64)
        ob = out.view(codes.dtype)
        fn = getattr(_kernels, f"reconstruct_{mode}{width}")
        fn(codes, lossless, ob, out, d)
        key = f"r{ci}"
        arrays[key + "_codes"] = codes
        arrays[key + "_lossless"] = lossless
        arrays[key + "_out"] = ob.copy()
        meta.append({"key": key, "mode": mode, "width": width, "derived_bits": cbits(d, width)})
    return arrays, meta


def gen_streams():
    """Stream digests: block-size grid, all modes/widths, worked example, empty input."""
    out = []
    for width in (32, 64):
        ft = np.float32 if width == 32 else np.float64
        bits = mixed_bits(width, 20000, 4242 + width)
        vals = np.concatenate([bits.view(ft), (np.cos(np.linspace(0, 90, 30000)) * 3).astype(ft)])
        for mode, eb, vr in ((ABS, 1e-3, None), (REL, 1e-3, None), (NOA, 1e-3, None),
                             (NOA, 1e-2, 2.5), (ABS, 1e-5, None), (REL, 1e-1, None)):
            for bs in (1, 2, 7, 64, 128, 192, 1000, 4095, 4096, 4097, 8192, 10000, 65536, 100000):
                for unsafe in (False, True) if bs == 4096 else (False,):
                    cfg = QuantConfig(mode=mode, eb=eb, width=width, block_size=bs,
                                      value_range=vr, unsafe_no_double_check=unsafe)
                    s, st = pipeline.compress(vals, cfg, workers=WORKERS)
                    out.append({"width": width, "mode": mode, "eb": eb, "value_range": vr,
                                "block_size": bs, "unsafe": unsafe, "n": len(vals),
                                "seed": 4242 + width, "sha256": sha(s), "bytes": len(s),
                                "triggers": st.triggers})
    # FORMAT.md worked example
    s, _ = pipeline.compress(np.array([3.2, np.nan, -0.75], dtype=np.float32),
                             QuantConfig(mode=ABS, eb=0.5))
    example = s.hex()
    empty = pipeline.compress(np.array([], dtype=np.float32), QuantConfig(mode=ABS, eb=1e-3))[0].hex()
    return out, example, empty


def _mutate_cases():
    rng = np.random.default_rng(2024)
    cases = []
    for name, mode, width, n, bs in (("rel32", REL, 32, 300, 128), ("abs64", ABS, 64, 500, 64),
                                     ("abs32", ABS, 32, 5000, 4096), ("rel64", REL, 64, 700, 100)):
        ft = np.float32 if width == 32 else np.float64
        bits = mixed_bits(width, n, 555 + n)[:n]
        cfg = QuantConfig(mode=mode, eb=1e-3, width=width, block_size=bs)
        base, _ = pipeline.compress(bits.view(ft), cfg, workers=1)
        cases.append((name, base, rng))
    return cases


def gen_decode_fuzz():
    """Byte-mutation fuzz of reference streams: exception class (or OK + digest) per mutation."""
    arrays = {}
    meta = []
    for name, base, rng in _mutate_cases():
        muts = []
        outcomes = []
        nmut = 3000
        for _ in range(nmut):
            k = int(rng.integers(1, 4))
            m = [(int(rng.integers(0, len(base))), int(rng.integers(1, 256))) for _ in range(k)]
            muts.append(m + [(-1, 0)] * (3 - k))
            s = bytearray(base)
            for p, x in m:
                s[p] ^= x
            try:
                out = pipeline.decompress_to_array(bytes(s), workers=1)
                outcomes.append("OK:" + sha(out.tobytes())[:16])
            except gebq.ContainerError as e:
                outcomes.append(type(e).__name__ + ":" + str(e))
        # truncations at every length class
        truncs = []
        for cut in sorted(set([0, 4, 47, 48, 51, 56, 63, 64, len(base) // 2, len(base) - 1,
                               len(base) - 2] + list(range(48, min(len(base), 140))))):
            try:
                pipeline.decompress_to_array(base[:cut], workers=1)
                truncs.append((cut, "OK"))
            except gebq.ContainerError as e:
                truncs.append((cut, type(e).__name__ + ":" + str(e)))
        arrays[name + "_base"] = np.frombuffer(base, dtype=np.uint8)
        arrays[name + "_muts"] = np.array(muts, dtype=np.int64)
        meta.append({"name": name, "outcomes": outcomes, "truncations": truncs})
    return arrays, meta


def gen_sweeps(full: bool):
    out = {"subrange": [], "full": [], "f64": [], "f32_random": []}
    sub = [
        (ABS, 1e-3, None, 0, 1 << 24, False), (REL, 1e-3, None, 0, 1 << 24, False),
        (REL, 1e-3, None, 0x7F000000, 1 << 24, False), (ABS, 1e-3, None, 0x3F800000, 1 << 22, True),
        (ABS, 1e-1, None, 0x40000000, 1 << 22, False), (REL, 1e-2, None, 0x3E000000, 1 << 22, False),
        (REL, 1e-5, None, 0xBF000000, 1 << 22, False), (REL, 1e-2, None, 0x3F000000, 1 << 22, True),
        (NOA, 1e-3, 1e10, 0x3F000000, 1 << 20, False), (NOA, 1e-4, 1.0, 0xC0000000, 1 << 22, False),
        (ABS, 1e-5, None, 0xFF000000, 1 << 24, False),
        (ABS, 1e-3, None, 0xFFF00000, 1 << 21, False),  # wraps past 2^32
    ]
    for mode, eb, vr, start, count, unsafe in sub:
        (r,) = sweep.sweep_f32(mode, [eb], value_range=vr, unsafe=unsafe, workers=WORKERS,
                               start=start, count=count)
        out["subrange"].append({"mode": mode, "eb": eb, "value_range": vr, "start": start,
                                "count": count, "unsafe": unsafe, "per_class": r.per_class,
                                "violations": r.violations,
                                "first_violation_bits": r.first_violation_bits})
    if full:
        grid = [(ABS, 1e-3, None), (ABS, 1e-1, None), (ABS, 1e-5, None), (REL, 1e-2, None),
                (REL, 1e-1, None), (REL, 1e-3, None), (REL, 1e-5, None), (NOA, 1e-4, 1.0),
                (NOA, 1e-3, 1.0), (NOA, 1e-3, 1e10), (NOA, 1e-3, 1e-10)]
        for mode, eb, vr in grid:
            (r,) = sweep.sweep_f32(mode, [eb], value_range=vr, workers=WORKERS)
            print("full", mode, eb, vr, r.summary(), flush=True)
            out["full"].append({"mode": mode, "eb": eb, "value_range": vr,
                                "per_class": r.per_class, "violations": r.violations})
    for mode in (ABS, REL):
        for n_random, seed in ((10**6, 0x5D0), (200000, 1)):
            (r,) = sweep.sweep_f64(mode, [1e-3], n_random=n_random, seed=seed, workers=WORKERS)
            out["f64"].append({"mode": mode, "eb": 1e-3, "n_random": n_random, "seed": seed,
                               "per_class": r.per_class, "violations": r.violations})
        (r,) = sweep.sweep_f32_random(mode, [1e-3], n=10**6, seed=42, workers=WORKERS)
        out["f32_random"].append({"mode": mode, "eb": 1e-3, "n": 10**6, "seed": 42,
                                  "per_class": r.per_class, "violations": r.violations})
    return out


def noa_input(rec):
    """Rebuild a NOA-range input from its fixture record (explicit hex or seeded recipe)."""
    if "hex" in rec:
        return np.frombuffer(bytes.fromhex(rec["hex"]), dtype=rec["dtype"]).copy()
    rng = np.random.default_rng(rec["seed"])
    x = rng.standard_normal(rec["n"]) * rec["scale"]
    return x.astype(rec["dtype"])


def gen_noa():
    cases = []
    inputs = {
        "basic": np.array([0.0, 10.0, 5.0], dtype=np.float32),
        "specials": np.array([1.0, np.nan, np.inf, 3.0], dtype=np.float32),
        "equal": np.array([7.0, 7.0], dtype=np.float32),
        "empty": np.array([], dtype=np.float32),
        "nan_only": np.array([np.nan], dtype=np.float32),
        "zeros_mixed": np.array([-0.0, 0.0, -0.0], dtype=np.float32),
        "overflow": np.array([3e38, -3e38], dtype=np.float32),
        "ovf64": np.array([1.7e308, -1.7e308, np.nan], dtype=np.float64),
        "denorm": np.array([1e-45, -1e-45, 0.0], dtype=np.float32),
        "inf_only64": np.array([np.inf, -np.inf], dtype=np.float64),
    }
    recs = [{"name": k, "dtype": str(v.dtype), "hex": v.tobytes().hex()} for k, v in inputs.items()]
    recs += [{"name": "normal32", "dtype": "float32", "seed": 8, "n": 100001, "scale": 1.0},
             {"name": "big64", "dtype": "float64", "seed": 9, "n": 70001, "scale": 1e300},
             {"name": "tiny32", "dtype": "float32", "seed": 10, "n": 4097, "scale": 1e-40}]
    for rec in recs:
        arr = noa_input(rec)
        r = quantizers.compute_noa_range(arr)
        rec["range_bits"] = cbits(r, 32 if arr.dtype == np.float32 else 64)
        cases.append(rec)
    return cases


def gen_workloads():
    out = []
    # C1 smooth field (full 256^3)
    x = workloads.smooth_field(256, 0, np.float32)
    for mode, eb in ((ABS, 1e-3), (NOA, 1e-4), (REL, 1e-2)):
        s, st = pipeline.compress(x, QuantConfig(mode=mode, eb=eb), workers=WORKERS)
        out.append({"workload": "c1", "mode": mode, "eb": eb, "n": len(x), "sha256": sha(s),
                    "bytes": len(s), "triggers": st.triggers,
                    "recon_sha256": sha(pipeline.decompress_to_array(s, workers=WORKERS).tobytes())})
    # C2 recipe at 2^22
    x2 = workloads.c2_values(1 << 22)
    s, st = pipeline.compress(x2, QuantConfig(mode=REL, eb=1e-2), workers=WORKERS)
    out.append({"workload": "c2", "mode": REL, "eb": 1e-2, "n": len(x2), "sha256": sha(s),
                "bytes": len(s), "triggers": st.triggers, "input_sha256": sha(x2.tobytes()),
                "recon_sha256": sha(pipeline.decompress_to_array(s, workers=WORKERS).tobytes())})
    # C5 random f64 at 2^20
    x5 = workloads.c5_random_values(1 << 20)
    for mode in (ABS, REL):
        s, st = pipeline.compress(x5, QuantConfig(mode=mode, eb=1e-3, width=64), workers=WORKERS)
        out.append({"workload": "c5r", "mode": mode, "eb": 1e-3, "n": len(x5), "sha256": sha(s),
                    "bytes": len(s), "triggers": st.triggers})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--full-sweeps", action="store_true")
    args = ap.parse_args()
    rec = verify.compute_golden_record(workers=WORKERS)
    assert verify.check_golden(workers=WORKERS)["passed"]
    extra = []
    for mode, eb, width, rng in verify.GOLDEN_CONFIGS:
        cfg = QuantConfig(mode=mode, eb=eb, width=width, value_range=rng)
        s, st = pipeline.compress(verify._golden_values(width), cfg, workers=WORKERS)
        extra.append({"bytes": len(s), "triggers": st.triggers,
                      "recon_sha256": sha(pipeline.decompress_to_array(s).tobytes())})
    for c, e in zip(rec["configs"], extra):
        c.update(e)
    with open(os.path.join(HERE, "golden_record.json"), "w") as f:
        json.dump(rec, f)

    ka, km = gen_kernels()
    ra, rm = gen_reconstruct()
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **ka, **ra)
    fa, fm = gen_decode_fuzz()
    np.savez_compressed(os.path.join(HERE, "decode_fuzz.npz"), **fa)
    streams, example, empty = gen_streams()
    doc = {
        "constants": gen_constants(),
        "kernel_cases": km,
        "reconstruct_cases": rm,
        "streams": streams,
        "format_example_hex": example,
        "empty_stream_hex": empty,
        "decode_fuzz": fm,
        "noa": gen_noa(),
        "workloads": gen_workloads(),
    }
    import gzip

    with gzip.open(os.path.join(HERE, "fixtures.json.gz"), "wt") as f:
        json.dump(doc, f)
    sw_path = os.path.join(HERE, "sweeps.json")
    prev = {}
    if os.path.exists(sw_path):
        with open(sw_path) as f:
            prev = json.load(f)
    sw = gen_sweeps(args.full_sweeps)
    if not args.full_sweeps and prev.get("full"):
        sw["full"] = prev["full"]
    with open(sw_path, "w") as f:
        json.dump(sw, f, indent=0)
    print("done")


if __name__ == "__main__":
    main()
