#!/usr/bin/env python
"""bench.py -- B200 quantize/dequantize throughput for the gebq hot path.

One *step* = one pass of the hot path over one batch: fused encode
(quantize + FORMAT.md pack, one kernel) then fused decode (unpack +
reconstruct, one kernel) of the batch, data resident in HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU)

Default workload = BASELINE.json configs[1] (C2): REL f32 eb=1e-2, 2^26
mixed values per GPU (NaN/Inf/denormal/huge outliers), weak scaling, no
data-path collective.  ``--workload c3`` runs NOA (range pass -> NCCL MAX
allreduce of the two order keys -> derive -> encode -> decode), strong
scaling over a 2^30-value field.

Metric basis: GB/s of uncompressed values through quantize + dequantize,
i.e. (n*W encoded + n*W decoded) / step time, summed over ranks (the
paper's input-bytes convention applied to both stages).  Rank 0 prints ONE
JSON line.  ``--impl reference`` times the reference algorithm on the host
cores instead (the plain-C oracle port, oracle/, all threads), same metric.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "quantize/dequantize GB/s at 1/2/4/8 B200 vs HBM roofline; 0 bound violations"

WORKLOADS = {
    "c3": dict(desc="C3: NOA f32 eb=1e-4, 1024^3 smooth field (2^30 values, counter-based noise, planted "
                    "NaN/+Inf/-7/+7) sharded over the GPUs",
               mode="noa", eb=1e-4, width=32, n=1 << 30, scaling="strong", cpu_sample=1 << 26),
    "c2": dict(desc="C2: REL f32 eb=1e-2, mixed NaN/Inf/denormal/huge (SURVEY App. C), 2^26 values per GPU",
               mode="rel", eb=1e-2, width=32, n=1 << 26, scaling="weak", cpu_sample=1 << 26),
    "c1": dict(desc="C1: ABS f32 eb=1e-3, 256^3 smooth field per GPU", mode="abs", eb=1e-3,
               width=32, n=1 << 24, scaling="weak", cpu_sample=1 << 24),
    "c5": dict(desc="C5: ABS f64 eb=1e-3, 2^30 random splitmix64 doubles per GPU", mode="abs",
               eb=1e-3, width=64, n=1 << 30, scaling="weak", cpu_sample=1 << 25),
    "c5rel": dict(desc="C5: REL f64 eb=1e-3, 2^30 random splitmix64 doubles per GPU", mode="rel",
                  eb=1e-3, width=64, n=1 << 30, scaling="weak", cpu_sample=1 << 25),
    "c5s": dict(desc="C5: ABS f64 eb=1e-3, 2^30-value smooth field (1024^3, counter-based noise) per GPU",
                mode="abs", eb=1e-3, width=64, n=1 << 30, scaling="weak", cpu_sample=1 << 25),
    "c5rels": dict(desc="C5: REL f64 eb=1e-3, 2^30-value smooth field (1024^3, counter-based noise) per GPU",
                   mode="rel", eb=1e-3, width=64, n=1 << 30, scaling="weak", cpu_sample=1 << 25),
    "c4": dict(desc="C4: exhaustive sweep of all 2^32 f32 patterns through ABS 1e-3, REL 1e-2 and "
                    "NOA 1e-4 (R=1), pattern range sharded over the GPUs", mode="sweep", eb=None,
               width=32, n=1 << 32, scaling="strong"),
}


def shard_size(wl: dict, world: int) -> int:
    return wl["n"] // world if wl["scaling"] == "strong" else wl["n"]


def config_dict(wl: dict, world: int, args) -> dict:
    """The config both arms print (identical keys and values for the same flags)."""
    n = shard_size(wl, world)
    W = wl["width"] // 8
    cfg = {"workload": wl["desc"], "n_per_gpu": n, "n_total": n * world, "block_size": 4096,
           "parallelism": f"dp{world} (contiguous block-aligned shards)",
           "l2": "inputs larger than L2 (values %d MiB per GPU)" % (n * W >> 20),
           "gbs_basis": "uncompressed bytes encoded + decoded per second, all GPUs"}
    if getattr(args, "unsafe", False):
        cfg["unsafe_no_double_check"] = True
    return cfg


# exhaustive 2^32 tallies (normal class quantized / lossless)
C4_CONFIGS = (("abs", 1e-3, None, 2443713898, 1817698966),
              ("rel", 1e-2, None, 3974120554, 287292310),
              ("noa", 1e-4, 1.0, 2363099024, 1898313840))


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c3")
    ap.add_argument("--variant", choices=["fused", "lib"], default="fused",
                    help="lib: the paper's approx-vs-library REL comparison (PAPER.md:366-386) -- the "
                         "CodedArray quantize -> pack -> unpack -> reconstruct chain with the library-log "
                         "kernels (_kernels.py:356-431) timed beside the same chain with the approx ones")
    ap.add_argument("--unsafe", action="store_true",
                    help="skip the double-check (the paper's 'unprotected' quantizer, PAPER.md:428-441)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    return ap.parse_args()


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def load_traffic(workload: str):
    """ncu dram bytes per launch for the dominant kernel, if a capture was committed."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(workload)
    except Exception:
        return None


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML, same counters as the nvidia-smi line)
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int, period_s: float = 0.002):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._th = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None
        self.period = period_s

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self._nv is not None:
            self._th = threading.Thread(target=self._run, daemon=True)
            self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._th is not None:
            self._th.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# inputs
# ---------------------------------------------------------------------------
def make_input(wl: dict, name: str, rank: int, world: int, device):
    """Per-rank shard on the device (contiguous, block-aligned part of a global array)."""
    import torch

    from paper_2407_15037_b200 import device as gdev
    from paper_2407_15037_b200 import workloads

    n = shard_size(wl, world)
    start = rank * n
    if name == "c2":
        return gdev.mixed_f32(n, workloads.C2_SEED, start, device=device), n
    if name in ("c5", "c5rel"):
        return gdev.splitmix64(n, workloads.C5_SEED, start, device=device), n
    if name == "c1":
        x = workloads.smooth_field(256, rank, np.float32)
        return torch.from_numpy(x.view(np.int32)).to(device), n
    if name == "c3":
        # counter-based field of the GLOBAL index: identical bits at every world size
        return gdev.smooth_field(n, workloads.C3_SIDE, workloads.C3_SEED, start, 32, plant=True,
                                 total=wl["n"], device=device), n
    if name in ("c5s", "c5rels"):
        return gdev.smooth_field(n, workloads.C3_SIDE, workloads.C5_SMOOTH_SEED, start, 64, plant=False,
                                 device=device), n
    raise ValueError(name)


# ---------------------------------------------------------------------------
# reference arm / CPU baseline: the oracle port on the host cores
# ---------------------------------------------------------------------------
def host_input(name: str, wl: dict, n: int) -> np.ndarray:
    """The first n values of rank 0's shard, built on the host by the same recipes
    (bit-identical to ``make_input``; tests/test_gpu_workloads.py checks it)."""
    from paper_2407_15037_b200 import workloads

    if name == "c2":
        return workloads.c2_values(n)
    if name in ("c5", "c5rel"):
        return workloads.splitmix64(n, workloads.C5_SEED).view(np.float64)
    if name == "c1":
        return workloads.smooth_field(256, 0, np.float32)[:n]
    if name == "c3":
        return workloads.smooth_field_cb(n, workloads.C3_SIDE, workloads.C3_SEED, 0, np.float32,
                                         plant=True, total=wl["n"])
    if name in ("c5s", "c5rels"):
        return workloads.smooth_field_cb(n, workloads.C3_SIDE, workloads.C5_SMOOTH_SEED, 0, np.float64,
                                         plant=False)
    raise ValueError(name)


def cpu_roundtrip_gbs(x: np.ndarray, wl: dict, workers: int, reps: int, unsafe: bool = False):
    """Median GB/s (same basis) of oracle compress + decompress on the host cores."""
    from oracle import oracle as orc

    orc.lib()
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        s, _, _ = orc.compress(x, wl["mode"], wl["eb"], unsafe=unsafe, workers=workers)
        y = orc.decompress_to_array(s, workers=workers)
        times.append(time.perf_counter() - t0)
        del s, y
    t = float(np.median(times))
    return 2 * x.nbytes / t / 1e9, t, times


def run_reference(args, wl, name):
    """--impl reference: the reference algorithm (oracle/ C port of gebq's numba
    loops) on all host threads; each step compresses + decompresses a bounded
    sample (the first ``cpu_sample`` values of rank 0's shard) of the workload."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    n = min(shard_size(wl, world), wl["cpu_sample"])
    cores = os.cpu_count() or 1
    x = host_input(name, wl, n)
    from oracle import oracle as orc

    orc.lib()
    for _ in range(max(args.warmup, 1)):
        s, _, _ = orc.compress(x, wl["mode"], wl["eb"], unsafe=args.unsafe, workers=cores)
        orc.decompress_to_array(s, workers=cores)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        s, _, _ = orc.compress(x, wl["mode"], wl["eb"], unsafe=args.unsafe, workers=cores)
        orc.decompress_to_array(s, workers=cores)
        times.append(time.perf_counter() - t0)
    t = float(np.mean(times))
    value = 2 * x.nbytes / t / 1e9
    sample = (f"first {n} values ({x.nbytes >> 20} MiB) of rank 0's {name} shard per step, "
              f"compress + decompress on {cores} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": wl["scaling"], "vs_baseline": None,
        "dtype": "f32" if wl["width"] == 32 else "f64", "data": "synthetic",
        "config": config_dict(wl, world, args),
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "reference algorithm = plain-C restatement of gebq's numba loops (oracle/, pinned "
                "to the reference's golden digests); the Python reference does not ship to the GPU box",
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# C4: exhaustive 2^32 sweeps (sweep.py:172-191), both arms
# ---------------------------------------------------------------------------
def _expected_tally(mode, q, l):
    t = np.zeros((5, 3), dtype=np.int64)
    t[3, 1] = 2                       # +-inf: lossless
    t[4, 1] = 16777214                # NaN: lossless
    if mode == "rel":
        t[0, 1], t[1, 1] = 2, 16777214   # zero / denormal: lossless (REL guard)
    else:
        t[0, 0], t[1, 0] = 2, 16777214   # zero / denormal: quantized
    t[2, 0], t[2, 1] = q, l
    return t


def sweep_config(wl: dict, world: int) -> dict:
    return {"workload": wl["desc"], "patterns_total": 1 << 32,
            "parallelism": f"dp{world} (contiguous pattern ranges)",
            "gbs_basis": "4 B per pattern x 3 configurations per step"}


def run_sweep_bench(args, wl):
    """One step = the three Appendix-B configurations swept over this rank's
    share of the 2^32 patterns (generated in-kernel: no HBM input).  value =
    3 x 2^32 x 4 B / step time (input-bytes convention), plus patterns/s."""
    world, rank, local = dist_env()
    total = 1 << 32
    if args.impl == "reference":
        if rank != 0:
            return 0
        from oracle import oracle as orc

        orc.lib()
        cores = os.cpu_count() or 1
        sample = 1 << 27                      # per config, a bounded slice of the range
        start = 0x3F000000
        for _ in range(max(args.warmup, 1)):
            orc.sweep_f32_range("abs", 1e-3, start, 1 << 22, workers=cores)
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            for mode, eb, vr, _q, _l in C4_CONFIGS:
                orc.sweep_f32_range(mode, eb, start, sample, value_range=vr, workers=cores)
            times.append(time.perf_counter() - t0)
        t = float(np.mean(times))
        pps = 3 * sample / t
        value = pps * 4 / 1e9
        line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic (all f32 bit patterns)",
                "config": sweep_config(wl, world),
                "patterns_per_s": pps,
                "cpu_baseline": {"value": value, "unit": "GB/s", "cores": cores, "kind": "port",
                                 "sample": "3 configs x 2^27 consecutive patterns per step"},
                "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0

    import torch
    import torch.distributed as dist

    from paper_2407_15037_b200 import _lib, device as gdev
    from paper_2407_15037_b200.quantizers import QuantConfig
    from paper_2407_15037_b200.sweep import sweep_f32

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    _lib.load()
    per = total // world
    start = rank * per
    count = total - start if rank == world - 1 else per
    cfgs = [QuantConfig(mode=m, eb=eb, width=32, value_range=vr) for m, eb, vr, _q, _l in C4_CONFIGS]
    tallies = [torch.zeros(15, dtype=torch.int64, device=dev) for _ in cfgs]
    firsts = [torch.full((1,), -1, dtype=torch.int64, device=dev) for _ in cfgs]
    st = torch.cuda.current_stream()

    def step(acc):
        for c, t, f in zip(cfgs, tallies, firsts):
            if not acc:
                t.zero_()
                f.fill_(-1)
            gdev.sweep(c, source=gdev.SOURCE_RANGE, start=start, count=count, tally=t, first=f)

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    # correctness of the last sweep against SURVEY Appendix B (summed over ranks)
    tl = torch.stack(tallies)
    if world > 1:
        dist.all_reduce(tl)
    tl = tl.cpu().numpy().reshape(3, 5, 3)
    match = all(np.array_equal(tl[i], _expected_tally(m, q, l)) for i, (m, _e, _v, q, l) in enumerate(C4_CONFIGS))
    violations = int(tl[:, :, 2].sum())
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0e = torch.cuda.Event(enable_timing=True)
    t1e = torch.cuda.Event(enable_timing=True)
    launches0 = _lib.launch_count()
    with ClockSampler(local) as clk:
        t0e.record(st)
        for _ in range(args.steps):
            step(False)
        t1e.record(st)
        torch.cuda.synchronize()
    launches = _lib.launch_count() - launches0
    ms = torch.tensor([t0e.elapsed_time(t1e) / args.steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    pps = 3 * total / (ms * 1e-3)
    value = pps * 4 / 1e9
    # e2e: the public API (sweep_f32 -> SweepReport on the host), this rank's share
    t0 = time.perf_counter()
    for m, eb, vr, _q, _l in C4_CONFIGS:
        sweep_f32(m, [eb], value_range=vr, start=start, count=count)
    torch.cuda.synchronize()
    el = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(el, op=dist.ReduceOp.MAX)
    e2e = 3 * total * 4 / float(el.item()) / 1e9
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as orc

        orc.lib()
        cores = os.cpu_count() or 1
        sample = 1 << 27
        t0 = time.perf_counter()
        for mth, eb, vr, _q, _l in C4_CONFIGS:
            orc.sweep_f32_range(mth, eb, 0x3F000000, sample, value_range=vr, workers=cores)
        tc = time.perf_counter() - t0
        cpu = {"value": 3 * sample * 4 / tc / 1e9, "unit": "GB/s", "cores": cores, "kind": "port",
               "sample": f"3 configs x 2^27 patterns from 0x3F000000 ({tc:.1f} s) on {cores} threads"}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic (all 2^32 f32 bit patterns, generated in-kernel)",
                "config": sweep_config(wl, world), "patterns_per_gpu": count,
                "patterns_per_s": pps, "violations": violations, "tallies_match_appendix_b": bool(match),
                "e2e": {"value": e2e, "unit": "GB/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 3 * 16 * 8,
                        "api": "paper_2407_15037_b200.sweep_f32 (SweepReport to the host)"},
                "roofline": {"bound": "alu", "achieved": None, "peak": None, "unit": None, "frac": None,
                             "traffic": None, "note": "no HBM input: patterns are generated in-kernel"},
                "cpu_baseline": cpu, "clocks": clk.summary(), "gpu_launches": launches}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# ---------------------------------------------------------------------------
# --variant lib: approx vs library log2/exp2 REL (the paper's Tables 4/6/7)
# ---------------------------------------------------------------------------
def run_variant_bench(args, wl):
    """REL f32 chain quantize -> pack -> unpack -> reconstruct, once with the
    conforming approx kernels and once with the library-log ones
    (quantize_rel32_lib / reconstruct_rel32_lib, non-conforming by design);
    same input, same stages, same timing.  value = the lib chain's GB/s."""
    import ctypes

    import torch

    from paper_2407_15037_b200 import _lib, device as gdev, stream
    from paper_2407_15037_b200.container import StreamHeader
    from paper_2407_15037_b200.quantizers import QuantConfig

    if wl["mode"] != "rel" or wl["width"] != 32:
        raise SystemExit("--variant lib needs a REL binary32 workload (the *_lib kernels are binary32)")
    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    _lib.load()
    x, n = make_input(wl, args.workload, rank, world, dev)
    cfg = QuantConfig(mode="rel", eb=wl["eb"], width=32, unsafe_no_double_check=args.unsafe)
    d = cfg.derived
    st = torch.cuda.current_stream()
    codes = torch.empty_like(x)
    ll = torch.empty(n, dtype=torch.uint8, device=dev)
    trig = torch.zeros(4, dtype=torch.int64, device=dev)
    out = torch.empty_like(x)
    hdr = StreamHeader(width=32, mode="rel", count=n, eb_bits=0, derived_bits=d.header_bits,
                       block_size=cfg.block_size)
    nblocks = -(-n // cfg.block_size)
    P = ctypes.c_void_p

    def chain(lib: bool):
        if lib:
            _lib.call("gebq_quantize_rel_lib_f32", P(x.data_ptr()), P(codes.data_ptr()), P(ll.data_ptr()), n,
                      float(d.op_eps), float(d.w), float(d.thr), int(args.unsafe), P(trig.data_ptr()),
                      P(st.cuda_stream))
        else:
            gdev.quantize(x, cfg, codes=codes, lossless=ll, trig=trig)
        enc = stream.encode_coded(codes, ll, cfg.block_size)
        c2, l2, _err = stream.decode_codes(enc.buf, hdr, nblocks)
        if lib:
            _lib.call("gebq_dequantize_rel_lib_f32", P(c2.data_ptr()), P(l2.data_ptr()), P(out.data_ptr()), n,
                      float(d.w), P(st.cuda_stream))
        else:
            gdev.reconstruct(c2, l2, "rel", d.w, out=out)
        return enc

    res = {}
    launches0 = _lib.launch_count()
    with ClockSampler(local) as clk:
        for lib in (False, True):
            for _ in range(args.warmup):
                enc = chain(lib)
            torch.cuda.synchronize()
            rl = int(enc.region_len.item())
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record(st)
            for _ in range(args.steps):
                chain(lib)
            t1.record(st)
            torch.cuda.synchronize()
            ms = t0.elapsed_time(t1) / args.steps
            res["lib" if lib else "approx"] = {"ms_per_step": ms, "gbs": 2 * n * 4 / (ms * 1e-3) / 1e9,
                                               "stream_bytes_per_value": (rl + 56 + 8 * nblocks) / n}
    launches = _lib.launch_count() - launches0
    line = {"metric": METRIC, "value": res["lib"]["gbs"], "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": res["lib"]["ms_per_step"], "higher_is_better": True,
            "scaling": wl["scaling"], "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": dict(config_dict(wl, world, args), variant="lib"),
            "variant_compare": dict(res, lib_over_approx=res["lib"]["gbs"] / res["approx"]["gbs"],
                                    ratio_loss_approx=res["approx"]["stream_bytes_per_value"]
                                    / res["lib"]["stream_bytes_per_value"] - 1.0,
                                    chain="CodedArray quantize -> pack -> unpack -> reconstruct (4 launches)"),
            "clocks": clk.summary(), "gpu_launches": launches}
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
def main():
    args = parse_args()
    args.warmup = max(args.warmup, 3)
    wl = WORKLOADS[args.workload]
    if args.workload == "c4":
        return run_sweep_bench(args, wl)
    if args.impl == "reference":
        return run_reference(args, wl, args.workload)
    if args.variant == "lib":
        return run_variant_bench(args, wl)

    import torch
    import torch.distributed as dist

    from paper_2407_15037_b200 import _lib, device as gdev, stream
    from paper_2407_15037_b200.container import StreamHeader
    from paper_2407_15037_b200.pipeline import compress, decompress_to_array
    from paper_2407_15037_b200.quantizers import NOA, QuantConfig

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    _lib.load()

    x, n = make_input(wl, args.workload, rank, world, dev)
    W = wl["width"] // 8
    cfg = QuantConfig(mode=wl["mode"], eb=wl["eb"], width=wl["width"], unsafe_no_double_check=args.unsafe)
    bs = cfg.block_size
    nblocks = -(-n // bs)
    buf = stream.alloc_stream(n, bs, wl["width"], dev)
    ws = torch.empty(max(stream.workspace_bytes(n, bs, wl["width"]), 16), dtype=torch.uint8, device=dev)
    trig = torch.zeros(4, dtype=torch.int64, device=dev)
    rlen = torch.empty(1, dtype=torch.int64, device=dev)
    out = torch.empty(n, dtype=x.dtype, device=dev)
    err = torch.full((1,), -1, dtype=torch.int64, device=dev)
    keys = torch.empty(2, dtype=torch.int64, device=dev)
    # decode header: NOA reconstructs with the ABS kernel and takes eb2 from the device
    hdr = StreamHeader(width=wl["width"], mode="abs" if wl["mode"] == NOA else wl["mode"],
                       count=n, eb_bits=0, derived_bits=cfg.derived.header_bits if wl["mode"] != NOA else 0,
                       block_size=bs)
    st = torch.cuda.current_stream()

    def step(ev=None):
        consts = None
        if wl["mode"] == NOA:
            gdev.noa_keys(x, keys)
            if world > 1:
                dist.all_reduce(keys, op=dist.ReduceOp.MAX)  # the one data-path collective
            consts, _ = gdev.noa_derive(keys, wl["eb"], wl["width"])
        if ev is not None:
            ev[0].record(st)
        trig.zero_()
        enc = stream.encode(x, cfg, consts_dev=consts, buf=buf, ws=ws, trig=trig, region_len=rlen)
        if ev is not None:
            ev[1].record(st)
        err.fill_(-1)
        stream.decode_values(buf, hdr, nblocks, out=out, err=err, region_len_dev=rlen,
                             derived_dev=None if consts is None else consts[1:])
        if ev is not None:
            ev[2].record(st)
        return enc

    # warm-up + one correctness probe: decoded stream must be error-free and,
    # for lossless values, the trigger counts must add up
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    stream_bytes = int(rlen.item()) + 56 + 8 * nblocks
    if not os.environ.get("GEBQ_B200_EXP"):
        assert int(err.item()) == -1, "decode reported an error on a freshly encoded stream"
    trig_h = trig.cpu().numpy().tolist()
    # bound check of the step's round trip on the device (verify.py:88-153)
    from paper_2407_15037_b200 import verify as verify_values

    ftype = torch.float32 if wl["width"] == 32 else torch.float64
    vr = None
    if wl["mode"] == NOA:
        _, rng_dev = gdev.noa_derive(keys, wl["eb"], wl["width"])
        vr = float(rng_dev.item())
    vrep = verify_values(x.view(ftype), out.view(ftype), wl["mode"], wl["eb"], vr)
    violations = vrep.violations + vrep.special_mismatch_count
    if world > 1:
        vt = torch.tensor([violations], dtype=torch.int64, device=dev)
        dist.all_reduce(vt)
        violations = int(vt.item())

    # timed region: K device steps, events on the launching stream
    events = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = _lib.launch_count()
    with ClockSampler(local) as clk:
        t_start.record(st)
        for i in range(args.steps):
            step(events[i])
        t_end.record(st)
        torch.cuda.synchronize()
    launches = _lib.launch_count() - launches0
    if world > 1:
        dist.barrier()
    total_ms = t_start.elapsed_time(t_end)
    enc_ms = float(np.mean([e[0].elapsed_time(e[1]) for e in events]))
    dec_ms = float(np.mean([e[1].elapsed_time(e[2]) for e in events]))
    t = torch.tensor([total_ms, enc_ms, dec_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, enc_ms, dec_ms = t.tolist()
    ms_per_step = total_ms / args.steps
    n_all = n * world
    value = 2 * n_all * W / (ms_per_step * 1e-3) / 1e9

    peak, peak_kind = load_peaks()
    enc_bytes = n * W + stream_bytes            # algorithmic: read values, write stream
    dec_bytes = stream_bytes + n * W            # read stream, write values
    enc_gbs = enc_bytes / (enc_ms * 1e-3) / 1e9
    dec_gbs = dec_bytes / (dec_ms * 1e-3) / 1e9
    dominant = ("encode", enc_ms, enc_bytes, enc_gbs) if enc_ms >= dec_ms else ("decode", dec_ms, dec_bytes, dec_gbs)
    traffic = load_traffic(args.workload)
    if isinstance(traffic, dict):
        traffic = traffic.get(dominant[0])

    # the CodedArray stage alone (quantize_* -> codes + flags, reconstruct_*), the
    # reference's quantizer boundary before the lossless container: not part of
    # the step, reported beside it (same batch, device resident)
    coded = None
    if not os.environ.get("GEBQ_B200_NO_CODED"):
        consts_c = None
        if wl["mode"] == NOA:
            consts_c, _ = gdev.noa_derive(keys, wl["eb"], wl["width"])
        codes_c = torch.empty_like(x)
        ll_c = torch.empty(n, dtype=torch.uint8, device=dev)
        trig_c = torch.zeros(4, dtype=torch.int64, device=dev)
        out_c = torch.empty_like(x)
        rmode = "abs" if wl["mode"] == NOA else wl["mode"]
        derived_c = None if consts_c is not None else cfg.derived.derived_value

        def coded_step(evq=None):
            if evq is not None:
                evq[0].record(st)
            gdev.quantize(x, cfg, codes=codes_c, lossless=ll_c, trig=trig_c, consts_dev=consts_c)
            if evq is not None:
                evq[1].record(st)
            dv = derived_c if derived_c is not None else float(consts_c[1].item())
            gdev.reconstruct(codes_c, ll_c, rmode, dv, out=out_c)
            if evq is not None:
                evq[2].record(st)

        if consts_c is not None:
            derived_c = float(consts_c[1].item())
        for _ in range(3):
            coded_step()
        torch.cuda.synchronize()
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
        for i in range(args.steps):
            coded_step(evs[i])
        torch.cuda.synchronize()
        q_ms = float(np.mean([e[0].elapsed_time(e[1]) for e in evs]))
        r_ms = float(np.mean([e[1].elapsed_time(e[2]) for e in evs]))
        cb = n * (2 * W + 1)
        coded = {"quantize": {"ms": q_ms, "gbs": cb / (q_ms * 1e-3) / 1e9, "frac": cb / (q_ms * 1e-3) / 1e9 / load_peaks()[0],
                              "bytes": cb, "basis": "n x (W read + W code + 1 flag)"},
                 "reconstruct": {"ms": r_ms, "gbs": cb / (r_ms * 1e-3) / 1e9, "frac": cb / (r_ms * 1e-3) / 1e9 / load_peaks()[0],
                                 "bytes": cb, "basis": "n x (W code + 1 flag read + W value)"},
                 "value_gbs": 2 * n_all * W / ((q_ms + r_ms) * 1e-3) / 1e9}

    # end-to-end through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        ft = np.float32 if wl["width"] == 32 else np.float64
        pinned = torch.empty(n, dtype=x.dtype, pin_memory=True)
        pinned.copy_(x)
        xh = pinned.numpy().view(ft)
        e2e_cfg = QuantConfig(mode=wl["mode"], eb=wl["eb"], width=wl["width"],
                              unsafe_no_double_check=args.unsafe)
        # warm-up with the timed loop's exact allocation pattern (the previous
        # step's stream and values stay alive while the next step allocates)
        s = y = None
        for _ in range(3):
            s, _ = compress(xh, e2e_cfg)
            y = decompress_to_array(s)
        k2 = args.e2e_steps or max(3, min(args.steps, 10))
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        h2d = d2h = 0
        for _ in range(k2):
            s, st_ = compress(xh, e2e_cfg)
            y = decompress_to_array(s)
            h2d += xh.nbytes + len(s)
            d2h += len(s) + y.nbytes
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        tt = torch.tensor([el], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        el = tt.item()
        e2e = {"value": 2 * n_all * W / (el / k2) / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": int(h2d / k2), "d2h_bytes_per_step": int(d2h / k2),
               "steps": k2, "ms_per_step": el / k2 * 1e3,
               "api": "paper_2407_15037_b200.compress + decompress_to_array (pinned numpy in, bytes/ndarray out)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        m = min(n, wl["cpu_sample"])
        xh_cpu = x[:m].cpu().numpy().view(np.float32 if wl["width"] == 32 else np.float64)  # same bits
        gbs, tmed, times = cpu_roundtrip_gbs(xh_cpu, wl, cores, reps=5, unsafe=args.unsafe)
        cpu = {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "port",
               "sample": f"first {m} values of the GPU arm's input (same bits), compress+decompress, "
                         f"median of 5 ({tmed * 1e3:.0f} ms each) on {cores} threads"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": wl["scaling"], "vs_baseline": None,
            "dtype": "f32" if wl["width"] == 32 else "f64", "data": "synthetic",
            "config": config_dict(wl, world, args),
            "e2e": e2e,
            "roofline": {"bound": "hbm", "kernel": dominant[0], "achieved": dominant[3],
                         "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": dominant[3] / peak, "traffic": traffic,
                         "algorithmic_bytes_per_launch": dominant[2],
                         "ms_per_launch": dominant[1]},
            "kernels": {"encode": {"ms": enc_ms, "gbs": enc_gbs, "frac": enc_gbs / peak,
                                   "bytes": enc_bytes, "input_gbs": n * W / (enc_ms * 1e-3) / 1e9},
                        "decode": {"ms": dec_ms, "gbs": dec_gbs, "frac": dec_gbs / peak,
                                   "bytes": dec_bytes, "input_gbs": n * W / (dec_ms * 1e-3) / 1e9}},
            "coded_stage": coded,
            "stream_bytes_per_value": stream_bytes / n, "triggers": trig_h,
            "violations": violations,
            "violations_check": "device verify (verify.py:88-153 predicates) of every decoded value, all ranks",
            "cpu_baseline": cpu, "clocks": clk.summary(), "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
