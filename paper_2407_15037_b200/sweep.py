"""Exhaustive and sampled round-trip sweeps on the GPU (drop-in for gebq.sweep).

Patterns are generated inside the kernel from the index (exhaustive f32) or
from splitmix64 (sampled), so a full 2^32 sweep moves no input through HBM
and no host arrays are materialised (the reference builds 2^24-pattern
numpy chunks per task, sweep.py:165-169).  Tallies merge commutatively, so
reports are independent of grid size and chunking, as in the reference.
"""

from __future__ import annotations

import json
import time
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from . import device
from .quantizers import REL, QuantConfig
from .workloads import splitmix64

__all__ = ["CLASS_NAMES", "SweepReport", "sweep_f32", "sweep_f32_random", "sweep_f64",
           "structured_f64_bits", "F32_TOTAL"]

CLASS_NAMES = ("zero", "denormal", "normal", "infinity", "nan")
OUTCOME_NAMES = ("quantized", "lossless", "violation")
F32_TOTAL = 1 << 32
DEFAULT_CHUNK = 1 << 24
_STRUCT_RANDOM_MANTISSAS = 4
_STRUCT_STREAM_RESERVED = _STRUCT_RANDOM_MANTISSAS * 2048


@dataclass
class SweepReport:
    """sweep.py:40-86 (same fields, same JSON)."""

    mode: str
    eb: float
    width: int
    patterns_tested: int = 0
    violations: int = 0
    per_class: dict = field(default_factory=dict)
    first_violation_bits: Optional[int] = None
    elapsed: float = 0.0
    value_range: Optional[float] = None
    unsafe: bool = False

    @property
    def lossless_fraction(self) -> float:
        total = sum(c["lossless"] for c in self.per_class.values())
        return total / self.patterns_tested if self.patterns_tested else 0.0

    @property
    def passed(self) -> bool:
        return self.violations == 0

    def to_dict(self) -> dict:
        return {"mode": self.mode, "eb": self.eb, "width": self.width,
                "value_range": self.value_range, "unsafe": self.unsafe,
                "patterns_tested": self.patterns_tested, "violations": self.violations,
                "first_violation_bits": self.first_violation_bits,
                "lossless_fraction": self.lossless_fraction, "per_class": self.per_class,
                "elapsed": self.elapsed}

    def to_json(self) -> str:
        return json.dumps(self.to_dict())

    def summary(self) -> str:
        state = "PASS" if self.passed else "FAIL"
        return (f"{state} mode={self.mode} eb={self.eb:g} f{self.width} "
                f"patterns={self.patterns_tested} violations={self.violations} "
                f"lossless={self.lossless_fraction:.4%} elapsed={self.elapsed:.1f}s")


def _tally_to_dict(tally: np.ndarray) -> dict:
    return {CLASS_NAMES[c]: {OUTCOME_NAMES[o]: int(tally[c, o]) for o in range(3)}
            for c in range(5)}


def _finish(report: SweepReport, tally: np.ndarray, t0: float) -> SweepReport:
    report.per_class = _tally_to_dict(tally)
    report.violations = int(tally[:, 2].sum())
    report.patterns_tested = int(tally.sum())
    report.elapsed = time.perf_counter() - t0
    return report


def _first(first_t) -> Optional[int]:
    f = int(first_t.item()) & ((1 << 64) - 1)
    return None if f == (1 << 64) - 1 else f


def sweep_f32(mode: str, eb_list: Sequence[float], value_range=None, unsafe: bool = False,
              workers: int = 1, chunk: int = DEFAULT_CHUNK, start: int = 0,
              count: int = F32_TOTAL, progress: Optional[Callable[[int, int], None]] = None):
    """Round-trip every f32 pattern in [start, start+count) (mod 2^32) for each bound."""
    reports = []
    for eb in eb_list:
        cfg = QuantConfig(mode=mode, eb=float(eb), width=32, value_range=value_range,
                          unsafe_no_double_check=unsafe)
        t0 = time.perf_counter()
        rep = SweepReport(mode=mode, eb=float(eb), width=32, value_range=value_range, unsafe=unsafe)
        tally, first = device.sweep(cfg, source=device.SOURCE_RANGE, start=start, count=count)
        tally_h = tally.cpu().numpy().reshape(5, 3)
        f = _first(first)
        if f is not None:
            rep.first_violation_bits = (start + f) & 0xFFFFFFFF
        if progress is not None:
            progress(count, count)
        reports.append(_finish(rep, tally_h, t0))
    return reports


def sweep_f32_random(mode: str, eb_list: Sequence[float], n: int, seed: int, value_range=None,
                     unsafe: bool = False, workers: int = 1, chunk: int = DEFAULT_CHUNK,
                     progress=None):
    """Sampled f32 sweep: the low words of n splitmix64 outputs (sweep.py:205-224)."""
    reports = []
    for eb in eb_list:
        cfg = QuantConfig(mode=mode, eb=float(eb), width=32, value_range=value_range,
                          unsafe_no_double_check=unsafe)
        t0 = time.perf_counter()
        rep = SweepReport(mode=mode, eb=float(eb), width=32, value_range=value_range, unsafe=unsafe)
        tally, first = device.sweep(cfg, source=device.SOURCE_SPLITMIX, start=0, count=n, seed=seed)
        f = _first(first)
        if f is not None:
            rep.first_violation_bits = int(splitmix64(1, seed, f)[0]) & 0xFFFFFFFF
        reports.append(_finish(rep, tally.cpu().numpy().reshape(5, 3), t0))
    return reports


def structured_f64_bits(seed: int) -> np.ndarray:
    """Every exponent x {0, all-ones, 4 random} mantissas x both signs (sweep.py:234-248)."""
    words = splitmix64(_STRUCT_STREAM_RESERVED, seed, 0)
    mant_mask = np.uint64((1 << 52) - 1)
    expos = np.arange(2048, dtype=np.uint64) << np.uint64(52)
    mants = np.concatenate([np.zeros((2048, 1), dtype=np.uint64),
                            np.full((2048, 1), (1 << 52) - 1, dtype=np.uint64),
                            (words & mant_mask).reshape(2048, _STRUCT_RANDOM_MANTISSAS)], axis=1)
    base = (expos[:, None] | mants).ravel()
    return np.concatenate([base, base | np.uint64(1 << 63)])


def sweep_f64(mode: str, eb_list: Sequence[float], n_random: int = 0, seed: int = 0,
              value_range=None, unsafe: bool = False, workers: int = 1, chunk: int = 1 << 22,
              progress=None):
    """Structured corpus + n_random splitmix64 patterns for each bound (sweep.py:251-275)."""
    structured = structured_f64_bits(seed)
    reports = []
    for eb in eb_list:
        cfg = QuantConfig(mode=mode, eb=float(eb), width=64, value_range=value_range,
                          unsafe_no_double_check=unsafe)
        t0 = time.perf_counter()
        rep = SweepReport(mode=mode, eb=float(eb), width=64, value_range=value_range, unsafe=unsafe)
        t1, f1 = device.sweep(cfg, source=device.SOURCE_ARRAY, count=len(structured),
                              bits=device.to_device(structured))
        t2, f2 = device.sweep(cfg, source=device.SOURCE_SPLITMIX, start=_STRUCT_STREAM_RESERVED,
                              count=n_random, seed=seed)
        a, b = _first(f1), _first(f2)
        if a is not None:
            rep.first_violation_bits = int(structured[a])
        elif b is not None:
            rep.first_violation_bits = int(splitmix64(1, seed, _STRUCT_STREAM_RESERVED + b)[0])
        tally = t1.cpu().numpy().reshape(5, 3) + t2.cpu().numpy().reshape(5, 3)
        reports.append(_finish(rep, tally, t0))
    return reports
