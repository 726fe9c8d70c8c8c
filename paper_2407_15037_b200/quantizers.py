"""Quantizer configuration and derived constants (host side, O(1) work).

Mirrors the reference's ``gebq.quantizers`` interface (quantizers.py:33-156):
same names, same argument meaning, same exceptions, same width-typed numpy
scalars -- so the GPU path is a drop-in.  The per-element work lives in the
CUDA kernels; the scalar helpers here (``quantize_abs`` etc.) run the very
same kernels on a one-element device array.
"""

from __future__ import annotations

from dataclasses import dataclass, replace
from functools import cached_property
from typing import Optional

import numpy as np

__all__ = [
    "ABS", "REL", "NOA", "MODES", "MAXBIN32", "MAXBIN64", "InvalidBound", "QuantConfig",
    "DerivedConstants", "CodedValue", "CodedArray", "det_log2", "compute_noa_range",
    "quantize", "quantize_abs", "quantize_rel", "reconstruct", "reconstruct_abs",
    "reconstruct_rel",
]

ABS = "abs"
REL = "rel"
NOA = "noa"
MODES = (ABS, REL, NOA)

MAXBIN32 = 1 << 30
MAXBIN64 = 1 << 62


class InvalidBound(ValueError):
    """The error bound is not a positive finite number (quantizers.py:61-62)."""


def det_log2(y, width: int = 64):
    """Deterministic binary log by digit recurrence (numerics.py:188-218).

    The integer exponent comes from the bit fields; 32 rounds of m := m*m
    (one rounded binary64 multiply each) emit the fraction bits MSB first;
    the result is assembled exactly in binary64 and rounded once to ``width``.
    """
    y64 = np.float64(y)
    if not np.isfinite(y64) or y64 <= 1.0:
        raise ValueError(f"det_log2 requires a finite argument > 1, got {y!r}")
    bits = int(y64.view(np.uint64))
    expo = ((bits >> 52) & 0x7FF) - 1023
    m = np.uint64((1023 << 52) | (bits & ((1 << 52) - 1))).view(np.float64)
    two = np.float64(2.0)
    half = np.float64(0.5)
    frac_bits = 0
    for _ in range(32):
        m = m * m
        bit = int(m >= two)
        frac_bits = (frac_bits << 1) | bit
        if bit:
            m = m * half
    acc = np.float64(expo) + np.float64(frac_bits) * np.float64(2.0 ** -32)
    return np.float32(acc) if width == 32 else acc


@dataclass(frozen=True)
class DerivedConstants:
    """Constants derived once per (mode, eb, width[, range]) (quantizers.py:65-89)."""

    width: int
    maxbin: int
    thr: np.floating
    eb_eff: Optional[np.floating] = None
    eb2: Optional[np.floating] = None
    inv_eb2: Optional[np.floating] = None
    op_eps: Optional[np.floating] = None
    w: Optional[np.floating] = None

    @property
    def header_bits(self) -> int:
        """Raw pattern of eb2 (ABS/NOA) or w (REL), zero-extended for f32."""
        v = self.w if self.eb2 is None else self.eb2
        if self.width == 32:
            return int(np.float32(v).view(np.uint32))
        return int(np.float64(v).view(np.uint64))

    @property
    def derived_value(self):
        return self.w if self.eb2 is None else self.eb2


def _derive(mode: str, eb: float, width: int, value_range) -> DerivedConstants:
    """quantizers.py:92-118: each constant is one rounded op in the value width."""
    ft = np.float32 if width == 32 else np.float64
    maxbin = MAXBIN32 if width == 32 else MAXBIN64
    thr = ft(maxbin - 1)
    with np.errstate(all="ignore"):
        if mode == REL:
            op_eps = ft(1.0) + ft(eb)
            if np.isinf(op_eps):
                w = ft(np.inf)
            elif op_eps <= ft(1.0):
                w = ft(0.0)  # eb underflowed at this width: everything goes lossless
            else:
                w = ft(2.0) * det_log2(op_eps, width)
            return DerivedConstants(width=width, maxbin=maxbin, thr=thr, op_eps=op_eps, w=w)
        eps_w = ft(eb)
        if mode == NOA:
            if value_range is None:
                raise ValueError("NOA constants need the data range; run the range pass first")
            eb_eff = eps_w * ft(value_range)
        else:
            eb_eff = eps_w
        eb2 = eb_eff + eb_eff
        inv_eb2 = ft(1.0) / eb2
    return DerivedConstants(width=width, maxbin=maxbin, thr=thr, eb_eff=eb_eff, eb2=eb2,
                            inv_eb2=inv_eb2)


@dataclass(frozen=True)
class QuantConfig:
    """User-facing quantizer configuration (quantizers.py:121-156)."""

    mode: str
    eb: float
    width: int = 32
    block_size: int = 4096
    unsafe_no_double_check: bool = False
    value_range: Optional[float] = None

    def __post_init__(self):
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}, got {self.mode!r}")
        if self.width not in (32, 64):
            raise ValueError(f"width must be 32 or 64, got {self.width!r}")
        eb = float(self.eb)
        if not np.isfinite(eb) or eb <= 0.0:
            raise InvalidBound(f"error bound must be positive and finite, got {self.eb!r}")
        if self.block_size < 1:
            raise ValueError(f"block_size must be >= 1, got {self.block_size!r}")

    @cached_property
    def derived(self) -> DerivedConstants:
        return _derive(self.mode, float(self.eb), self.width, self.value_range)

    def with_range(self, value_range: float) -> "QuantConfig":
        return replace(self, value_range=float(value_range))


@dataclass(frozen=True)
class CodedValue:
    """One coded value: a bin (+ REL sign) or a raw lossless pattern (quantizers.py:159-178)."""

    lossless: bool
    bin: int = 0
    sign: int = 0
    raw: int = 0

    @classmethod
    def quantized(cls, bin: int, sign: int = 0) -> "CodedValue":
        return cls(lossless=False, bin=bin, sign=sign)

    @classmethod
    def from_raw(cls, raw: int) -> "CodedValue":
        return cls(lossless=True, raw=int(raw))


@dataclass
class CodedArray:
    """Structure-of-arrays wire codes + lossless flags (quantizers.py:181-206)."""

    mode: str
    width: int
    lossless: np.ndarray
    codes: np.ndarray

    def __len__(self) -> int:
        return len(self.codes)

    def __eq__(self, other) -> bool:
        return (isinstance(other, CodedArray) and self.mode == other.mode
                and self.width == other.width
                and np.array_equal(self.lossless, other.lossless)
                and np.array_equal(self.codes, other.codes))


def compute_noa_range(values):
    """R = max - min over the finite values, in the input dtype (quantizers.py:337-351).

    Runs the GPU range pass (order-key min/max reduction); plain sequences
    are converted to float64 exactly as the reference does.
    """
    from . import device

    arr = np.asarray(values)
    if arr.dtype not in (np.float32, np.float64):
        arr = arr.astype(np.float64)
    arr = np.ascontiguousarray(arr).ravel()
    return device.noa_range_host(arr)


# ---------------------------------------------------------------------------
# scalar helpers: one value through the GPU kernels (same code path as arrays)
# ---------------------------------------------------------------------------

def _wire_to_coded(code: int, lossless: bool, mode: str) -> CodedValue:
    if lossless:
        return CodedValue.from_raw(code)
    if mode == REL:
        z = code >> 1
        return CodedValue.quantized((z >> 1) ^ -(z & 1), sign=code & 1)
    return CodedValue.quantized((code >> 1) ^ -(code & 1))


def _coded_to_wire(c: CodedValue, mode: str, width: int) -> int:
    if c.lossless:
        return c.raw
    z = ((c.bin << 1) ^ (c.bin >> 63)) & ((1 << 64) - 1)
    code = (z << 1) | c.sign if mode == REL else z
    if code >= 1 << width:
        raise ValueError(f"bin {c.bin} exceeds the {width}-bit code range")
    return code


def quantize(bits: int, cfg: QuantConfig) -> CodedValue:
    """Quantize one value given as its bit pattern (NOA uses the ABS kernel)."""
    from . import device

    itype = np.uint32 if cfg.width == 32 else np.uint64
    codes, lossless, _ = device.quantize_host(np.array([int(bits)], dtype=itype), cfg)
    return _wire_to_coded(int(codes[0]), bool(lossless[0]), cfg.mode)


def quantize_abs(bits: int, cfg: QuantConfig) -> CodedValue:
    return quantize(bits, cfg if cfg.mode != REL else replace(cfg, mode=ABS))


def quantize_rel(bits: int, cfg: QuantConfig) -> CodedValue:
    return quantize(bits, cfg if cfg.mode == REL else replace(cfg, mode=REL))


def reconstruct(c: CodedValue, cfg: QuantConfig) -> int:
    """Bit pattern of the reconstruction of one coded value."""
    from . import device

    itype = np.uint32 if cfg.width == 32 else np.uint64
    code = np.array([_coded_to_wire(c, cfg.mode, cfg.width)], dtype=itype)
    out = device.reconstruct_host(code, np.array([c.lossless]), cfg.mode,
                                  cfg.derived.derived_value)
    return int(out[0])


def reconstruct_abs(c: CodedValue, cfg: QuantConfig) -> int:
    return reconstruct(c, cfg if cfg.mode != REL else replace(cfg, mode=ABS))


def reconstruct_rel(c: CodedValue, cfg: QuantConfig) -> int:
    return reconstruct(c, cfg if cfg.mode == REL else replace(cfg, mode=REL))
