"""End-to-end compression / decompression on the B200 (drop-in for gebq.pipeline).

Same public surface as the reference (pipeline.py:30-228): ``compress``,
``compress_coded``, ``decompress``, ``decompress_to_array``,
``CompressStats``, ``LengthNotMultipleOfWidth``, ``default_workers``.
``workers`` is accepted for signature compatibility; the parallelism is the
GPU grid, and outputs are byte-identical for any value (as in the reference).

compress():    host values --H2D--> [NOA range pass -> derive, on device]
               -> fused quantize+pack kernel -> D2H of index + region
decompress():  host stream --H2D--> fused unpack+reconstruct kernel -> D2H
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import device, stream
from .container import StreamHeader, parse_layout
from .quantizers import NOA, REL, CodedArray, InvalidBound, QuantConfig

__all__ = [
    "CompressStats", "LengthNotMultipleOfWidth", "InvalidBound", "compress", "compress_coded",
    "decompress", "decompress_to_array", "default_workers",
]

TASK_VALUES = 1 << 20


class LengthNotMultipleOfWidth(ValueError):
    """Raw input byte length is not a multiple of the value width."""


@dataclass
class CompressStats:
    """Per-run accounting (pipeline.py:48-81); triggers split the lossless count."""

    values_total: int = 0
    values_lossless: int = 0
    bytes_in: int = 0
    bytes_out: int = 0
    triggers: dict = field(default_factory=lambda: {"nan": 0, "inf": 0, "guard": 0, "double_check": 0})
    wall_time: dict = field(default_factory=dict)

    @property
    def lossless_fraction(self) -> float:
        return self.values_lossless / self.values_total if self.values_total else 0.0

    @property
    def double_check_fraction(self) -> float:
        return self.triggers["double_check"] / self.values_total if self.values_total else 0.0

    @property
    def ratio(self) -> float:
        return self.bytes_in / self.bytes_out if self.bytes_out else 0.0

    def to_dict(self) -> dict:
        return {
            "values_total": self.values_total, "values_lossless": self.values_lossless,
            "lossless_fraction": self.lossless_fraction, "bytes_in": self.bytes_in,
            "bytes_out": self.bytes_out, "ratio": self.ratio, "triggers": dict(self.triggers),
            "wall_time": dict(self.wall_time),
        }


def default_workers() -> int:
    env = os.environ.get("GEBQ_THREADS")
    if env:
        return max(1, int(env))
    return os.cpu_count() or 1


def _as_value_array(values, width: int) -> np.ndarray:
    """pipeline.py:91-103: raw bytes are little-endian; arrays must have the exact dtype."""
    ftype = np.float32 if width == 32 else np.float64
    if isinstance(values, (bytes, bytearray, memoryview)):
        nbytes = len(values)
        if nbytes % (width // 8):
            raise LengthNotMultipleOfWidth(f"{nbytes} bytes is not a multiple of {width // 8}")
        return np.frombuffer(values, dtype=np.dtype(ftype).newbyteorder("<"))
    arr = np.ascontiguousarray(values)
    if arr.dtype != ftype:
        raise TypeError(f"expected {np.dtype(ftype)} values for width {width}, got {arr.dtype}")
    return arr.ravel()


def _upload(arr: np.ndarray) -> torch.Tensor:
    """H2D copy of the value bits (pinned sources go at full link speed, pageable
    ones through the pinned staging ring)."""
    from . import hostio

    dev = device.require_cuda()
    t = torch.empty(arr.size, dtype=torch.int32 if arr.dtype.itemsize == 4 else torch.int64,
                    device=dev)
    if arr.size:
        hostio.h2d(hostio.host_u8(arr), t.view(torch.uint8))
    return t


def _trig_dict(trig: np.ndarray) -> dict:
    return {"nan": int(trig[0]), "inf": int(trig[1]), "guard": int(trig[2]),
            "double_check": int(trig[3])}


def _range_on_device(x: torch.Tensor, cfg: QuantConfig):
    """NOA range pass + constants on the device; returns (cfg with range, consts_dev)."""
    keys = device.noa_keys(x)
    consts, rng = device.noa_derive(keys, float(cfg.eb), cfg.width)
    r = rng.item()  # the host needs R for the header and for the returned cfg
    return cfg.with_range(float(np.float32(r)) if cfg.width == 32 else r), consts


def compress_coded(values, cfg: QuantConfig, workers: Optional[int] = None):
    """Quantize without serializing; returns (CodedArray, cfg, stats) (pipeline.py:112-167)."""
    arr = _as_value_array(values, cfg.width)
    stats = CompressStats(values_total=len(arr), bytes_in=arr.nbytes)
    t0 = time.perf_counter()
    if arr.size == 0:
        if cfg.mode == NOA and cfg.value_range is None:
            cfg = cfg.with_range(0.0)
        stats.wall_time["range_s"] = time.perf_counter() - t0
        stats.wall_time["quantize_s"] = 0.0
        itype = np.uint32 if cfg.width == 32 else np.uint64
        return CodedArray(mode=cfg.mode, width=cfg.width, lossless=np.empty(0, np.bool_),
                          codes=np.empty(0, itype)), cfg, stats
    x = _upload(arr)
    consts = None
    if cfg.mode == NOA and cfg.value_range is None:
        cfg, consts = _range_on_device(x, cfg)
    stats.wall_time["range_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    codes, lossless, trig = device.quantize(x, cfg, consts_dev=consts)
    itype = np.uint32 if cfg.width == 32 else np.uint64
    codes_h = codes.cpu().numpy().view(itype)
    ll_h = lossless.cpu().numpy().view(np.bool_)
    trig_h = trig.cpu().numpy()
    stats.wall_time["quantize_s"] = time.perf_counter() - t0
    stats.triggers = _trig_dict(trig_h)
    stats.values_lossless = int(trig_h.sum())
    return CodedArray(mode=cfg.mode, width=cfg.width, lossless=ll_h, codes=codes_h), cfg, stats


def compress(values, cfg: QuantConfig, workers: Optional[int] = None):
    """Compress a float array (or raw little-endian bytes) to a stream (pipeline.py:170-192).

    Returns (stream bytes, CompressStats).  Fused single-pass encode on the GPU.
    """
    arr = _as_value_array(values, cfg.width)
    stats = CompressStats(values_total=len(arr), bytes_in=arr.nbytes)
    t0 = time.perf_counter()
    if arr.size == 0:
        if cfg.mode == NOA and cfg.value_range is None:
            cfg = cfg.with_range(0.0)
        header = stream.header_for(cfg, 0)
        s = header.pack() + (0).to_bytes(8, "little")
        stats.wall_time.update({"range_s": 0.0, "quantize_s": 0.0, "encode_s": 0.0})
        stats.bytes_out = len(s)
        return s, stats
    if (cfg.mode != NOA or cfg.value_range is not None) and arr.nbytes > 2 * stream.COMPRESS_CHUNK:
        # constants known up front: PCIe in/out overlapped with the encode
        stats.wall_time["range_s"] = 0.0
        t0 = time.perf_counter()
        s, trig_h = stream.compress_pipelined(arr, cfg, stream.header_for(cfg, len(arr)))
    else:
        x = _upload(arr)
        consts = None
        if cfg.mode == NOA and cfg.value_range is None:
            cfg, consts = _range_on_device(x, cfg)
        stats.wall_time["range_s"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        enc = stream.encode(x, cfg, consts_dev=consts)
        header = stream.header_for(cfg, len(arr))
        s = stream.stream_to_host(enc, header)
        trig_h = enc.trig.cpu().numpy()
    stats.wall_time["quantize_s"] = 0.0  # fused into the encode kernel
    stats.wall_time["encode_s"] = time.perf_counter() - t0
    stats.triggers = _trig_dict(trig_h)
    stats.values_lossless = int(trig_h.sum())
    stats.bytes_out = len(s)
    return s, stats


def decompress_to_array(stream_bytes, workers: Optional[int] = None) -> np.ndarray:
    """Decompress a stream to a float array using only header constants (pipeline.py:195-223)."""
    header, nblocks, index_pos = parse_layout(stream_bytes)
    return stream.decode_values_host(stream_bytes, header, nblocks, index_pos)


def decompress(stream_bytes, workers: Optional[int] = None) -> bytes:
    """Decompress a stream to raw little-endian value bytes."""
    return decompress_to_array(stream_bytes, workers).tobytes()
