"""Device-resident API over torch CUDA tensors (zero-copy into the C ABI).

PyTorch only supplies device memory, streams and ``torch.distributed``; every
byte of the hot path is produced by libgebq_b200.so.  Tensors carry value bit
patterns as int32 / int64 (the unsigned wire codes reinterpret losslessly)
and lossless flags as uint8.  All calls are stream-ordered on the current
torch stream and never synchronise unless a host result is requested.
"""

from __future__ import annotations

import ctypes
from typing import Optional

import numpy as np
import torch

from . import _lib
from .quantizers import NOA, REL, QuantConfig, _derive

_ITYPE = {32: torch.int32, 64: torch.int64}
_FTYPE = {32: torch.float32, 64: torch.float64}
_NP_ITYPE = {32: np.uint32, 64: np.uint64}
_NP_SITYPE = {32: np.int32, 64: np.int64}


class NoDeviceError(RuntimeError):
    """Raised when no CUDA device is visible: the B200 backend has no CPU fallback."""


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise NoDeviceError("no CUDA device visible: the gebq B200 backend has no CPU fallback")
    _lib.load()
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


def _s():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _p(t: torch.Tensor):
    return ctypes.c_void_p(t.data_ptr())


def _width_of(t: torch.Tensor) -> int:
    if t.dtype in (torch.float32, torch.int32, torch.uint32):
        return 32
    if t.dtype in (torch.float64, torch.int64, torch.uint64):
        return 64
    raise TypeError(f"expected a 32- or 64-bit tensor, got {t.dtype}")


def as_bits(t: torch.Tensor) -> torch.Tensor:
    """Contiguous integer view of a float or integer CUDA tensor."""
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    t = t.contiguous().reshape(-1)
    return t.view(_ITYPE[_width_of(t)])


def _f(width):
    return ctypes.c_float if width == 32 else ctypes.c_double


# ---------------------------------------------------------------------------
# quantize / reconstruct (CodedArray level)
# ---------------------------------------------------------------------------

def quantize(x: torch.Tensor, cfg: QuantConfig, *, codes: Optional[torch.Tensor] = None,
             lossless: Optional[torch.Tensor] = None, trig: Optional[torch.Tensor] = None,
             consts_dev: Optional[torch.Tensor] = None):
    """quantize_{abs,rel}{32,64} on device.  Returns (codes, lossless_u8, trig_i64[4]).

    ``consts_dev`` (NOA only) takes the constants from device memory as written
    by :func:`noa_derive`, so the range pass -> derive -> quantize chain never
    synchronises with the host.  ``trig`` accumulates (zeroed if allocated here).
    """
    xb = as_bits(x)
    width = _width_of(xb)
    n = xb.numel()
    if codes is None:
        codes = torch.empty(n, dtype=_ITYPE[width], device=xb.device)
    if lossless is None:
        lossless = torch.empty(n, dtype=torch.uint8, device=xb.device)
    if trig is None:
        trig = torch.zeros(4, dtype=torch.int64, device=xb.device)
    sfx = "f32" if width == 32 else "f64"
    F = _f(width)
    unsafe = int(bool(cfg.unsafe_no_double_check))
    if consts_dev is not None:
        _lib.call(f"gebq_quantize_noa_dev_{sfx}", _p(xb), _p(codes), _p(lossless), n,
                  _p(consts_dev), unsafe, _p(trig), _s())
        return codes, lossless, trig
    d = cfg.derived
    if cfg.mode == REL:
        _lib.call(f"gebq_quantize_rel_{sfx}", _p(xb), _p(codes), _p(lossless), n, F(d.op_eps),
                  F(d.w), F(d.thr), unsafe, _p(trig), _s())
    else:
        _lib.call(f"gebq_quantize_abs_{sfx}", _p(xb), _p(codes), _p(lossless), n, F(d.eb_eff),
                  F(d.eb2), F(d.inv_eb2), F(d.thr), unsafe, _p(trig), _s())
    return codes, lossless, trig


def reconstruct(codes: torch.Tensor, lossless: torch.Tensor, mode: str, derived, *,
                out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """reconstruct_{abs,rel}{32,64}: returns the value bit patterns (int tensor)."""
    cb = as_bits(codes)
    width = _width_of(cb)
    n = cb.numel()
    if lossless.dtype == torch.bool:
        lossless = lossless.view(torch.uint8)
    if out is None:
        out = torch.empty(n, dtype=_ITYPE[width], device=cb.device)
    sfx = "f32" if width == 32 else "f64"
    kind = "rel" if mode == REL else "abs"
    _lib.call(f"gebq_dequantize_{kind}_{sfx}", _p(cb), _p(lossless.contiguous()), _p(out), n,
              _f(width)(derived), _s())
    return out


# ---------------------------------------------------------------------------
# NOA range pass
# ---------------------------------------------------------------------------

def noa_keys(x: torch.Tensor, keys: Optional[torch.Tensor] = None) -> torch.Tensor:
    """int64[2] order keys of (max, min) over the finite values -- MAX-combinable."""
    xb = as_bits(x)
    width = _width_of(xb)
    if keys is None:
        keys = torch.empty(2, dtype=torch.int64, device=xb.device)
    _lib.call(f"gebq_noa_minmax_{'f32' if width == 32 else 'f64'}", _p(xb), xb.numel(), _p(keys),
              _s())
    return keys


def noa_derive(keys: torch.Tensor, eb: float, width: int):
    """keys -> (consts_dev [eb_eff, eb2, inv_eb2, thr] in the value width, range_f64[1])."""
    consts = torch.empty(4, dtype=_FTYPE[width], device=keys.device)
    rng = torch.empty(1, dtype=torch.float64, device=keys.device)
    _lib.call(f"gebq_noa_derive_{'f32' if width == 32 else 'f64'}", _p(keys), float(eb),
              _p(consts), _p(rng), _s())
    return consts, rng


def noa_range_host(arr: np.ndarray):
    """compute_noa_range for a host array: the value-dtype scalar R."""
    dev = require_cuda()
    width = 32 if arr.dtype == np.float32 else 64
    ft = np.float32 if width == 32 else np.float64
    if arr.size == 0:
        return ft(0.0)
    x = torch.from_numpy(arr.view(_NP_SITYPE[width])).to(dev)
    keys = noa_keys(x)
    _, rng = noa_derive(keys, 1.0, width)
    return ft(rng.item())


# ---------------------------------------------------------------------------
# sweeps
# ---------------------------------------------------------------------------

SOURCE_RANGE, SOURCE_ARRAY, SOURCE_SPLITMIX = 0, 1, 2


def sweep(cfg: QuantConfig, *, source: int, count: int, start: int = 0,
          bits: Optional[torch.Tensor] = None, seed: int = 0, tally=None, first=None):
    """Accumulate (tally[15] i64, first_violation u64-as-i64) device tensors for one sweep."""
    dev = require_cuda()
    width = cfg.width
    if tally is None:
        tally = torch.zeros(15, dtype=torch.int64, device=dev)
    if first is None:
        first = torch.full((1,), -1, dtype=torch.int64, device=dev)  # UINT64_MAX
    d = cfg.derived
    F = _f(width)
    sfx = "f32" if width == 32 else "f64"
    bp = _p(as_bits(bits)) if bits is not None else ctypes.c_void_p(0)
    unsafe = int(bool(cfg.unsafe_no_double_check))
    if cfg.mode == REL:
        _lib.call(f"gebq_sweep_rel_{sfx}", source, bp, start & (2 ** 64 - 1), count,
                  seed & (2 ** 64 - 1), F(d.op_eps), F(d.w), F(d.thr), unsafe, _p(tally),
                  _p(first), _s())
    else:
        _lib.call(f"gebq_sweep_abs_{sfx}", source, bp, start & (2 ** 64 - 1), count,
                  seed & (2 ** 64 - 1), F(d.eb_eff), F(d.eb2), F(d.inv_eb2), F(d.thr), unsafe,
                  _p(tally), _p(first), _s())
    return tally, first


# ---------------------------------------------------------------------------
# generators
# ---------------------------------------------------------------------------

def splitmix64(n: int, seed: int, start_index: int = 0, device=None) -> torch.Tensor:
    dev = require_cuda(device)
    out = torch.empty(n, dtype=torch.int64, device=dev)
    _lib.call("gebq_splitmix64_fill", _p(out), n, seed & (2 ** 64 - 1), start_index, _s())
    return out


def mixed_f32(n: int, seed: int, start_index: int = 0, device=None) -> torch.Tensor:
    """C2 mixed-class f32 patterns as an int32 tensor."""
    dev = require_cuda(device)
    out = torch.empty(n, dtype=torch.int32, device=dev)
    _lib.call("gebq_gen_mixed_f32", _p(out), n, seed & (2 ** 64 - 1), start_index, _s())
    return out


def smooth_field(n: int, side: int, seed: int, start_index: int = 0, width: int = 32,
                 plant: bool = True, total: Optional[int] = None, device=None) -> torch.Tensor:
    """Counter-based C3 / C5-smooth field (``workloads.smooth_field_cb``) as an
    int32 / int64 bit tensor, generated on the device from the global index."""
    from . import workloads

    dev = require_cuda(device)
    total = side ** 3 if total is None else total
    tab = torch.from_numpy(workloads.smooth_tables(side).reshape(-1).copy()).to(dev)
    out = torch.empty(n, dtype=_ITYPE[width], device=dev)
    _lib.call("gebq_gen_smooth", width, _p(out), n, side, _p(tab), seed & (2 ** 64 - 1), start_index,
              int(bool(plant)), total, workloads.SMOOTH_NOISE_SCALE, _s())
    return out


# ---------------------------------------------------------------------------
# host conveniences (numpy in / numpy out) used by the drop-in shims
# ---------------------------------------------------------------------------

def to_device(a: np.ndarray, device=None) -> torch.Tensor:
    dev = require_cuda(device)
    a = np.ascontiguousarray(a)
    if a.dtype in (np.uint32, np.float32):
        a = a.view(np.int32)
    elif a.dtype in (np.uint64, np.float64):
        a = a.view(np.int64)
    elif a.dtype == np.bool_:
        a = a.view(np.uint8)
    return torch.from_numpy(a).to(dev, non_blocking=False)


def to_host(t: torch.Tensor, np_dtype) -> np.ndarray:
    return t.cpu().numpy().view(np_dtype)


def quantize_host(bits: np.ndarray, cfg: QuantConfig):
    """numpy bits -> (codes, lossless bool, trig int64[4]) through the GPU kernels."""
    width = 32 if bits.dtype in (np.uint32, np.float32, np.int32) else 64
    if cfg.mode == NOA and cfg.value_range is None:
        raise ValueError("NOA constants need the data range; run the range pass first")
    if bits.size == 0:
        return (np.empty(0, _NP_ITYPE[width]), np.empty(0, np.bool_), np.zeros(4, np.int64))
    x = to_device(bits)
    codes, lossless, trig = quantize(x, cfg)
    return (to_host(codes, _NP_ITYPE[width]), to_host(lossless, np.uint8).view(np.bool_),
            trig.cpu().numpy().astype(np.int64))


def reconstruct_host(codes: np.ndarray, lossless: np.ndarray, mode: str, derived) -> np.ndarray:
    width = 32 if codes.dtype in (np.uint32, np.int32) else 64
    if codes.size == 0:
        return np.empty(0, _NP_ITYPE[width])
    out = reconstruct(to_device(codes), to_device(np.asarray(lossless, dtype=np.bool_)), mode,
                      derived)
    return to_host(out, _NP_ITYPE[width])


def derive_for(mode: str, eb: float, width: int, value_range=None):
    return _derive(mode, eb, width, value_range)
