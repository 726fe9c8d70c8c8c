"""ctypes binding of libgebq_b200.so (the C ABI in include/gebq_b200.h).

There is deliberately no fallback: if the CUDA library is missing or no GPU
is visible, every call raises.  Build it with ``python -m
paper_2407_15037_b200._build`` (or ``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes
import os
import threading

LIB_PATH = os.environ.get("GEBQ_B200_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                            "libgebq_b200.so")


class GebqCudaError(RuntimeError):
    """A CUDA launch or runtime error reported by libgebq_b200.so."""


_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_f32 = ctypes.c_float
_f64 = ctypes.c_double
_int = ctypes.c_int

# name -> argtypes (all return int status unless listed in _RESTYPES)
SIGNATURES = {
    "gebq_b200_abi_version": [],
    "gebq_b200_last_error": [],
    "gebq_b200_sm_count": [],
    "gebq_b200_launch_count": [],
    "gebq_quantize_abs_f32": [_vp, _vp, _vp, _i64, _f32, _f32, _f32, _f32, _int, _vp, _vp],
    "gebq_quantize_abs_f64": [_vp, _vp, _vp, _i64, _f64, _f64, _f64, _f64, _int, _vp, _vp],
    "gebq_quantize_rel_f32": [_vp, _vp, _vp, _i64, _f32, _f32, _f32, _int, _vp, _vp],
    "gebq_quantize_rel_f64": [_vp, _vp, _vp, _i64, _f64, _f64, _f64, _int, _vp, _vp],
    "gebq_quantize_noa_dev_f32": [_vp, _vp, _vp, _i64, _vp, _int, _vp, _vp],
    "gebq_quantize_noa_dev_f64": [_vp, _vp, _vp, _i64, _vp, _int, _vp, _vp],
    "gebq_dequantize_abs_f32": [_vp, _vp, _vp, _i64, _f32, _vp],
    "gebq_dequantize_abs_f64": [_vp, _vp, _vp, _i64, _f64, _vp],
    "gebq_dequantize_rel_f32": [_vp, _vp, _vp, _i64, _f32, _vp],
    "gebq_dequantize_rel_f64": [_vp, _vp, _vp, _i64, _f64, _vp],
    "gebq_noa_minmax_f32": [_vp, _i64, _vp, _vp],
    "gebq_noa_minmax_f64": [_vp, _i64, _vp, _vp],
    "gebq_noa_allreduce": [_vp, _vp, _vp],
    "gebq_noa_derive_f32": [_vp, _f64, _vp, _vp, _vp],
    "gebq_noa_derive_f64": [_vp, _f64, _vp, _vp, _vp],
    "gebq_sweep_abs_f32": [_int, _vp, _u64, _i64, _u64, _f32, _f32, _f32, _f32, _int, _vp, _vp, _vp],
    "gebq_sweep_rel_f32": [_int, _vp, _u64, _i64, _u64, _f32, _f32, _f32, _int, _vp, _vp, _vp],
    "gebq_sweep_abs_f64": [_int, _vp, _u64, _i64, _u64, _f64, _f64, _f64, _f64, _int, _vp, _vp, _vp],
    "gebq_sweep_rel_f64": [_int, _vp, _u64, _i64, _u64, _f64, _f64, _f64, _int, _vp, _vp, _vp],
    "gebq_splitmix64_fill": [_vp, _i64, _u64, _i64, _vp],
    "gebq_gen_mixed_f32": [_vp, _i64, _u64, _i64, _vp],
    "gebq_gen_smooth": [_int, _vp, _i64, _i64, _vp, _u64, _i64, _int, _i64, _f64, _vp],
    "gebq_quantize_rel_lib_f32": [_vp, _vp, _vp, _i64, _f32, _f32, _f32, _int, _vp, _vp],
    "gebq_dequantize_rel_lib_f32": [_vp, _vp, _vp, _i64, _f32, _vp],
    "gebq_verify_f32": [_vp, _vp, _i64, _int, _f32, _vp, _vp, _vp],
    "gebq_verify_f64": [_vp, _vp, _i64, _int, _f64, _vp, _vp, _vp],
    "gebq_encode_region_capacity": [_i64, _i64, _int],
    "gebq_encode_workspace_bytes": [_i64, _i64, _int],
    "gebq_encode_abs_f32": [_vp, _i64, _f32, _f32, _f32, _f32, _int, _i64, _vp, _vp, _i64, _vp,
                            ctypes.c_size_t, _vp, _vp, _vp],
    "gebq_encode_abs_f64": [_vp, _i64, _f64, _f64, _f64, _f64, _int, _i64, _vp, _vp, _i64, _vp,
                            ctypes.c_size_t, _vp, _vp, _vp],
    "gebq_encode_rel_f32": [_vp, _i64, _f32, _f32, _f32, _int, _i64, _vp, _vp, _i64, _vp,
                            ctypes.c_size_t, _vp, _vp, _vp],
    "gebq_encode_rel_f64": [_vp, _i64, _f64, _f64, _f64, _int, _i64, _vp, _vp, _i64, _vp,
                            ctypes.c_size_t, _vp, _vp, _vp],
    "gebq_encode_noa_dev_f32": [_vp, _i64, _vp, _int, _i64, _vp, _vp, _i64, _vp, ctypes.c_size_t,
                                _vp, _vp, _vp],
    "gebq_encode_noa_dev_f64": [_vp, _i64, _vp, _int, _i64, _vp, _vp, _i64, _vp, ctypes.c_size_t,
                                _vp, _vp, _vp],
    "gebq_encode_coded_u32": [_vp, _vp, _i64, _i64, _vp, _vp, _i64, _vp, ctypes.c_size_t, _vp, _vp],
    "gebq_encode_coded_u64": [_vp, _vp, _i64, _i64, _vp, _vp, _i64, _vp, ctypes.c_size_t, _vp, _vp],
    "gebq_validate_index": [_vp, _i64, _i64, _vp, _vp],
    "gebq_decode_abs_f32": [_vp, _i64, _vp, _vp, _i64, _i64, _i64, _f32, _vp, _vp, _vp, _vp],
    "gebq_decode_abs_f64": [_vp, _i64, _vp, _vp, _i64, _i64, _i64, _f64, _vp, _vp, _vp, _vp],
    "gebq_decode_rel_f32": [_vp, _i64, _vp, _vp, _i64, _i64, _i64, _f32, _vp, _vp, _vp, _vp],
    "gebq_decode_rel_f64": [_vp, _i64, _vp, _vp, _i64, _i64, _i64, _f64, _vp, _vp, _vp, _vp],
    "gebq_decode_span_abs_f32": [_vp, _i64, _vp, _i64, _i64, _i64, _f32, _i64, _i64, _vp, _vp, _vp],
    "gebq_decode_span_abs_f64": [_vp, _i64, _vp, _i64, _i64, _i64, _f64, _i64, _i64, _vp, _vp, _vp],
    "gebq_decode_span_rel_f32": [_vp, _i64, _vp, _i64, _i64, _i64, _f32, _i64, _i64, _vp, _vp, _vp],
    "gebq_decode_span_rel_f64": [_vp, _i64, _vp, _i64, _i64, _i64, _f64, _i64, _i64, _vp, _vp, _vp],
    "gebq_selfcheck_abs_f32": [_u64, _i64, _f32, _f32, _f32, _f32, _int, _vp, _vp],
    "gebq_selfcheck_rel_filter_f32": [_u64, _i64, _f32, _f32, _f32, _int, _vp, _vp],
    "gebq_selfcheck_abs_f64": [_u64, _i64, _f64, _f64, _f64, _f64, _int, _vp, _vp],
    "gebq_selfcheck_rel_f64": [_u64, _i64, _f64, _f64, _f64, _int, _vp, _vp],
    "gebq_selfcheck_div_f32": [_u64, _i64, _vp, _vp],
    "gebq_decode_blocks_u32": [_vp, _vp, _i64, _i64, _i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp],
    "gebq_decode_blocks_u64": [_vp, _vp, _i64, _i64, _i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp],
    "gebq_block_sizes_u32": [_vp, _i64, _i64, _i64, _i64, _vp, _vp],
    "gebq_block_sizes_u64": [_vp, _i64, _i64, _i64, _i64, _vp, _vp],
    "gebq_emit_blocks_u32": [_vp, _vp, _i64, _i64, _i64, _i64, _vp, _vp, _vp],
    "gebq_emit_blocks_u64": [_vp, _vp, _i64, _i64, _i64, _i64, _vp, _vp, _vp],
}
_RESTYPES = {"gebq_b200_last_error": ctypes.c_char_p, "gebq_b200_launch_count": ctypes.c_ulonglong, "gebq_encode_region_capacity": _i64,
             "gebq_encode_workspace_bytes": ctypes.c_size_t}

_lock = threading.Lock()
_lib = None


def load():
    """Load (once) and return the CDLL; raises if the library was not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: build the CUDA backend with "
                    "`python -m paper_2407_15037_b200._build` (nvcc, sm_100a)")
            L = ctypes.CDLL(LIB_PATH)
            for name, args in SIGNATURES.items():
                fn = getattr(L, name)
                fn.argtypes = args
                fn.restype = _RESTYPES.get(name, ctypes.c_int)
            _lib = L
    return _lib


def last_error() -> str:
    return load().gebq_b200_last_error().decode(errors="replace")


def call(name: str, *args) -> int:
    """Invoke one C-ABI entry point; raise GebqCudaError on a nonzero status."""
    rc = getattr(load(), name)(*args)
    if rc != 0:
        raise GebqCudaError(f"{name} failed ({rc}): {last_error()}")
    return rc


def exported_symbols() -> list[str]:
    return list(SIGNATURES)


def launch_count() -> int:
    """Kernels launched by libgebq_b200.so so far in this process."""
    return int(load().gebq_b200_launch_count())
