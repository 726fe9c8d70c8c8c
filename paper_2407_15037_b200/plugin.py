"""Plug the B200 kernels into an installed reference ``gebq`` package.

The reference resolves its hot-path operators by module-attribute lookup at
call time -- ``_kernels.quantize_*`` (pipeline.py:106-109), ``reconstruct_*``
(pipeline.py:203-206), ``block_sizes_*`` / ``emit_blocks_*`` /
``decode_blocks_*`` (container.py:243-305), ``sweep_*_on`` (sweep.py:96-102)
and ``splitmix64_fill`` (verify.py:185-194) -- and ``compute_noa_range`` is
bound by name into ``gebq.pipeline`` (pipeline.py:21-28).  ``install``
rebinds exactly those names to the drop-ins in ``_kernels`` / ``quantizers``,
so ``gebq.compress`` / ``decompress_to_array`` / ``sweep_f32`` run their
per-element work on the GPU with unchanged Python around it.
"""

from __future__ import annotations

import importlib

_SAVED: dict = {}

KERNEL_NAMES = (
    "quantize_abs32", "quantize_abs64", "quantize_rel32", "quantize_rel64",
    "reconstruct_abs32", "reconstruct_abs64", "reconstruct_rel32", "reconstruct_rel64",
    "block_sizes_u32", "block_sizes_u64", "emit_blocks_u32", "emit_blocks_u64",
    "decode_blocks_u32", "decode_blocks_u64", "sweep_abs32_on", "sweep_abs64_on",
    "sweep_rel32_on", "sweep_rel64_on", "splitmix64_fill", "quantize_rel32_lib",
    "reconstruct_rel32_lib",
)


def install(gebq_module) -> None:
    """Rebind ``gebq._kernels.*`` and ``gebq.pipeline.compute_noa_range`` to the B200 path."""
    from . import _kernels as ours
    from .quantizers import compute_noa_range

    ours_lib = importlib.import_module("paper_2407_15037_b200._lib")
    ours_lib.load()  # fail loudly now if the CUDA backend is missing
    ref_kernels = importlib.import_module(gebq_module.__name__ + "._kernels")
    ref_pipeline = importlib.import_module(gebq_module.__name__ + ".pipeline")
    key = gebq_module.__name__
    if key not in _SAVED:
        _SAVED[key] = ({n: getattr(ref_kernels, n) for n in KERNEL_NAMES},
                       ref_pipeline.compute_noa_range)
    for n in KERNEL_NAMES:
        setattr(ref_kernels, n, getattr(ours, n))
    ref_pipeline.compute_noa_range = compute_noa_range


def uninstall(gebq_module) -> None:
    key = gebq_module.__name__
    if key not in _SAVED:
        return
    kernels, cnr = _SAVED.pop(key)
    ref_kernels = importlib.import_module(key + "._kernels")
    ref_pipeline = importlib.import_module(key + ".pipeline")
    for n, f in kernels.items():
        setattr(ref_kernels, n, f)
    ref_pipeline.compute_noa_range = cnr
