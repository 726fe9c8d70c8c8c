"""Fixture for the library-log REL variant, produced by running the REFERENCE.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_lib_variant.py

Writes tests/golden/lib_variant.npz: inputs and the reference's
quantize_rel32_lib / reconstruct_rel32_lib outputs (_kernels.py:356-431).
The variant uses the platform binary64 log2/exp2 and is non-conforming by
design, so the GPU test checks the bound and the agreement rate, not bits.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from gebq import _kernels  # noqa: E402  (the reference, via PYTHONPATH)
from gebq.quantizers import QuantConfig  # noqa: E402

from paper_2407_15037_b200 import workloads  # noqa: E402  (input recipes only)


def main():
    x = workloads.c2_values(1 << 16)
    out = {"x": x.view(np.uint32)}
    for eb in (1e-2, 1e-3):
        d = QuantConfig(mode="rel", eb=eb, width=32).derived
        codes = np.empty(len(x), np.uint32)
        ll = np.empty(len(x), np.bool_)
        trig = _kernels.quantize_rel32_lib(x.view(np.uint32), x, codes, ll, d.op_eps, d.w, d.thr, False)
        rec = np.empty(len(x), np.float32)
        _kernels.reconstruct_rel32_lib(codes, ll, rec.view(np.uint32), rec, d.w)
        tag = f"{eb:g}"
        out[f"codes_{tag}"] = codes
        out[f"lossless_{tag}"] = ll
        out[f"trig_{tag}"] = np.asarray(trig, np.int64)
        out[f"recon_{tag}"] = rec.view(np.uint32)
    np.savez_compressed(os.path.join(HERE, "lib_variant.npz"), **out)
    print({k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
