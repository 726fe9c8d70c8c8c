"""Synthetic inputs for the BASELINE.json configurations.

Host (numpy) recipes are the normative definitions; the device generators in
``device.py`` reproduce the integer-only recipes bit-for-bit on the GPU so
that 2^26..2^30-element inputs never have to cross PCIe.

* C1 -- ABS f32 eb=1e-3, 256^3 smooth field:
  x[i,j,k] = f32(5 sin(2 pi i/256) cos(2 pi j/256) sin(2 pi k/128) + 0.02 z),
  z = default_rng(0).standard_normal((256,)*3), f64 math then one cast.
* C2 -- REL f32 eb=1e-2, 2^26 mixed values, integer-only splitmix64 recipe
  (seed 0x5EED0002); exercises every outlier path.
* C3 -- NOA f32 eb=1e-4, 2^30 values: the 1024^3 version of the C1 formula
  (periods 1024/1024/512) with planted NaN/+Inf and min -7 / max +7 at the two
  ends so the range needs the global reduction.  The noise is counter-based
  (``smooth_field_cb``): a function of the GLOBAL index only, built from
  IEEE-exact binary64 operations on host-computed sine tables, so the device
  generator (``device.smooth_field``), this numpy recipe, every shard of every
  world size and the CPU baseline see identical bits.
* C5 -- f64: (i) raw splitmix64 words, seed 0x5EED0005; (ii) the smooth field
  (``smooth_field_cb`` in binary64, seed C5_SMOOTH_SEED, not planted).
"""

from __future__ import annotations

import numpy as np

C2_SEED = 0x5EED0002
C5_SEED = 0x5EED0005
C3_SEED = 0x5EED0003
C5_SMOOTH_SEED = 0x5EED0015
C3_SIDE = 1024
# 0.02 / std of the sum of four uniform 16-bit integers: unit-variance noise x 0.02
SMOOTH_NOISE_SCALE = 0.02 / float(np.sqrt(4.0 * (65536.0 ** 2 - 1.0) / 12.0))


def splitmix64(n: int, seed: int, start_index: int = 0) -> np.ndarray:
    """splitmix64 output numbers start_index+1 .. start_index+n (vectorised numpy).

    Same recurrence as the reference's ``splitmix64_fill`` (_kernels.py:671-685).
    """
    with np.errstate(over="ignore"):
        idx = np.arange(start_index + 1, start_index + n + 1, dtype=np.uint64)
        z = np.uint64(seed) + np.uint64(0x9E3779B97F4A7C15) * idx
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def c2_bits_from_words(w: np.ndarray) -> np.ndarray:
    """map splitmix64 words to mixed-class f32 patterns."""
    w = w.astype(np.uint64)
    sel = w >> np.uint64(56)
    sign = ((w >> np.uint64(55)) & np.uint64(1)) << np.uint64(31)
    lo = w & np.uint64(0xFFFFFFFF)
    mant = lo & np.uint64(0x7FFFFF)
    default = sign | ((np.uint64(107) + (w >> np.uint64(32)) % np.uint64(41)) << np.uint64(23)) | mant
    out = default
    out = np.where(sel < 16, sign | (np.uint64(0x7F7FFF00) + (lo & np.uint64(0xFF))), out)
    out = np.where(sel < 12, sign | mant, out)
    out = np.where(sel < 8, sign | np.uint64(0x7F800000), out)
    out = np.where(sel < 4, sign | np.uint64(0x7F800000) | (mant | np.uint64(1)), out)
    return out.astype(np.uint32)


def c2_values(n: int = 1 << 26, seed: int = C2_SEED, start_index: int = 0) -> np.ndarray:
    return c2_bits_from_words(splitmix64(n, seed, start_index)).view(np.float32)


def smooth_field(side: int = 256, seed: int = 0, dtype=np.float32) -> np.ndarray:
    """C1 (side=256) field; C3 uses side=1024 with seed 1 (host version)."""
    rng = np.random.default_rng(seed)
    z = rng.standard_normal((side,) * 3)
    i = np.arange(side, dtype=np.float64)
    a = np.sin(2 * np.pi * i / side)[:, None, None]
    b = np.cos(2 * np.pi * i / side)[None, :, None]
    c = np.sin(2 * np.pi * i / (side // 2))[None, None, :]
    x = 5.0 * a * b * c + 0.02 * z
    return x.astype(dtype).ravel()


def smooth_tables(side: int) -> np.ndarray:
    """(3, side) binary64: sin(2 pi i/side), cos(2 pi j/side), sin(2 pi k/(side/2))."""
    i = np.arange(side, dtype=np.float64)
    return np.stack([np.sin(2 * np.pi * i / side), np.cos(2 * np.pi * i / side),
                     np.sin(2 * np.pi * i / (side // 2))])


def smooth_field_cb(n: int, side: int = C3_SIDE, seed: int = C3_SEED, start_index: int = 0,
                    dtype=np.float32, plant: bool = True, total: int | None = None,
                    chunk: int = 1 << 22) -> np.ndarray:
    """Counter-based smooth field, values g = start_index .. start_index+n-1.

    v = ((5 * A[ii]) * B[j]) * C[k] + (s - 131070) * SMOOTH_NOISE_SCALE, each
    operation one binary64 rounding (numpy elementwise ops are IEEE, no
    contraction), s = sum of the four 16-bit fields of splitmix64(seed, g+1);
    (ii, j, k) are the base-``side`` digits of g.  Planted (C3): g=0 NaN,
    g=1 +Inf, g=2 -7, g=total-1 +7.  Same recipe as ``k_gen_smooth``."""
    total = side ** 3 if total is None else total
    tab = smooth_tables(side)
    out = np.empty(n, dtype=dtype)
    for c0 in range(0, n, chunk):
        m = min(chunk, n - c0)
        g = np.arange(start_index + c0, start_index + c0 + m, dtype=np.int64)
        w = splitmix64(m, seed, start_index + c0)
        s = ((w & np.uint64(0xFFFF)) + ((w >> np.uint64(16)) & np.uint64(0xFFFF))
             + ((w >> np.uint64(32)) & np.uint64(0xFFFF)) + (w >> np.uint64(48))).astype(np.int64)
        noise = (s - 131070).astype(np.float64) * SMOOTH_NOISE_SCALE
        k = g % side
        j = (g // side) % side
        ii = (g // (side * side)) % side
        v = 5.0 * tab[0][ii]
        v = v * tab[1][j]
        v = v * tab[2][k]
        v = v + noise
        if plant:
            for gi, val in ((0, np.nan), (1, np.inf), (2, -7.0), (total - 1, 7.0)):
                if start_index + c0 <= gi < start_index + c0 + m:
                    v[gi - start_index - c0] = val
        out[c0:c0 + m] = v.astype(dtype)
    return out


def plant_noa_extremes(x: np.ndarray) -> np.ndarray:
    """C3: NaN at x[0], +Inf at x[1], global min -7 in the first block and max +7
    in the last block, so R = 14 needs a cross-shard reduction."""
    x = x.copy()
    x[0] = np.nan
    x[1] = np.inf
    x[2] = -7.0
    x[-1] = 7.0
    return x


def c5_random_values(n: int, seed: int = C5_SEED) -> np.ndarray:
    return splitmix64(n, seed).view(np.float64)
