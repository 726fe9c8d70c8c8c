"""Shared test helpers: fixture decoding and value generators."""

import numpy as np

CLASS_NAMES = ("zero", "denormal", "normal", "infinity", "nan")
OUTCOME_NAMES = ("quantized", "lossless", "violation")


def tally_from_per_class(per_class) -> np.ndarray:
    t = np.zeros((5, 3), dtype=np.int64)
    for ci, c in enumerate(CLASS_NAMES):
        for oi, o in enumerate(OUTCOME_NAMES):
            t[ci, oi] = per_class[c][o]
    return t


def trig_list(triggers: dict):
    return [triggers["nan"], triggers["inf"], triggers["guard"], triggers["double_check"]]


def noa_input(rec):
    """Rebuild a NOA-range input from its fixture record (make_golden.noa_input)."""
    if "hex" in rec:
        return np.frombuffer(bytes.fromhex(rec["hex"]), dtype=rec["dtype"]).copy()
    rng = np.random.default_rng(rec["seed"])
    x = rng.standard_normal(rec["n"]) * rec["scale"]
    return x.astype(rec["dtype"])


def stream_values(width, seed):
    """The mixed + smooth corpus behind fixtures['streams'] (make_golden.gen_streams)."""
    ft = np.float32 if width == 32 else np.float64
    bits = mixed_bits(width, 20000, seed)
    return np.concatenate([bits.view(ft), (np.cos(np.linspace(0, 90, 30000)) * 3).astype(ft)])


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


def verify_numpy(o, r, mode, d, value_range=None):
    """numpy restatement of the reference's verify predicates (verify.py:88-153):
    returns (violations, first_violation_index, special_mismatch_count, max_err)."""
    itype = np.uint32 if o.dtype == np.float32 else np.uint64
    ob, rb = o.view(itype), r.view(itype)
    eq = ob == rb
    special = np.isnan(o) | np.isinf(o)
    spec = int(np.count_nonzero(special & ~eq))
    inexact = ~special & ~eq
    with np.errstate(all="ignore"):
        if mode == "rel":
            q = np.abs(r) / np.abs(o)
            ok = (np.signbit(o) == np.signbit(r)) & (q <= d["op_eps"]) & (q * d["op_eps"] >= o.dtype.type(1.0))
            dev = np.abs(q[inexact].astype(np.float64) - 1.0)
        else:
            err = np.abs(o - r)
            ok = err <= d["eb_eff"]
            dev = err[inexact].astype(np.float64)
    mx = float(np.max(np.where(np.isnan(dev), np.inf, dev))) if dev.size else 0.0
    bad = ~special & ~(eq | ok)
    viol = int(np.count_nonzero(bad))
    first = int(np.flatnonzero(bad)[0]) if viol else None
    return viol, first, spec, mx
