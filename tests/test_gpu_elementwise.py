"""GPU parity: CodedArray-level quantize / reconstruct, NOA range, sweeps and
generators, bit-exact against the reference fixtures and the CPU oracle."""

import numpy as np
import pytest
import torch

from helpers import mixed_bits, noa_input, tally_from_per_class, trig_list

pytestmark = pytest.mark.gpu


def _cfg(mode, eb, width, vr=None, unsafe=False):
    from paper_2407_15037_b200.quantizers import QuantConfig

    return QuantConfig(mode=mode, eb=eb, width=width, value_range=vr, unsafe_no_double_check=unsafe)


def test_kernel_cases(cuda, fixtures, kernel_arrays):
    from paper_2407_15037_b200 import device

    for meta in fixtures["kernel_cases"]:
        ci = meta["key"].split("_")[0]
        bits = kernel_arrays[ci + "_bits"]
        cfg = _cfg(meta["mode"], meta["eb"], meta["width"], meta["value_range"], meta["unsafe"])
        codes, lossless, trig = device.quantize_host(bits, cfg)
        np.testing.assert_array_equal(codes, kernel_arrays[meta["key"] + "_codes"])
        np.testing.assert_array_equal(lossless, kernel_arrays[meta["key"] + "_lossless"])
        assert list(trig) == trig_list(meta["triggers"]), meta
        if not meta["unsafe"]:
            rec = device.reconstruct_host(codes, lossless, meta["mode"], cfg.derived.derived_value)
            np.testing.assert_array_equal(rec, kernel_arrays[meta["key"] + "_recon"])


def test_reconstruct_adversarial(cuda, fixtures, kernel_arrays):
    from paper_2407_15037_b200 import device

    for meta in fixtures["reconstruct_cases"]:
        k = meta["key"]
        w = meta["width"]
        d = (np.uint32(meta["derived_bits"]).view(np.float32) if w == 32
             else np.uint64(meta["derived_bits"]).view(np.float64))
        out = device.reconstruct_host(kernel_arrays[k + "_codes"], kernel_arrays[k + "_lossless"],
                                      meta["mode"], d)
        np.testing.assert_array_equal(out, kernel_arrays[k + "_out"])


@pytest.mark.parametrize("width", [32, 64])
@pytest.mark.parametrize("mode,eb,vr", [("abs", 1e-3, None), ("rel", 1e-2, None),
                                        ("rel", 1e-5, None), ("noa", 1e-4, 3.5),
                                        ("abs", 1e-7, None)])
@pytest.mark.parametrize("unsafe", [False, True])
def test_large_vs_oracle(cuda, oracle, width, mode, eb, vr, unsafe):
    """2^21+ mixed patterns + a smooth field, every offset/tail case, against the oracle."""
    from paper_2407_15037_b200 import device

    ft = np.float32 if width == 32 else np.float64
    n = (1 << 21) + 4093
    bits = mixed_bits(width, n // 2, 17 + width)
    smooth = (np.sin(np.linspace(0, 3000, n - len(bits))) * 7.0).astype(ft).view(bits.dtype)
    bits = np.concatenate([bits, smooth])
    cfg = _cfg(mode, eb, width, vr, unsafe)
    c = oracle.derive(mode, eb, width, vr)
    exp_codes, exp_ll, exp_trig = oracle.quantize(bits, mode, c, unsafe)
    codes, ll, trig = device.quantize_host(bits, cfg)
    np.testing.assert_array_equal(codes, exp_codes)
    np.testing.assert_array_equal(ll, exp_ll)
    np.testing.assert_array_equal(trig, exp_trig)
    exp_rec = oracle.reconstruct(exp_codes, exp_ll, mode, c["header"])
    rec = device.reconstruct_host(codes, ll, mode, cfg.derived.derived_value)
    np.testing.assert_array_equal(rec, exp_rec)


@pytest.mark.parametrize("offset", [1, 3, 5])
def test_misaligned_views(cuda, oracle, offset):
    """Unaligned device views take the scalar path and must agree bit-for-bit."""
    from paper_2407_15037_b200 import device

    bits = mixed_bits(32, 50000, 5)
    cfg = _cfg("rel", 1e-3, 32)
    x = device.to_device(bits)
    view = x[offset:]
    codes, ll, trig = device.quantize(view, cfg)
    c = oracle.derive("rel", 1e-3, 32)
    ec, el, et = oracle.quantize(bits[offset:], "rel", c)
    np.testing.assert_array_equal(codes.cpu().numpy().view(np.uint32), ec)
    np.testing.assert_array_equal(ll.cpu().numpy().view(np.bool_), el)
    np.testing.assert_array_equal(trig.cpu().numpy(), et)


def test_noa_range(cuda, fixtures):
    from paper_2407_15037_b200.quantizers import compute_noa_range

    for rec in fixtures["noa"]:
        arr = noa_input(rec)
        r = compute_noa_range(arr)
        assert r.dtype == arr.dtype
        bits = int(np.float32(r).view(np.uint32)) if arr.dtype == np.float32 else int(np.float64(r).view(np.uint64))
        assert bits == rec["range_bits"], rec["name"]


@pytest.mark.parametrize("width", [32, 64])
def test_noa_device_chain(cuda, oracle, width):
    """minmax -> derive -> quantize with device-resident constants == host-derived path."""
    from paper_2407_15037_b200 import device, workloads

    ft = np.float32 if width == 32 else np.float64
    x = workloads.plant_noa_extremes(workloads.smooth_field(64, 3, ft))
    xd = device.to_device(x)
    keys = device.noa_keys(xd)
    consts, rng = device.noa_derive(keys, 1e-4, width)
    R = oracle.noa_range(x)
    assert rng.item() == float(R) == 14.0
    cfg = _cfg("noa", 1e-4, width, float(R))
    codes, ll, trig = device.quantize(xd, cfg, consts_dev=consts)
    c = oracle.derive("noa", 1e-4, width, float(R))
    ec, el, et = oracle.quantize(x.view(np.uint32 if width == 32 else np.uint64), "abs", c)
    np.testing.assert_array_equal(codes.cpu().numpy().view(ec.dtype), ec)
    np.testing.assert_array_equal(ll.cpu().numpy().view(np.bool_), el)
    np.testing.assert_array_equal(trig.cpu().numpy(), et)


def _sweep_host(cfg, **kw):
    from paper_2407_15037_b200 import device

    tally, first = device.sweep(cfg, **kw)
    f = int(first.item()) & (2**64 - 1)
    return tally.cpu().numpy().reshape(5, 3), (None if f == 2**64 - 1 else f)


def test_sweep_subranges(cuda, sweeps_fixture):
    from paper_2407_15037_b200 import device

    for rec in sweeps_fixture["subrange"]:
        cfg = _cfg(rec["mode"], rec["eb"], 32, rec["value_range"], rec["unsafe"])
        tally, first = _sweep_host(cfg, source=device.SOURCE_RANGE, start=rec["start"],
                                   count=rec["count"])
        np.testing.assert_array_equal(tally, tally_from_per_class(rec["per_class"]))
        exp = rec["first_violation_bits"]
        assert (None if first is None else (rec["start"] + first) & 0xFFFFFFFF) == exp


def test_sweep_full_appendix_b(cuda, sweeps_fixture):
    """All 11 exhaustive 2^32 sweeps of SURVEY Appendix B: tallies exact, 0 violations."""
    from paper_2407_15037_b200 import device

    for rec in sweeps_fixture["full"]:
        cfg = _cfg(rec["mode"], rec["eb"], 32, rec["value_range"])
        tally, first = _sweep_host(cfg, source=device.SOURCE_RANGE, start=0, count=1 << 32)
        np.testing.assert_array_equal(tally, tally_from_per_class(rec["per_class"]))
        assert first is None


def test_sweep_f64_and_random(cuda, sweeps_fixture):
    from paper_2407_15037_b200 import device
    from paper_2407_15037_b200.workloads import splitmix64

    for rec in sweeps_fixture["f64"]:
        words = splitmix64(4 * 2048, rec["seed"], 0)
        mants = np.concatenate([np.zeros((2048, 1), np.uint64),
                                np.full((2048, 1), (1 << 52) - 1, np.uint64),
                                (words & np.uint64((1 << 52) - 1)).reshape(2048, 4)], axis=1)
        base = ((np.arange(2048, dtype=np.uint64) << np.uint64(52))[:, None] | mants).ravel()
        structured = np.concatenate([base, base | np.uint64(1 << 63)])
        cfg = _cfg(rec["mode"], rec["eb"], 64)
        t1, _ = _sweep_host(cfg, source=device.SOURCE_ARRAY, count=len(structured),
                            bits=device.to_device(structured))
        t2, _ = _sweep_host(cfg, source=device.SOURCE_SPLITMIX, start=4 * 2048,
                            count=rec["n_random"], seed=rec["seed"])
        np.testing.assert_array_equal(t1 + t2, tally_from_per_class(rec["per_class"]))
    for rec in sweeps_fixture["f32_random"]:
        cfg = _cfg(rec["mode"], rec["eb"], 32)
        t, _ = _sweep_host(cfg, source=device.SOURCE_SPLITMIX, start=0, count=rec["n"],
                           seed=rec["seed"])
        np.testing.assert_array_equal(t, tally_from_per_class(rec["per_class"]))


def test_unsafe_sweep_finds_violation(cuda, oracle):
    from paper_2407_15037_b200 import device

    cfg = _cfg("abs", 1e-3, 32, unsafe=True)
    tally, first = _sweep_host(cfg, source=device.SOURCE_RANGE, start=0x3F800000, count=1 << 22)
    et, ef = oracle.sweep_f32_range("abs", 1e-3, 0x3F800000, 1 << 22, unsafe=True, workers=8)
    np.testing.assert_array_equal(tally, et)
    assert tally[:, 2].sum() > 0
    assert (0x3F800000 + first) & 0xFFFFFFFF == ef


def test_generators(cuda):
    from paper_2407_15037_b200 import device, workloads

    a = device.splitmix64(100003, 0x9E3779B97F4A7C15, 7).cpu().numpy().view(np.uint64)
    np.testing.assert_array_equal(a, workloads.splitmix64(100003, 0x9E3779B97F4A7C15, 7))
    b = device.mixed_f32(1 << 20, workloads.C2_SEED).cpu().numpy().view(np.uint32)
    np.testing.assert_array_equal(b, workloads.c2_values(1 << 20).view(np.uint32))


@pytest.mark.parametrize("eb", [1e-2, 1e-3])
def test_library_log_variant(cuda, eb):
    """quantize_rel32_lib / reconstruct_rel32_lib (_kernels.py:356-431) against the
    reference's own outputs (tests/golden/lib_variant.npz).  The variant uses the
    platform binary64 log2/exp2 and is non-conforming by design, so: the bound
    holds for every value, and codes / reconstructions agree with the CPU
    reference except for rare last-ulp libm differences."""
    import os

    import paper_2407_15037_b200 as g
    from paper_2407_15037_b200 import _kernels as K
    from paper_2407_15037_b200.quantizers import QuantConfig

    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "lib_variant.npz"))
    bits = z["x"]
    x = bits.view(np.float32)
    tag = f"{eb:g}"
    d = QuantConfig(mode="rel", eb=eb, width=32).derived
    codes = np.empty(len(bits), np.uint32)
    ll = np.empty(len(bits), np.bool_)
    trig = K.quantize_rel32_lib(bits, x, codes, ll, d.op_eps, d.w, d.thr, False)
    rec = np.empty(len(bits), np.float32)
    K.reconstruct_rel32_lib(codes, ll, rec.view(np.uint32), rec, d.w)
    rep = g.verify(x, rec, "rel", eb)
    assert rep.passed, rep.summary()
    agree = np.mean((codes == z[f"codes_{tag}"]) & (ll == z[f"lossless_{tag}"]))
    assert agree > 0.999, agree
    assert np.mean(rec.view(np.uint32) == z[f"recon_{tag}"]) > 0.999
    assert abs(int(trig.sum()) - int(z[f"trig_{tag}"].sum())) <= len(bits) // 1000
