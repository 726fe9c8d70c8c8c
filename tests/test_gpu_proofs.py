"""Proof-by-enumeration of the production quantizers where they are not the
reference op sequence verbatim (SURVEY.md §8(a5/a6)):

* binary32 REL (exact-division stream encoder + division-free filter): every
  one of the 2^32 patterns, for a grid of 40+ bounds (log-spaced 1e-7 .. 0.5
  plus every REL constant of the reference fixture), safe and unsafe;
* the FCHK-free division itself for ARBITRARY bounds w in [2^-100, 2^100]
  (10^11 sampled (l, w) pairs and double-check quotients vs div.rn);
* binary64 ABS / REL production quantizers vs the reference op sequences over
  >= 10^11 sampled patterns concentrated on decision edges;
* the Appendix-B binary64 sweep (sweep.py:251-275, test_output.txt:29-31):
  1 000 024 576 patterns, exact tallies, 0 violations.
"""

import ctypes

import numpy as np
import pytest

from helpers import tally_from_per_class

pytestmark = pytest.mark.gpu

REL_GRID = sorted(set([float(x) for x in np.geomspace(1e-7, 0.5, 36)] +
                      [1e-1, 1e-2, 1e-3, 1e-4, 1e-5, 1e-6, 0.3, 0.05]))


def _stream():
    import torch

    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _rel_filter_bad(eb, unsafe):
    import torch

    from paper_2407_15037_b200 import _lib
    from paper_2407_15037_b200.quantizers import QuantConfig

    d = QuantConfig(mode="rel", eb=eb, width=32, unsafe_no_double_check=unsafe).derived
    out = torch.zeros(2, dtype=torch.int64, device="cuda")
    _lib.call("gebq_selfcheck_rel_filter_f32", 0, 1 << 32, ctypes.c_float(d.op_eps),
              ctypes.c_float(d.w), ctypes.c_float(d.thr), int(unsafe),
              ctypes.c_void_p(out.data_ptr()), _stream())
    return out


@pytest.mark.parametrize("unsafe", [False, True])
def test_rel_f32_exhaustive_bound_grid(cuda, fixtures, unsafe):
    """All 2^32 patterns x every bound of the grid and of the reference's
    fixtures: (code, trigger) of both production binary32 REL quantizers equal
    the reference sequence (quantize_rel32, _kernels.py:165-224)."""
    from paper_2407_15037_b200.quantizers import QuantConfig

    ebs = list(REL_GRID)
    for rec in fixtures.get("constants", []):
        if rec.get("mode") == "rel" and rec.get("width") == 32:
            ebs.append(float(rec["eb"]))
    # bounds whose w lies outside [2^-100, 2^100] never reach the exact-division
    # encoder (the launcher routes them to the generic kernel)
    ebs = sorted(eb for eb in set(ebs)
                 if 2.0 ** -100 <= float(QuantConfig(mode="rel", eb=eb, width=32).derived.w) <= 2.0 ** 100)
    assert len(ebs) >= 40
    outs = [(eb, _rel_filter_bad(eb, unsafe)) for eb in ebs]
    bad = {eb: int(o[0].item()) for eb, o in outs if int(o[0].item())}
    assert not bad, bad


def test_div32_any_bound_sampled(cuda):
    """div_refined == __fdiv_rn on 2 x 5e10 sampled operand pairs: the t = l / w
    division for random w in [2^-100, 2^100] and the double-check quotient."""
    import torch

    from paper_2407_15037_b200 import _lib

    out = torch.zeros(2, dtype=torch.int64, device="cuda")
    per = 1 << 33
    n = 0
    for s in range(6):
        _lib.call("gebq_selfcheck_div_f32", 0xD1F0 + s, per, ctypes.c_void_p(out.data_ptr()), _stream())
        n += per
    bad, seen = out.cpu().tolist()
    assert bad == 0
    assert seen >= int(0.9e11)


F64_CASES = [("abs", 1e-3, None), ("abs", 1e-1, None), ("abs", 1e-6, None), ("abs", 1e-12, None),
             ("noa", 1e-4, 14.0), ("rel", 1e-3, None), ("rel", 1e-1, None), ("rel", 1e-6, None),
             ("rel", 1e-12, None), ("rel", 0.5, None)]


@pytest.mark.parametrize("unsafe", [False, True])
def test_f64_quantizers_sampled(cuda, unsafe):
    """binary64 production quantizers == reference op sequences (quantize_abs64 /
    quantize_rel64, _kernels.py:126-285): >= 10^11 patterns per safety mode over
    ten configurations, most of them on bin and double-check edges."""
    import torch

    from paper_2407_15037_b200 import _lib
    from paper_2407_15037_b200.quantizers import QuantConfig

    per = 10_000_000_000 // 1   # 10^10 per configuration
    total = 0
    bad = {}
    for i, (mode, eb, vr) in enumerate(F64_CASES):
        d = QuantConfig(mode=mode, eb=eb, width=64, value_range=vr, unsafe_no_double_check=unsafe).derived
        out = torch.zeros(2, dtype=torch.int64, device="cuda")
        F = ctypes.c_double
        seed = 0xF64C0000 + 16 * i + int(unsafe)
        if mode == "rel":
            _lib.call("gebq_selfcheck_rel_f64", seed, per, F(d.op_eps), F(d.w), F(d.thr), int(unsafe),
                      ctypes.c_void_p(out.data_ptr()), _stream())
        else:
            _lib.call("gebq_selfcheck_abs_f64", seed, per, F(d.eb_eff), F(d.eb2), F(d.inv_eb2), F(d.thr),
                      int(unsafe), ctypes.c_void_p(out.data_ptr()), _stream())
        b, seen = out.cpu().tolist()
        assert seen == per
        total += seen
        if b:
            bad[(mode, eb)] = b
    assert not bad, bad
    assert total >= 10 ** 11


# Appendix B (test_output.txt:29-31): sweep_f64(mode, [1e-3], n_random=10**9, seed=0x5D0)
F64_APPENDIX_B = {
    "abs": {"zero": (2, 0), "denormal": (489082, 0), "normal": (524163067, 474884102),
            "infinity": (0, 2), "nan": (0, 488321)},
    "rel": {"zero": (0, 2), "denormal": (0, 489082), "normal": (931240611, 67806558),
            "infinity": (0, 2), "nan": (0, 488321)},
}


@pytest.mark.parametrize("mode", ["abs", "rel"])
def test_sweep_f64_appendix_b(cuda, mode):
    import paper_2407_15037_b200 as g

    (rep,) = g.sweep_f64(mode, [1e-3], n_random=10 ** 9, seed=0x5D0)
    t = tally_from_per_class(rep.per_class)
    assert int(t.sum()) == 1_000_024_576
    assert rep.violations == 0 and int(t[:, 2].sum()) == 0
    for ci, cls in enumerate(("zero", "denormal", "normal", "infinity", "nan")):
        assert (int(t[ci, 0]), int(t[ci, 1])) == F64_APPENDIX_B[mode][cls], (mode, cls)


@pytest.mark.parametrize("mode,eb,vr,unsafe", [
    ("abs", 1e-3, None, False), ("abs", 1e-3, None, True), ("abs", 1e-1, None, False),
    ("abs", 1e-7, None, False), ("noa", 1e-4, 1.0, False), ("rel", 1e-2, None, False),
])
def test_stream_encoder_exhaustive_f32(cuda, mode, eb, vr, unsafe):
    """Every f32 pattern through the fused stream encoder (k_encode4k_sp, whose
    full-tile rows have their own fast quantize / length paths): the stream
    decodes (k_decode4k_sp, codes sink) to exactly the codes and lossless flags
    of the stand-alone quantizer k_quantize (itself proven against the
    reference op sequence over all 2^32 patterns above), with equal trigger
    counts.  Patterns enter in 16 chunks of 2^28, shuffled within each chunk by
    a fixed bijection so every tile mixes magnitudes and signs."""
    import torch

    from paper_2407_15037_b200 import device as gdev, stream
    from paper_2407_15037_b200.quantizers import QuantConfig

    cfg = QuantConfig(mode=mode, eb=eb, width=32, value_range=vr, unsafe_no_double_check=unsafe)
    n = 1 << 28
    idx = torch.arange(n, dtype=torch.int64, device="cuda")
    # odd multiplier mod 2^28: a bijection of the chunk; keep tiles of runs too
    perm = (idx * 0x9E3779B1) & (n - 1)
    hdr = stream.header_for(cfg, n)
    nblocks = -(-n // cfg.block_size)
    for c in range(16):
        bits = ((perm if c % 2 else idx) + (c << 28)).to(torch.int32)
        enc = stream.encode(bits, cfg)
        rl = int(enc.region_len.item())
        buf = enc.buf[:enc.region_off + rl]
        codes, ll, err = stream.decode_codes(buf, hdr, nblocks)
        q, qll, qtrig = gdev.quantize(bits, cfg)
        assert int(err.item()) == -1, c
        assert torch.equal(codes, q), c
        assert torch.equal(ll, qll), c
        assert enc.trig.cpu().tolist() == qtrig.cpu().tolist(), c
        del enc, buf, codes, ll, q, qll
