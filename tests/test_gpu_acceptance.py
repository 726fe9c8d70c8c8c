"""The reference's acceptance criteria that exercise the hot path, run through
the GPU (SURVEY.md §8(f1/f2); /root/reference/pkg/tests/test_acceptance.py):

* criterion 4 (test_acceptance.py:119-146): the 900 000-value ABS bin-edge
  adversarial corpus -- protected 0 violations, unprotected exactly the
  oracle's count, which the reference's recorded run gives as 34 167
  (test_output.txt:35);
* criterion 9 (test_acceptance.py:307-329) at full scale: 10^5 byte mutations
  of encoded streams, each decoded on the GPU with the same outcome as the
  oracle -- the same typed error at the same byte position, or the same codes.
"""

import re

import numpy as np
import pytest

from helpers import mixed_bits, verify_numpy

pytestmark = pytest.mark.gpu


def bin_edge_corpus(eb2: np.float32, n_k: int = 10 ** 5) -> np.ndarray:
    """test_acceptance.py:122-134: (k + 1/2) * eb2 in binary64, cast, +-4 ulps."""
    rng = np.random.default_rng(2718)
    k = rng.integers(-(10 ** 6), 10 ** 6, n_k)
    base = ((k.astype(np.float64) + 0.5) * np.float64(eb2)).astype(np.float32)
    parts = [base]
    up, down = base.copy(), base.copy()
    for _ in range(4):
        up = np.nextafter(up, np.float32(np.inf))
        down = np.nextafter(down, np.float32(-np.inf))
        parts.append(up.copy())
        parts.append(down.copy())
    return np.concatenate(parts)


def test_criterion_4_bin_edge_corpus(cuda, oracle):
    import paper_2407_15037_b200 as g

    cfg = g.QuantConfig(mode="abs", eb=1e-3)
    corpus = bin_edge_corpus(cfg.derived.eb2)
    assert len(corpus) == 900_000
    prot, _ = g.compress(corpus, cfg)
    unprot, _ = g.compress(corpus, g.QuantConfig(mode="abs", eb=1e-3, unsafe_no_double_check=True))
    rp = g.verify(corpus, g.decompress_to_array(prot), "abs", 1e-3)
    ru = g.verify(corpus, g.decompress_to_array(unprot), "abs", 1e-3)
    assert rp.violations == 0 and rp.special_mismatch_count == 0
    # the oracle's unprotected stream and its violation count
    so, _, _ = oracle.compress(corpus, "abs", 1e-3, unsafe=True, workers=8)
    assert so == unprot
    d = oracle.derive("abs", 1e-3, 32)
    viol, _, _, _ = verify_numpy(corpus, oracle.decompress_to_array(so, workers=8), "abs", d)
    assert ru.violations == viol == 34167


def _ours(g, data):
    try:
        _, ca = g.decode_stream(data)
        return "OK", ca.codes.tobytes() + ca.lossless.tobytes()
    except g.ContainerError as e:
        m = re.search(r"byte (\d+)", str(e))
        return type(e).__name__, (int(m.group(1)) if m else None)


def _ref(oracle, data):
    try:
        _, codes, ll = oracle.decode_stream(data)
        return "OK", codes.tobytes() + ll.tobytes()
    except oracle.DecodeError as e:
        m = re.search(r"byte (\d+)", str(e))
        return e.kind, (int(m.group(1)) if m else None)


@pytest.mark.parametrize("case", ["rel32_bs128", "abs64_bs4096"])
def test_criterion_9_fuzz_1e5(cuda, oracle, case):
    """10^5 mutations in total (7.5 x 10^4 of the reference's own 500-value base,
    2.5 x 10^4 of a 33-block stream), 1-4 byte XORs each anywhere in the
    stream (header, index, region): outcome == oracle's."""
    import paper_2407_15037_b200 as g

    if case == "rel32_bs128":   # the reference's own base: 500 REL values, block_size 128
        x = mixed_bits(32, 500, 98765).view(np.float32)[:500]
        base, _, _ = oracle.compress(x, "rel", 1e-2, block_size=128)
    else:                        # 33 full 4096-value blocks: the fast decode kernels
        x = mixed_bits(64, 33 * 4096 - 5, 4321).view(np.float64)
        base, _, _ = oracle.compress(x, "abs", 1e-3, workers=8)
    rng = np.random.default_rng(98765 if case == "rel32_bs128" else 1234)
    counts = {}
    n_mut = 75_000 if case == "rel32_bs128" else 25_000
    for _ in range(n_mut):
        s = bytearray(base)
        for _ in range(int(rng.integers(1, 5))):
            pos = int(rng.integers(0, len(s)))
            s[pos] ^= int(rng.integers(1, 256))
        s = bytes(s)
        got, exp = _ours(g, s), _ref(oracle, s)
        assert got == exp, (case, got[0], exp[0], got[1] if got[0] != "OK" else "", exp[1] if exp[0] != "OK" else "")
        counts[got[0]] = counts.get(got[0], 0) + 1
    assert sum(counts.values()) == n_mut
    assert len(counts) >= 3, counts
