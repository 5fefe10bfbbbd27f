"""Pins for oracle.philox: published Random123 known-answer vectors (tests/golden/philox_kat.json)
and agreement of the scalar and vectorised implementations."""
import json
import os

import numpy as np
from hypothesis import given, settings, strategies as st

from oracle import philox

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _kat():
    with open(os.path.join(GOLD, "philox_kat.json")) as fh:
        return json.load(fh)["vectors"]


def test_kat_scalar():
    for v in _kat():
        ctr = [int(x, 16) for x in v["ctr"]]
        key = [int(x, 16) for x in v["key"]]
        out = philox.philox4x32_10(ctr, key)
        assert ["%08x" % o for o in out] == v["out"]


def test_kat_vectorised():
    for v in _kat():
        ctr = [np.array([int(x, 16)], dtype=np.uint64) for x in v["ctr"]]
        key = [int(x, 16) for x in v["key"]]
        out = philox.philox4x32_10_np(*ctr, *key)
        assert ["%08x" % int(o[0]) for o in out] == v["out"]


@settings(max_examples=200, deadline=None)
@given(st.lists(st.integers(0, 2**32 - 1), min_size=6, max_size=6))
def test_scalar_equals_vectorised(words):
    c = words[:4]
    k = words[4:]
    a = philox.philox4x32_10(c, k)
    b = philox.philox4x32_10_np(*[np.array([x], dtype=np.uint64) for x in c], *k)
    assert tuple(int(x[0]) for x in b) == a


def test_counter_layout():
    """ctr = (p, 0, batch_lo, stream<<24 | batch_hi), key = (seed_lo, seed_hi)  (R18)."""
    seed, batch = (0xABCDEF12 << 32) | 0x3456789A, (0x12 << 32) | 0x345
    w = philox.stream_words(5, seed, batch, 2)
    for p in range(5):
        ref = philox.philox4x32_10((p, 0, 0x345, (2 << 24) | 0x12), (0x3456789A, 0xABCDEF12))
        assert tuple(int(x[p]) for x in w) == ref


def test_redirect_keys_60_bits_and_w1_values():
    k = philox.redirect_keys(4, 2025, 0)
    assert np.all(k < (np.uint64(1) << np.uint64(60)))
    with open(os.path.join(GOLD, "w1.json")) as fh:
        w1 = json.load(fh)
    for p, hx in enumerate(w1["key64_hex_p0_3"]):
        assert int(k[p]) | (2 << 60) == int(hx, 16)


def test_uniform_words_are_uniform():
    u = philox.uniform_words(200_000, 7, 3).astype(np.float64) / 2**32
    hist, _ = np.histogram(u, bins=16, range=(0, 1))
    exp = len(u) / 16
    chi2 = float(np.sum((hist - exp) ** 2 / exp))
    assert chi2 < 45.0   # 15 dof, p ~ 1e-4
