"""Pins of oracle/cache.py (R25-R27) against things other than itself:
the SPEC insert examples and a textbook LRU built on collections.OrderedDict."""
from collections import OrderedDict

import numpy as np
import pytest

from oracle import cache as OC
from oracle import route as O


def _unit(rng, n, d):
    x = rng.standard_normal((n, d))
    return (x / np.linalg.norm(x, axis=1, keepdims=True)).astype(np.float32)


def test_spec_insert_examples():
    rng = np.random.default_rng(0)
    v = _unit(rng, 1, 16)
    st = OC.LruStore(capacity=8, d=16)
    st.insert(v)
    g, rows = st.contents()
    s = O.similarity_A(v, rows)
    assert s.max() == pytest.approx(1.0, abs=1e-12)                 # insert v then nearest(v) -> 1.0
    a, b, c = _unit(rng, 3, 16)
    st = OC.LruStore(capacity=2, d=16)
    ga = st.insert(a[None])[0]
    st.insert(b[None])
    gc = st.insert(c[None])[0]
    assert gc == ga                                                   # capacity 2, insert a,b,c -> a evicted
    live = [st.rows[g] for g in sorted(st.rows)]
    assert not any(np.array_equal(r, a) for r in live)
    assert any(np.array_equal(r, b) for r in live) and any(np.array_equal(r, c) for r in live)


class TextbookLru:
    """collections.OrderedDict LRU: every access moves a key to the end; evict from the front.
    Accesses of one tick are applied in ascending gid order (so equal ticks tie by gid, R26)."""

    def __init__(self, capacity):
        self.capacity = capacity
        self.od = OrderedDict()
        self.next = 0

    def insert(self, n):
        fresh = list(range(self.next, min(self.next + n, self.capacity)))
        self.next += len(fresh)
        evicted = []
        for _ in range(n - len(fresh)):
            g, _ = self.od.popitem(last=False)
            evicted.append(g)
        gids = fresh + sorted(evicted)
        for g in sorted(gids):
            self.od[g] = True
            self.od.move_to_end(g)
        return gids

    def touch(self, gids):
        for g in sorted(set(int(x) for x in gids if x >= 0)):
            self.od.move_to_end(g)


def test_lru_matches_textbook_ordereddict():
    rng = np.random.default_rng(1)
    for trial in range(40):
        cap = int(rng.integers(1, 40))
        st = OC.LruStore(capacity=cap, d=4)
        ref = TextbookLru(cap)
        for step in range(60):
            if rng.random() < 0.5:
                n = int(rng.integers(1, cap + 1))
                got = st.insert(_unit(rng, n, 4))
                exp = ref.insert(n)
                assert got == exp, (trial, step, got, exp)
            elif st.rows:
                live = np.array(sorted(st.rows))
                top1 = rng.choice(live, size=int(rng.integers(1, 10)))
                top1[rng.random(len(top1)) < 0.2] = -1                  # cold / invalid prompts
                st.touch(top1, np.ones(len(top1), bool))
                ref.touch(top1)
            assert sorted(st.rows) == sorted(ref.od)
            assert all(0 <= g < cap for g in st.rows)


def test_slot_reuse_and_touch_protects():
    rng = np.random.default_rng(2)
    st = OC.LruStore(capacity=5, d=8)
    g0 = st.insert(_unit(rng, 5, 8))
    assert g0 == [0, 1, 2, 3, 4] and st.used == 5
    st.touch([0, 1], [True, True])                 # 0, 1 used by a batch: newer than 2, 3, 4
    g1 = st.insert(_unit(rng, 2, 8))
    assert g1 == [2, 3]                            # the two least recently used slots, reused
    st.touch([4, 2], [True, False])                # an unusable prompt does not touch
    g2 = st.insert(_unit(rng, 3, 8))
    assert g2 == [0, 1, 2]                         # stamps 0,1: 2 (touched) < 2,3: 3 (inserted) < 4: 4
    assert sorted(st.rows) == [0, 1, 2, 3, 4]
    with pytest.raises(ValueError):
        st.insert(_unit(rng, 6, 8))                # more rows than capacity


def test_load_then_insert_appends_before_evicting():
    rng = np.random.default_rng(3)
    st = OC.LruStore(capacity=10, d=8)
    st.load(_unit(rng, 7, 8))
    g = st.insert(_unit(rng, 5, 8))
    assert g == [7, 8, 9, 0, 1]                    # 3 free slots first, then the 2 oldest loaded
    with pytest.raises(ValueError):
        st.load(_unit(rng, 1, 8))                  # bulk load never evicts


def test_vanilla_rows_policy():
    P = np.arange(12, dtype=np.float32).reshape(6, 2)
    lp = np.array([0, 2, 0, 0, 1, 0])
    valid = np.array([True, True, False, True, True, True])
    rows, idx = OC.vanilla_rows(P, lp, valid)
    assert list(idx) == [0, 3, 5] and np.array_equal(rows, P[[0, 3, 5]])
