"""NEXT f2: approximate-cache maintenance on the (sharded) store -- LRU eviction with slot reuse.

Test infrastructure only (see oracle/__init__.py).  Plain restatement, no tuning.

Passages followed
-----------------
P:57   the method reuses "prior intermediate states based on input prompt closeness with the cache";
P:102  the Optimal-K Selector "first retrieves the nearest cache" -- the top-1 entry is the one whose
       state is reused;
P:248  dissimilar prompts are redirected "to vanilla diffusion process" -- the generations that
       produce new cache entries.
SPEC S:144-147 (CacheStore: capacity, LRU eviction), S:172-179 (insert: "LRU eviction when over
capacity"; "capacity 2, insert a,b,c -> a evicted"; insert v then nearest(v) = 1.0), S:186 (warm-up:
every completed vanilla generation inserts its embedding; approximate hits do not insert).

Readings (R25-R27)
----------------------------
R25  Population: the embeddings of prompts served by vanilla diffusion (K' = 0) are inserted when
     their generations complete, in prompt order; invalid embeddings are never inserted.
R26  Recency: a logical clock ticks once per routed batch, per insert call and per bulk load.  An
     entry's stamp is the tick of its insertion or of the last batch in which it was a routed
     prompt's top-1 (the entry whose state is reused).  When an insert of n rows finds fewer
     than n free slots, the entries with the smallest (stamp, gid) are evicted -- exactly as many as
     needed; rows inserted by the same call never evict each other (n <= capacity).
R27  Identity: a gid names a slot of the global store (capacity = G x rows per rank; round-robin,
     slot g on rank g mod G).  New rows take the free slots at the end first (ascending), then the
     evicted slots in ascending gid order; a gid is stable from its insert until it is evicted, then
     reused.  Routing results refer to the store as it is when the batch runs.

Pins (tests/test_oracle_cache.py): SPEC S:178-179 examples, a textbook LRU built on
collections.OrderedDict (move_to_end / popitem(last=False)) over random insert / touch sequences,
slot-reuse invariants, the vanilla-insert policy.  "parity unpinned vs the paper's own numbers":
the paper gives no cache policy or sizes.
"""
from __future__ import annotations

import numpy as np


class LruStore:
    """Global view of the store: gid -> row (the caller's original fp32 row) and stamp."""

    def __init__(self, capacity: int, d: int):
        if capacity < 1:
            raise ValueError("capacity must be >= 1")
        self.capacity = capacity
        self.d = d
        self.rows = {}          # gid -> fp32 row
        self.stamp = {}         # gid -> last-use tick
        self.used = 0           # slots handed out so far (append frontier)
        self.tick = 0

    # -- R26 clock -------------------------------------------------------------------------
    def load(self, rows: np.ndarray):
        """Bulk append (pas_cache_load): no eviction; the store must have room."""
        n = len(rows)
        if self.used + n > self.capacity:
            raise ValueError("store full")
        self.tick += 1
        gids = list(range(self.used, self.used + n))
        for g, r in zip(gids, rows):
            self.rows[g] = np.asarray(r, dtype=np.float32)
            self.stamp[g] = self.tick
        self.used += n
        return gids

    def victims(self, n: int):
        """The n entries smallest in (stamp, gid) (R26)."""
        order = sorted(self.stamp.items(), key=lambda kv: (kv[1], kv[0]))
        return [g for g, _ in order[:n]]

    def insert(self, rows: np.ndarray):
        """LRU insert (pas_cache_insert): returns the gid given to each row, in row order (R27)."""
        n = len(rows)
        if n > self.capacity:
            raise ValueError("more rows than capacity")
        self.tick += 1
        n_append = min(n, self.capacity - self.used)
        gids = list(range(self.used, self.used + n_append))
        evicted = sorted(self.victims(n - n_append))
        gids += evicted
        for g in evicted:
            del self.rows[g]
            del self.stamp[g]
        for g, r in zip(gids, rows):
            self.rows[g] = np.asarray(r, dtype=np.float32)
            self.stamp[g] = self.tick
        self.used += n_append
        return gids

    def touch(self, top1_gids, usable):
        """One routed batch: the top-1 entry of every usable prompt gets this batch's tick."""
        self.tick += 1
        for g, ok in zip(top1_gids, usable):
            if ok and g >= 0:
                self.stamp[int(g)] = self.tick

    # -- contents ----------------------------------------------------------------------------
    def contents(self):
        """(gids ascending, rows [n, d]) of the live entries."""
        g = np.array(sorted(self.rows), dtype=np.int64)
        if len(g) == 0:
            return g, np.zeros((0, self.d), dtype=np.float32)
        return g, np.stack([self.rows[int(x)] for x in g])


def vanilla_rows(P: np.ndarray, level_prime: np.ndarray, valid: np.ndarray):
    """R25: the prompts served at K' = 0 (level 0) with a valid embedding, in prompt order."""
    take = (np.asarray(level_prime) == 0) & np.asarray(valid, dtype=bool)
    return P[take], np.nonzero(take)[0]
