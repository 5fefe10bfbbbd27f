"""CPU oracle for the prompt-routing hot path of arxiv 2502.06798 (test infrastructure).

THIS PACKAGE IS TEST INFRASTRUCTURE, NOT PART OF THE PRODUCT.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
legs may import it.  It shares no code with ``paper_2502_06798_b200`` (the CUDA path)
and imports nothing from it; the two meet only through the seeded input generator
in ``synth/``, which holds none of the method's arithmetic.

It is a plain, slow, obviously-correct restatement of what the paper's Query
Dispatcher and K-to-K' Route Planner compute for one batch of prompts
(PAPER.md P:88-P:104, Eq. 1 at P:96), in float64 unless a step fixes another
precision, following the readings R1..R27 listed in DESIGN.md.

Modules
-------
philox  -- Philox4x32-10 counter-based generator (Random123), scalar and vectorised.
route   -- O1..O10: similarity, top-k, optimal-K, H_K, apportionment, Eq. 1 plan,
           D_Q, redirection, route-and-batch, buckets, and the composite ``route``.
forecast-- NEXT f1: the forecast-driven streaming mode (ring-buffer H_K predictor,
           fixed-point Eq. 1 plan, i.i.d. K' sampling, L2 forecast error; R21-R24).
cache   -- NEXT f2: LRU maintenance of the store (vanilla-completion inserts, eviction with
           slot reuse; R25-R27).

Parity status of every function is stated in its docstring; functions whose
result is pinned only by internal invariants (no paper-printed value exists)
say "parity unpinned vs the paper" -- see DESIGN.md section "Oracle pins".
"""
