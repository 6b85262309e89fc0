"""Oracle for Blink (arXiv:1910.04940): plain, slow, obviously-correct CPU code.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import anything
under ``oracle/``.  The product (``paper_1910_04940_b200``) never imports it,
and this package never imports the product: the two share no code.  The only
shared module is ``synth`` (seeded input generators, no method arithmetic).

Citations: ``P:<line>`` is ``/root/reference/PAPER.md`` line <line>; the
section/equation is named beside it.  Readings of ambiguous passages are listed
in DESIGN.md ("Readings of the paper") and referenced here as ``R#<n>``.

Modules
-------
graphs       link-graph model (Sec. 3.1) and the DGX-1 presets (P:56-61,
             reconstructed; R#17), induced sub-allocations.
bounds       Edmonds/Lovasz broadcast bound, Nash-Williams
             undirected bound, brute-force packing LP by tree enumeration
             (Eqs. 1-3).
packing      MWU approximate packing (Sec. 3.2), ILP tree-count
             minimisation with relaxation (Sec. 3.2.1, Eqs. 4-7),
             bidirectional AllReduce trees (Sec. 3.3), one-hop trees
             on a switch (Sec. 3.5), weight-proportional split
             (P:477).
model        chunk-pipelining model (discrete-event simulation vs the
             (c+h-1)/c closed form) and bytes per directed link of a
             plan.
collectives  Broadcast / AllReduce values along packed trees (P:477-487,
             Sec. 4.1): per-tree post-order combine in a fixed operand order,
             fp32 accumulation, one RNE rounding per node (R#12, R#13).

Parity status: every function here is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py`` except where a docstring says "parity unpinned".
"""
