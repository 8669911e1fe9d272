"""CPU oracle for the Atom (arXiv 2403.10504) swapped GPT training step.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2403_10504_b200``) never imports it, and
this package imports nothing from the product; the two share no code.  The
only shared module is ``synth`` (seeded input generators, no method math).

Contents (each function cites the PAPER.md / SPEC.md passage it follows;
``P:n`` = PAPER.md line n, ``S:n`` = SPEC.md line n):

* ``gpt``      -- plain fp64 GPT-3 (minGPT, pre-LN) forward and hand-written
                  backward, loss = mean token cross-entropy.
* ``adamw``    -- AdamW with linear warm-up, torch semantics.
* ``peers``    -- n-peer replica training with periodic parameter averaging
                  (P:410).
* ``planner``  -- the partition cost model, Algorithm 1 written literally
                  (P:334-386), a brute-force enumerator and an exact DP, plan
                  selection and the choice of C.
* ``schedule`` -- the sub-model swap schedule and its
                  integer-time 3-lane simulation.

Pins (tests/test_oracle_*.py): finite differences, torch-CPU fp64 autograd of
an independently written module, closed forms (initial loss ~ ln V, AdamW
step 1, Table II payloads, P:184/P:295/P:479 byte counts), invariants
(causality, T=1 attention), brute force (planner) and SPEC worked examples.
Parity status of every function is listed in DESIGN.md §3.
"""
