"""CPU oracle of TaNG's classification hot path — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs may import anything under `oracle/`.  The product
path (`paper_2601_03187_b200`, `libtang.so`) never imports, links or executes
it, and the two share no code: the only common module is `tang_inputs`, which
draws seeded inputs and holds none of the method's arithmetic.

The oracle is plain and slow on purpose: Python dictionaries for the tuple
space, NumPy float64 for the MLP, no blocking, fusion or reordering beyond what
the paper states.  Every function cites the PAPER.md line (P:NNN) and section it
follows; SURVEY.md §8(c) lists the readings adopted where the paper is silent or
garbled (also restated in DESIGN.md §2).

Modules
  rules     O1 match, O2 brute-force highest-priority scan          (§2.1, §4.2)
  tss       O3 tuples, O4 placement/insert, O5 delete, O9 in-tuple
            lookup, O10 ordered post-verification search, O11 strict (§4.3, §5.1.1,
                                                                     P:325-335 §5.2.1)
  mlp       O6 features, O7 residual MLP (fp32 / bf16-emulated),
            O8 argmax / top-k                                       (§6.2, Eq.1-2)
  pipeline  two-stage classify (paper and strict mode), statistics  (§5.1.1, Tables 2/3)

Pins (tests/test_oracle_*.py, `-m "not gpu"`): Table 1 exhaustive universe and
its worked examples (tests/golden/table1.txt), the truncation / R9 / R10
examples, brute force on tiny rulesets, correct-fallback and pruning
invariants, the feature example, closed-form MLP special cases and a torch
float64 reference module.  Parity status per function is in DESIGN.md §2; no
function of this oracle is "parity unpinned", but the *paper's trained model*
is (no weights ship with the paper).
"""
