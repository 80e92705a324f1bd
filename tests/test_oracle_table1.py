"""Pins of the oracle against the paper's Table 1 and worked examples.

The golden grid is derived by hand (tests/golden/table1.txt); an independent
painter's-algorithm evaluation below re-derives it without the oracle's scan.
"""
import numpy as np
import pytest

import tang_inputs as ti
from oracle import pipeline, rules as orules, tss as otss

NM = orules.NO_MATCH


def _rules(table1, extra=()):
    rows = []
    for name, prio, x, y, lx, ly in list(table1["rules"]) + list(extra):
        sx, _ = ti.bits3(x)
        sy, _ = ti.bits3(y)
        rows.append(dict(id=int(name[1:]), priority=prio, sip=sx, sip_len=lx, dip=sy, dip_len=ly))
    return ti.make_rules(rows)


def _grid_ids(table1):
    out = np.full(64, NM, dtype=np.uint32)
    for x in range(8):
        for y, cell in enumerate(table1["grid"][x]):
            out[x * 8 + y] = NM if cell == "-" else int(cell[1:])
    return out


def test_rules_fixture_matches_inputs_module(table1):
    a = _rules(table1)
    b = ti.table1_rules()
    assert (a == b).all()


def test_brute_force_equals_hand_grid(table1):
    R = _rules(table1)
    U = ti.table1_universe()
    want = _grid_ids(table1)
    got_loop = np.array([orules.brute_force_one(R, h) for h in U], dtype=np.uint32)
    got_vec = orules.brute_force(R, U)
    assert (got_loop == want).all()
    assert (got_vec == want).all()
    assert int((want != NM).sum()) == table1["counts"]["matched"] == 41


def test_painter_algorithm_independent_of_scan(table1):
    """Paint every rule's box from lowest to highest precedence: the last paint wins."""
    grid = np.full((8, 8), NM, dtype=np.int64)
    for name, prio, x, y, lx, ly in sorted(table1["rules"], key=lambda r: -r[1]):
        xs = [v for v in range(8) if format(v, "03b")[:lx] == x[:lx]]
        ys = [v for v in range(8) if format(v, "03b")[:ly] == y[:ly]]
        for a in xs:
            for b in ys:
                grid[a, b] = int(name[1:])
    assert (grid.ravel().astype(np.uint32) == _grid_ids(table1)).all()


def test_section_4_2_example():
    """the point in R1 ∩ R6 ∩ R8 goes to R1."""
    R = ti.table1_rules()
    h = ti.make_headers(0b000 << 29, 0b011 << 29)[0]
    assert all(orules.matches(R[i], h) for i in (0, 5, 7))
    assert orules.brute_force_one(R, h) == 1


def test_tuples_and_membership(table1):
    R = _rules(table1)
    sigs = otss.signatures_first_occurrence(R)
    assert sigs == [(lx, ly) for _, lx, ly, _ in table1["tuples"]]
    T = otss.Tss(sigs, R)
    for j, (_, _, _, members) in enumerate(table1["tuples"]):
        got = sorted(r["id"] for r in T.rules() if T.tuple_of(r["id"]) == j)
        assert got == sorted(int(m[1:]) for m in members)
    assert T.mismatch_count == 0


def test_truncation_example(table1):
    """11* under prefix length 2 of a 3-bit field -> 110."""
    for pat, l, want in table1["trunc"]:
        v, _ = ti.bits3(pat)
        T = otss.Tss([(l, 0)])
        _, ms, _ = T.key_of(0, v, 0)
        assert ms == int(want, 2) << 29
        # and a packet 111 truncates to the same key as the rule 11*
        _, mp, _ = T.key_of(0, 0b111 << 29, 0)
        assert mp == ms


def test_insert_examples(table1):
    """R9 -> T1 (exact signature); R10 -> T3 (restricted insert)."""
    R = _rules(table1)
    T = otss.Tss(otss.signatures_first_occurrence(R), R)
    names = [t[0] for t in table1["tuples"]]
    for name, prio, x, y, want in table1["inserts"]:
        sx, lx = ti.bits3(x)
        sy, ly = ti.bits3(y)
        r = ti.make_rules([dict(id=int(name[1:]), priority=prio, sip=sx, sip_len=lx, dip=sy, dip_len=ly)])[0]
        j = T.insert(r)
        assert names[j] == want
    # R9 is exact, R10 is not: one mismatching rule
    assert T.mismatch_count == 1
    # candidates for (3,1) are exactly T3 and T5 (T4=(0,3) fails l^T <= l^R)
    cands = [j for j, (a, b) in enumerate(T.sigs) if a <= 3 and b <= 1]
    assert [names[j] for j in cands] == ["T3", "T5"]


def test_restricted_insert_matches_by_full_rule():
    """R10 = {100, 0**} lives in T3 keyed by X=100 only; the match still checks Y (reading 16)."""
    R = ti.table1_rules()
    T = otss.Tss(otss.signatures_first_occurrence(R), R)
    r10 = ti.make_rules([dict(id=10, priority=10, sip=0b100 << 29, sip_len=3, dip=0, dip_len=1)])[0]
    T.insert(r10)
    inside = ti.make_headers(0b100 << 29, 0b001 << 29)[0]
    outside = ti.make_headers(0b100 << 29, 0b101 << 29)[0]
    assert T.lookup_in_tuple(2, inside)[0] == (10, 10)
    assert T.lookup_in_tuple(2, outside)[0] is None


def test_spec_lookup_examples():
    """SPEC.md:160-162 (derived from Table 1): in-tuple lookups and access counts."""
    R = ti.table1_rules()
    T = otss.Tss(otss.signatures_first_occurrence(R), R)
    p = ti.make_headers(0b000 << 29, 0b011 << 29)[0]
    assert T.lookup_in_tuple(0, p) == ((1, 1), 2)
    assert T.lookup_in_tuple(2, p) == (None, 1)
    q = ti.make_headers(0b110 << 29, 0b011 << 29)[0]
    assert T.lookup_in_tuple(3, q)[0] == (6, 6)
    assert orules.brute_force_one(R, q) == 4          # R4 beats R6


def test_exhaustive_forced_predictions(table1):
    """All 64 points x 5 forced tuples: paper mode equals brute force on the coverage
    set G (no match in the prediction, or the prediction hosts the winner); the
    remaining pairs are exactly the scenario-1 pairs; strict mode is always brute force."""
    R = ti.table1_rules()
    U = ti.table1_universe()
    T = otss.Tss(otss.signatures_first_occurrence(R), R)
    truth = _grid_ids(table1)
    scen1 = 0
    for j in range(5):
        pred = np.full((64, 1), j)
        rid, fell, _ = pipeline.classify_with_pred(T, U, pred, "paper")
        srid, _, _ = pipeline.classify_with_pred(T, U, pred, "strict")
        assert (srid == truth).all()
        for i in range(64):
            in_tuple = T.lookup_in_tuple(j, U[i])[0]
            hosts = truth[i] != NM and T.tuple_of(truth[i]) == j
            if in_tuple is None:
                assert fell[i] and rid[i] == truth[i]
            elif hosts:
                assert not fell[i] and rid[i] == truth[i]
            else:
                scen1 += 1
                assert rid[i] != truth[i] and rid[i] == in_tuple[1]
    assert scen1 == table1["counts"]["scenario1"] == 13


def test_delete_keeps_tuple_and_reroutes():
    """deleting R3 empties T2 but keeps 5 tuples; deleting R1 makes
    (000,011) fall through T1 to R6."""
    R = ti.table1_rules()
    T = otss.Tss(otss.signatures_first_occurrence(R), R)
    assert T.delete(3) and len(T.sigs) == 5 and T.tuple_best(1) is None
    assert not T.delete(99)
    assert T.delete(1)
    p = ti.make_headers(0b000 << 29, 0b011 << 29)
    rid, fell, _ = pipeline.classify_with_pred(T, p, np.array([[0]]))
    assert fell[0] and rid[0] == 6


def test_pruning_is_sound_on_universe():
    R = ti.table1_rules()
    T = otss.Tss(otss.signatures_first_occurrence(R), R)
    for h in ti.table1_universe():
        a, _ = T.ordered_search(h, prune=True)
        b, _ = T.ordered_search(h, prune=False)
        assert a == b


def test_no_tuple_for_insert():
    T = otss.Tss([(8, 8)])
    with pytest.raises(otss.NoTuple):
        T.choose_tuple(4, 32)


@pytest.mark.parametrize("j,won,cls_ok", [
    (0, 2, 64),    # T1 = {R1, R2}: wins (000,011), (000,101); holds no lower-priority match anywhere
    (1, 4, 64),    # T2 = {R3}: wins 00*,11* (4 points); R3 is only ever beaten where it does not match
    (2, 16, 64),   # T3 = {R4, R5}: rows 110, 111
    (3, 11, 59),   # T4 = {R6, R7}: wins column 010 rows 0-5 (6) + column 011 rows 1-5 (5); R6/R7 returned
                   # at (000,011), (110,010), (110,011), (111,010), (111,011) (scenario 1)
    (4, 8, 56),    # T5 = {R8}: 8 points of 0**,0** won elsewhere -> R8 returned (scenario 1);
                   # 5 + 8 = the golden file's 13 scenario-1 pairs
])
def test_statistics_on_table1_with_a_fixed_prediction(table1, j, won, cls_ok):
    """O12 (Tables 2/3): predicting tuple j for every point of the 64-point universe.
    Model accuracy = matched points whose brute-force winner lives in tuple j / 41 (counted by hand
    from the grid); classification accuracy = points whose paper-mode result equals the brute force
    / 64 (scenario-1 points keep the in-tuple match)."""
    R = _rules(table1)
    U = ti.table1_universe()
    sigs = otss.signatures_first_occurrence(R)
    tss = otss.Tss(sigs, R)
    pred = np.full((U.size, 1), j)
    rid, fell, acc = pipeline.classify_with_pred(tss, U, pred, "paper")
    truth = orules.brute_force(R, U)
    st = pipeline.statistics(tss, pred, rid, truth, acc)
    assert st["tuples"] == 5
    assert st["model_accuracy"] == won / 41
    assert st["classification_accuracy"] == cls_ok / 64
    assert st["mean_accesses"] == float(np.mean(acc))
