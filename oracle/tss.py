"""O3-O5, O9-O11: the TSS middleware of TaNG, written out plainly (test infrastructure only).

P:236 (§4.3): rules are grouped into tuples by prefix-length signature, here over
SIP and DIP ("tuples built from SIP and DIP fields"); each rule maps to exactly
one tuple.  P:240-241: inside a tuple, rules are truncated to the tuple's
signature and kept in a hash table indexed by the truncated values
(example: r_f = 11* under prefix length 2 of a 3-bit field truncates to 110).
P:274 (§5.1.1): lookup truncates the packet the same way, hashes, and compares
the bucket's rules one by one, returning the highest-priority match.
P:276: if the predicted tuple holds no match, an ordered search across the
remaining tuples locates the highest-priority rule (post-verification).
P:328-333 (§5.2.1): the tuple set is fixed; delete edits in place; insertion goes
to the exact-signature tuple, else the first tuple with the maximal sum of
lengths among those with l^T <= l^R in every field, truncating the rule's prefixes.

The hash table here is a Python dict keyed by the truncated key itself, which is
the "any hash, exact-key compare" reading (SURVEY.md §8(c) reading 10).
"""
from __future__ import annotations

import bisect

from .rules import matches, prefix_mask

NO_MATCH = 0xFFFFFFFF


class NoTuple(Exception):
    """Insertion with no candidate tuple (restricted insertion fails)."""


def signatures_first_occurrence(rules):
    """O3 for a fresh build: one tuple per distinct (lsip, ldip), in rule-file order
    (class order is carried in the model blob, SURVEY.md §8(c) reading 8)."""
    seen, out = set(), []
    for r in rules:
        s = (int(r["sip_len"]), int(r["dip_len"]))
        if s not in seen:
            seen.add(s)
            out.append(s)
    return out


def _as_dict(r):
    return {k: int(r[k]) for k in ("id", "priority", "sip", "dip", "sp_lo", "sp_hi", "dp_lo",
                                     "dp_hi", "sip_len", "dip_len", "proto", "proto_mask", "action")}


class Tss:
    """Tuple space with a fixed, ordered tuple set (class j = tuple j)."""

    def __init__(self, signatures, rules=()):
        self.sigs = [(int(a), int(b)) for a, b in signatures]
        self.buckets = {}          # (j, msip, mdip) -> list of rule dicts sorted by (priority, id)
        self.where = {}            # rule id -> bucket key
        self.mismatch_count = 0
        self._order = None
        for r in rules:
            self.insert(r, counting=False)

    # -- O4 -------------------------------------------------------------------------
    def choose_tuple(self, sip_len: int, dip_len: int) -> int:
        """Exact signature if present; else among tuples with l^T <= l^R in both fields,
        the first (lowest index) with maximal l_sip^T + l_dip^T (§5.2.1)."""
        for j, s in enumerate(self.sigs):
            if s == (sip_len, dip_len):
                return j
        best, best_sum = None, -1
        for j, (ls, ld) in enumerate(self.sigs):
            if ls <= sip_len and ld <= dip_len and ls + ld > best_sum:
                best, best_sum = j, ls + ld
        if best is None:
            raise NoTuple((sip_len, dip_len))
        return best

    def key_of(self, j: int, sip: int, dip: int):
        """Truncated key of (sip, dip) under tuple j's signature."""
        ls, ld = self.sigs[j]
        return (j, sip & prefix_mask(ls), dip & prefix_mask(ld))

    def insert(self, rule, counting=True) -> int:
        r = rule if isinstance(rule, dict) else _as_dict(rule)
        if r["id"] in self.where:
            raise ValueError(f"duplicate rule id {r['id']}")
        j = self.choose_tuple(r["sip_len"], r["dip_len"])
        if counting and self.sigs[j] != (r["sip_len"], r["dip_len"]):
            self.mismatch_count += 1     # rules in a non-matching tuple (§5.2.2)
        k = self.key_of(j, r["sip"], r["dip"])
        lst = self.buckets.setdefault(k, [])
        bisect.insort(lst, r, key=lambda x: (x["priority"], x["id"]))   # keep (priority, id) order
        self.where[r["id"]] = k
        self._order = None
        return j

    # -- O5 -------------------------------------------------------------------------
    def delete(self, rule_id: int) -> bool:
        """Remove by id; tuples are never removed, even when empty."""
        k = self.where.pop(int(rule_id), None)
        if k is None:
            return False
        self.buckets[k] = [x for x in self.buckets[k] if x["id"] != int(rule_id)]
        self._order = None
        return True

    def tuple_of(self, rule_id: int) -> int:
        return self.where[int(rule_id)][0]

    def tuple_best(self, j: int):
        """Smallest (priority, id) among tuple j's rules, or None if it is empty."""
        best = None
        for k, lst in self.buckets.items():
            if k[0] == j and lst:
                key = (lst[0]["priority"], lst[0]["id"])
                if best is None or key < best:
                    best = key
        return best

    def precedence_order(self):
        """[(best key, j)] for non-empty tuples, ascending; cached until the next update."""
        if self._order is None:
            order = []
            for j in range(len(self.sigs)):
                b = self.tuple_best(j)
                if b is not None:
                    order.append((b, j))
            order.sort()
            self._order = order
        return self._order

    def rules(self):
        for lst in self.buckets.values():
            yield from lst

    # -- O9 -------------------------------------------------------------------------
    def lookup_in_tuple(self, j: int, hdr):
        """Probe tuple j's bucket for the packet's truncated key and return the first
        rule, in (priority, id) order, that matches in full (§5.1.1).
        Returns ((priority, id) or None, accesses) with accesses = 1 probe + rules compared."""
        lst = self.buckets.get(self.key_of(j, int(hdr["sip"]), int(hdr["dip"])))
        acc = 1
        if lst:
            for r in lst:
                acc += 1
                if matches(r, hdr):
                    return (r["priority"], r["id"]), acc
        return None, acc

    # -- O10 / O11 ------------------------------------------------------------------
    def ordered_search(self, hdr, skip=(), bound=None, prune=True):
        """Post-verification (§5.1.1): search the tuples not in `skip` and return
        the smallest (priority, id) match, or None.  Visit order is ascending tuple
        best-priority (PSTSS order); with `prune`, a tuple whose best key is not
        below the current best is skipped.  `bound` seeds the current best (strict
        mode: only tuples that could beat the in-tuple match are searched)."""
        skip = set(int(s) for s in skip)
        bests = [(b, j) for b, j in self.precedence_order() if j not in skip]
        best, acc = bound, 0
        for b, j in bests:
            if prune and best is not None and b >= best:
                break
            m, a = self.lookup_in_tuple(j, hdr)
            acc += a
            if m is not None and (best is None or m < best):
                best = m
        return best, acc
