"""O1/O2: rule matching and the brute-force highest-priority scan (test infrastructure only).

P:77 (§2.1): "a packet P matches a rule R if every field p_i satisfies r_i";
IP fields are prefixes, ports are ranges, protocol is exact-or-wildcard.
P:195 (§4.2) + Table 1: a smaller priority number wins (R1 beats R6, R8).
Ties in priority go to the smaller rule id (SURVEY.md §8(c) reading 13).
"""
from __future__ import annotations

import numpy as np

NO_MATCH = 0xFFFFFFFF


def prefix_mask(length: int) -> int:
    """32-bit mask keeping the top `length` bits; mask(0) = 0, mask(32) = 0xFFFFFFFF."""
    if length <= 0:
        return 0
    return (0xFFFFFFFF << (32 - length)) & 0xFFFFFFFF


def matches(rule, hdr) -> bool:
    """O1: every field condition of `rule` holds for header `hdr` (§2.1).

    SIP/DIP: the top len bits are equal (prefix).  SP/DP: lo <= p <= hi
    (inclusive ranges).  PRO: (p & mask) == value (mask 0 = wildcard).
    """
    ms = prefix_mask(int(rule["sip_len"]))
    md = prefix_mask(int(rule["dip_len"]))
    if (int(hdr["sip"]) & ms) != (int(rule["sip"]) & ms):
        return False
    if (int(hdr["dip"]) & md) != (int(rule["dip"]) & md):
        return False
    if not (int(rule["sp_lo"]) <= int(hdr["sp"]) <= int(rule["sp_hi"])):
        return False
    if not (int(rule["dp_lo"]) <= int(hdr["dp"]) <= int(rule["dp_hi"])):
        return False
    return (int(hdr["proto"]) & int(rule["proto_mask"])) == (int(rule["proto"]) & int(rule["proto_mask"]))


def brute_force_one(rules, hdr):
    """O2 for one packet, plain loop: argmin over matching rules of (priority, id)."""
    best = None
    for r in rules:
        if matches(r, hdr):
            key = (int(r["priority"]), int(r["id"]))
            if best is None or key < best:
                best = key
    return NO_MATCH if best is None else best[1]


def _masks(lengths: np.ndarray) -> np.ndarray:
    l = lengths.astype(np.uint64)
    return np.where(l == 0, np.uint64(0),
                    (np.uint64(0xFFFFFFFF) << (np.uint64(32) - l)) & np.uint64(0xFFFFFFFF))


def brute_force(rules: np.ndarray, headers: np.ndarray, chunk: int = 1 << 22) -> np.ndarray:
    """O2 for a batch: the same definition as brute_force_one, evaluated with NumPy
    broadcasting (packets x rules) in chunks; returns rule ids (NO_MATCH if none)."""
    n = headers.size
    out = np.full(n, NO_MATCH, dtype=np.uint32)
    if rules.size == 0 or n == 0:
        return out
    # order rules by (priority, id) once: the first matching column is the winner
    order = np.lexsort((rules["id"], rules["priority"]))
    R = rules[order]
    ms, md = _masks(R["sip_len"]), _masks(R["dip_len"])
    rs = R["sip"].astype(np.uint64) & ms
    rd = R["dip"].astype(np.uint64) & md
    spl, sph = R["sp_lo"].astype(np.int64), R["sp_hi"].astype(np.int64)
    dpl, dph = R["dp_lo"].astype(np.int64), R["dp_hi"].astype(np.int64)
    pm = R["proto_mask"].astype(np.int64)
    pv = R["proto"].astype(np.int64) & pm
    ids = R["id"].astype(np.uint32)
    step = max(1, chunk // max(1, rules.size))
    for a in range(0, n, step):
        h = headers[a:a + step]
        s = h["sip"].astype(np.uint64)[:, None]
        d = h["dip"].astype(np.uint64)[:, None]
        sp = h["sp"].astype(np.int64)[:, None]
        dp = h["dp"].astype(np.int64)[:, None]
        pr = h["proto"].astype(np.int64)[:, None]
        m = ((s & ms) == rs) & ((d & md) == rd) & (sp >= spl) & (sp <= sph) & \
            (dp >= dpl) & (dp <= dph) & ((pr & pm) == pv)
        anym = m.any(axis=1)
        first = m.argmax(axis=1)
        out[a:a + step] = np.where(anym, ids[first], NO_MATCH)
    return out
