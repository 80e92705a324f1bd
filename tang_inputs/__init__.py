"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of TaNG's arithmetic: no matching, no tuple grouping, no
hashing, no MLP evaluation.  It only draws rulesets, packet traces and model
weights from seeded generators and defines the plain record layouts both sides
consume (the 16-byte header and 32-byte rule structs of include/tang.h).

Workload recipe (DESIGN.md §3 restates it):

* Rulesets are ClassBench-shaped (the paper uses ClassBench-ng acl/fw/ipc sets,
  PAPER.md:410 §7.1).  Each rule draws its (SIP, DIP) prefix-length pair from a
  family-specific categorical over the 33x33 grid whose support size is tuned so
  the number of distinct pairs ("tuples") lands in the paper's per-family range
  (Table 3: ACL 139-391, FW 71-144, IPC 31-362 at 512k).
  Addresses come from a shared pool so prefixes nest and overlap; ports use the
  ClassBench classes WC / HI / LO / EM / AR; protocol is tcp/udp/icmp/wildcard.
  Priority = line order, rule id = line index.
* Traces "randomly match the rules" (§7.1): pick a rule (uniform,
  or Zipf(s) over a seeded permutation of ranks) and draw a point uniformly
  inside its hyper-rectangle.
* Weights: He-uniform fp32, stored [in][out] as in the paper's x.w (Eq. 1,
  PAPER.md:377).
"""
from __future__ import annotations

import numpy as np

# struct tang_header (include/tang.h): 16 bytes
HEADER_DTYPE = np.dtype([("sip", "<u4"), ("dip", "<u4"), ("sp", "<u2"), ("dp", "<u2"),
                         ("proto", "u1"), ("pad", "u1", (3,))])
assert HEADER_DTYPE.itemsize == 16

# struct tang_rule (include/tang.h): 32 bytes
RULE_DTYPE = np.dtype([("id", "<u4"), ("priority", "<u4"), ("sip", "<u4"), ("dip", "<u4"),
                       ("sp_lo", "<u2"), ("sp_hi", "<u2"), ("dp_lo", "<u2"), ("dp_hi", "<u2"),
                       ("sip_len", "u1"), ("dip_len", "u1"), ("proto", "u1"), ("proto_mask", "u1"),
                       ("action", "<u4")])
assert RULE_DTYPE.itemsize == 32

NO_MATCH = 0xFFFFFFFF
FAMILIES = ("acl", "fw", "ipc")


def _canon(addr: np.ndarray, length: np.ndarray) -> np.ndarray:
    """Zero the host bits of a prefix (rules are canonical)."""
    length = length.astype(np.uint64)
    keep = np.where(length == 0, np.uint64(0),
                    (np.uint64(0xFFFFFFFF) << (np.uint64(32) - length)) & np.uint64(0xFFFFFFFF))
    return (addr.astype(np.uint64) & keep).astype(np.uint32)


def make_rules(rows) -> np.ndarray:
    """Build a rule array from dicts (missing fields default to wildcards)."""
    out = np.zeros(len(rows), dtype=RULE_DTYPE)
    for i, r in enumerate(rows):
        out[i]["id"] = r.get("id", i)
        out[i]["priority"] = r.get("priority", i)
        out[i]["sip_len"] = r.get("sip_len", 0)
        out[i]["dip_len"] = r.get("dip_len", 0)
        out[i]["sip"] = r.get("sip", 0)
        out[i]["dip"] = r.get("dip", 0)
        out[i]["sp_lo"] = r.get("sp_lo", 0)
        out[i]["sp_hi"] = r.get("sp_hi", 0xFFFF)
        out[i]["dp_lo"] = r.get("dp_lo", 0)
        out[i]["dp_hi"] = r.get("dp_hi", 0xFFFF)
        out[i]["proto"] = r.get("proto", 0)
        out[i]["proto_mask"] = r.get("proto_mask", 0)
        out[i]["action"] = r.get("action", i)
    out["sip"] = _canon(out["sip"], out["sip_len"])
    out["dip"] = _canon(out["dip"], out["dip_len"])
    return out


def make_headers(sip, dip, sp=0, dp=0, proto=0) -> np.ndarray:
    sip = np.atleast_1d(np.asarray(sip, dtype=np.uint64))
    n = sip.shape[0]
    h = np.zeros(n, dtype=HEADER_DTYPE)
    h["sip"] = sip.astype(np.uint32)
    h["dip"] = np.broadcast_to(np.asarray(dip, dtype=np.uint64), (n,)).astype(np.uint32)
    h["sp"] = np.broadcast_to(np.asarray(sp), (n,)).astype(np.uint16)
    h["dp"] = np.broadcast_to(np.asarray(dp), (n,)).astype(np.uint16)
    h["proto"] = np.broadcast_to(np.asarray(proto), (n,)).astype(np.uint8)
    return h


# ---------------------------------------------------------------------------------
# Table 1 of the paper: 8 rules over two 3-bit fields X, Y.
# Embedded in the 5-tuple as the top 3 bits of SIP (X) and DIP (Y); ports and
# protocol are wildcards.  A 3-bit prefix of length l is a 32-bit prefix of length l.
# ---------------------------------------------------------------------------------
TABLE1 = [  # (name, priority, X, Y) with '*' wildcard bits
    ("R1", 1, "000", "011"), ("R2", 2, "000", "101"), ("R3", 3, "00*", "11*"),
    ("R4", 4, "110", "***"), ("R5", 5, "111", "***"), ("R6", 6, "***", "011"),
    ("R7", 7, "***", "010"), ("R8", 8, "0**", "0**"),
]


def bits3(pattern: str):
    """'01*' -> (value << 29, prefix length)."""
    l = len(pattern.rstrip("*"))
    v = int(pattern.replace("*", "0"), 2)
    return v << 29, l


def table1_rules(extra=()) -> np.ndarray:
    rows = []
    for k, (name, prio, x, y) in enumerate(list(TABLE1) + list(extra)):
        sx, lx = bits3(x)
        sy, ly = bits3(y)
        rows.append(dict(id=int(name[1:]), priority=prio, sip=sx, sip_len=lx, dip=sy, dip_len=ly))
    return make_rules(rows)


def table1_universe() -> np.ndarray:
    """All 64 points (x, y) of the 3-bit x 3-bit space, x-major."""
    xs, ys = np.meshgrid(np.arange(8, dtype=np.uint64), np.arange(8, dtype=np.uint64), indexing="ij")
    return make_headers(xs.ravel() << np.uint64(29), ys.ravel() << np.uint64(29))


# ---------------------------------------------------------------------------------
# ClassBench-shaped synthetic rulesets
# ---------------------------------------------------------------------------------
# Per family: number of distinct (lsip, ldip) pairs in the support, marginal
# length weights, Zipf exponent of the pair weights, port-class weights and
# protocol weights.  Port classes: WC 0:65535, HI 1024:65535, LO 0:1023, EM x:x, AR a:b.
_FAMILY = {
    "acl": dict(support=300, zipf=0.9,
                sip_len={0: 3, 8: 1, 16: 2, 24: 3, 28: 2, 32: 6},
                dip_len={0: 1, 16: 2, 24: 4, 28: 3, 32: 8},
                sp=(0.85, 0.05, 0.02, 0.05, 0.03), dp=(0.10, 0.08, 0.04, 0.60, 0.18),
                proto=(0.6, 0.25, 0.05, 0.10)),
    "fw": dict(support=110, zipf=0.8,
               sip_len={0: 6, 8: 1, 16: 2, 24: 3, 32: 3},
               dip_len={0: 3, 8: 1, 16: 2, 24: 3, 32: 5},
               sp=(0.45, 0.15, 0.05, 0.15, 0.20), dp=(0.20, 0.15, 0.05, 0.40, 0.20),
               proto=(0.45, 0.25, 0.05, 0.25)),
    "ipc": dict(support=200, zipf=1.0,
                sip_len={0: 2, 8: 1, 16: 2, 24: 4, 28: 2, 32: 5},
                dip_len={0: 2, 8: 1, 16: 2, 24: 4, 28: 2, 32: 5},
                sp=(0.65, 0.10, 0.05, 0.10, 0.10), dp=(0.25, 0.10, 0.05, 0.45, 0.15),
                proto=(0.5, 0.3, 0.1, 0.1)),
}


def _length_marginal(anchors: dict, rng) -> np.ndarray:
    """Probability over lengths 0..32: anchor weights plus a thin spread nearby."""
    w = np.full(33, 0.02)
    for l, a in anchors.items():
        w[l] += a
        for d in (1, 2, 3):
            for m in (l - d, l + d):
                if 0 <= m <= 32:
                    w[m] += a * 0.08 / d
    return w / w.sum()


def classbench_ruleset(family: str, n: int, seed: int) -> np.ndarray:
    """A seeded ClassBench-shaped ruleset of n rules (priority = line order)."""
    if family not in _FAMILY:
        raise ValueError(f"unknown family {family!r}")
    p = _FAMILY[family]
    rng = np.random.default_rng(seed)
    ms = _length_marginal(p["sip_len"], rng)
    md = _length_marginal(p["dip_len"], rng)
    joint = np.outer(ms, md)
    # ClassBench seeds rarely pair two short prefixes: such rules overlap almost everything
    tot = np.add.outer(np.arange(33), np.arange(33))
    joint = np.where(tot < 24, joint * 0.03, np.where(tot < 40, joint * 0.3, joint)).ravel()
    joint /= joint.sum()
    support = rng.choice(33 * 33, size=p["support"], replace=False, p=joint)
    w = 1.0 / np.arange(1, support.size + 1) ** p["zipf"]
    w = w / w.sum()
    pick = support[rng.choice(support.size, size=n, p=w)]
    sip_len = (pick // 33).astype(np.uint8)
    dip_len = (pick % 33).astype(np.uint8)

    # hierarchical address pools: a few /8 roots, /16 children, host addresses below,
    # so prefixes of different lengths nest and overlap as in ClassBench seeds
    def pool_addr(m):
        roots = rng.integers(0, 256, size=max(8, int(np.sqrt(n)) // 2 + 8), dtype=np.uint64)
        mids = rng.integers(0, 1 << 16, size=max(64, n // 8 + 64), dtype=np.uint64)
        r = roots[rng.integers(0, roots.size, size=m)]
        mid = mids[rng.integers(0, mids.size, size=m)] & np.uint64(0xFFFF)
        lo = rng.integers(0, 1 << 16, size=m, dtype=np.uint64)
        return (r << np.uint64(24)) | ((mid & np.uint64(0xFF)) << np.uint64(16)) | lo

    rules = np.zeros(n, dtype=RULE_DTYPE)
    rules["id"] = np.arange(n, dtype=np.uint32)
    rules["priority"] = np.arange(n, dtype=np.uint32)
    rules["sip_len"] = sip_len
    rules["dip_len"] = dip_len
    rules["sip"] = _canon(pool_addr(n), sip_len)
    rules["dip"] = _canon(pool_addr(n), dip_len)
    for fld, probs in (("sp", p["sp"]), ("dp", p["dp"])):
        cls = rng.choice(5, size=n, p=probs)
        lo = np.zeros(n, dtype=np.int64)
        hi = np.full(n, 65535, dtype=np.int64)
        m = cls == 1
        lo[m] = 1024
        m = cls == 2
        hi[m] = 1023
        m = cls == 3
        common = np.array([80, 443, 53, 22, 25, 110, 123, 161, 389, 1521, 3306, 8080])
        em = np.where(rng.random(n) < 0.6, common[rng.integers(0, common.size, n)],
                      rng.integers(0, 65536, n))
        lo[m] = em[m]
        hi[m] = em[m]
        m = cls == 4
        a = rng.integers(0, 65536, n)
        b = np.minimum(65535, a + rng.integers(1, 4096, n))
        lo[m] = a[m]
        hi[m] = b[m]
        rules[fld + "_lo"] = lo.astype(np.uint16)
        rules[fld + "_hi"] = hi.astype(np.uint16)
    pc = rng.choice(4, size=n, p=p["proto"])
    rules["proto"] = np.array([6, 17, 1, 0], dtype=np.uint8)[pc]
    rules["proto_mask"] = np.where(pc == 3, 0, 0xFF).astype(np.uint8)
    rules["action"] = rng.integers(0, 1 << 16, size=n, dtype=np.uint32)
    return rules


# ---------------------------------------------------------------------------------
# Traces
# ---------------------------------------------------------------------------------
def _points_inside(rules: np.ndarray, idx: np.ndarray, rng) -> np.ndarray:
    r = rules[idx]
    n = idx.size
    h = np.zeros(n, dtype=HEADER_DTYPE)

    def fill(addr, length):
        host = rng.integers(0, 1 << 32, size=n, dtype=np.uint64)
        length = length.astype(np.uint64)
        hostmask = np.where(length == 0, np.uint64(0xFFFFFFFF),
                            (np.uint64(1) << (np.uint64(32) - length)) - np.uint64(1))
        return (addr.astype(np.uint64) | (host & hostmask)).astype(np.uint32)

    h["sip"] = fill(r["sip"], r["sip_len"])
    h["dip"] = fill(r["dip"], r["dip_len"])
    for f in ("sp", "dp"):
        lo = r[f + "_lo"].astype(np.int64)
        hi = r[f + "_hi"].astype(np.int64)
        h[f] = (lo + (rng.random(n) * (hi - lo + 1)).astype(np.int64)).clip(lo, hi).astype(np.uint16)
    anyp = rng.choice(np.array([6, 17, 1, 47, 50], dtype=np.uint8), size=n)
    h["proto"] = np.where(r["proto_mask"] == 0xFF, r["proto"], anyp)
    return h


def uniform_trace(rules: np.ndarray, n: int, seed: int) -> np.ndarray:
    """Pick a rule uniformly, then a point uniformly inside it."""
    rng = np.random.default_rng(seed)
    if rules.size == 0 or n == 0:
        return np.zeros(n, dtype=HEADER_DTYPE)
    return _points_inside(rules, rng.integers(0, rules.size, size=n), rng)


def zipf_trace(rules: np.ndarray, n: int, seed: int, s: float = 1.0, perm_seed: int | None = None) -> np.ndarray:
    """Pick a rule by Zipf(s) over a seeded permutation of rule ranks, then a point inside.
    perm_seed (default: seed) fixes the popularity ranking separately from the draws, so traces
    of one workload (ranks, training history) can share which rules are hot."""
    rng = np.random.default_rng(seed)
    if rules.size == 0 or n == 0:
        return np.zeros(n, dtype=HEADER_DTYPE)
    perm = rng.permutation(rules.size) if perm_seed is None else \
        np.random.default_rng(perm_seed).permutation(rules.size)
    cdf = np.cumsum(1.0 / np.arange(1, rules.size + 1) ** s)
    cdf /= cdf[-1]
    rank = np.searchsorted(cdf, rng.random(n), side="right").clip(0, rules.size - 1)
    return _points_inside(rules, perm[rank], rng)


def random_headers(n: int, seed: int) -> np.ndarray:
    """Uniformly random headers (most match nothing in sparse rulesets)."""
    rng = np.random.default_rng(seed)
    h = np.zeros(n, dtype=HEADER_DTYPE)
    h["sip"] = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    h["dip"] = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    h["sp"] = rng.integers(0, 1 << 16, n).astype(np.uint16)
    h["dp"] = rng.integers(0, 1 << 16, n).astype(np.uint16)
    h["proto"] = rng.integers(0, 256, n).astype(np.uint8)
    return h


# ---------------------------------------------------------------------------------
# Model weights (random init; the plain trainer overwrites them)
# ---------------------------------------------------------------------------------
def random_weights(S: int, N: int, B: int, C: int, seed: int, gain: float = 1.0) -> dict:
    """He-uniform fp32 weights in [in][out] layout (x.w, Eq. 1).

    Keys: W0 [S,N], b0 [N], W1[i] / W2[i] [N,N], b1[i] / b2[i] [N], Wo [N,C], bo [C].
    Inputs to layer 0 are in [0,1) (16-bit chunks / 65536) so W0 is scaled up.
    """
    rng = np.random.default_rng(seed)

    def lin(fan_in, fan_out, scale=1.0):
        lim = gain * scale * np.sqrt(6.0 / fan_in)
        return (rng.uniform(-lim, lim, size=(fan_in, fan_out)).astype(np.float32),
                rng.uniform(-0.1, 0.1, size=fan_out).astype(np.float32))

    W0, b0 = lin(S, N, 4.0)
    W1, b1, W2, b2 = [], [], [], []
    for _ in range(B):
        w, b = lin(N, N, 0.7)
        W1.append(w), b1.append(b)
        w, b = lin(N, N, 0.35)
        W2.append(w), b2.append(b)
    Wo, bo = lin(N, C)
    return dict(S=S, N=N, B=B, C=C, W0=W0, b0=b0, W1=W1, b1=b1, W2=W2, b2=b2, Wo=Wo, bo=bo)


def rules_to_classbench(rules: np.ndarray) -> str:
    """ClassBench text (one '@' line per rule, priority = line order)."""
    def ip(a):
        a = int(a)
        return f"{a >> 24 & 255}.{a >> 16 & 255}.{a >> 8 & 255}.{a & 255}"
    lines = []
    for r in rules:
        lines.append(f"@{ip(r['sip'])}/{r['sip_len']}\t{ip(r['dip'])}/{r['dip_len']}\t"
                     f"{r['sp_lo']} : {r['sp_hi']}\t{r['dp_lo']} : {r['dp_hi']}\t"
                     f"0x{int(r['proto']):02x}/0x{int(r['proto_mask']):02x}")
    return "\n".join(lines) + ("\n" if lines else "")


# ---------------------------------------------------------------------------------------
# committed models (models/*.npz): data handling only.  W1, W2, Wo must already hold bf16 values
# (the trainer rounds them, train.round_weights_bf16) and are stored as their top 16 bits; W0 and
# the biases stay fp32.  Loaded by bench.py's GPU leg, its oracle leg and the full-size parity test.
# ---------------------------------------------------------------------------------------
def _top16(a) -> np.ndarray:
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    if (u & np.uint32(0xFFFF)).any():
        raise ValueError("W1/W2/Wo must hold bf16 values (round them first)")
    return (u >> np.uint32(16)).astype(np.uint16)


def _from_top16(u) -> np.ndarray:
    return (np.asarray(u, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def save_model(path: str, sigs, w: dict, meta: dict) -> None:
    import json
    np.savez_compressed(
        path, sigs=np.asarray(sigs, dtype=np.int32).reshape(-1, 2),
        dims=np.array([w["S"], w["N"], w["B"], w["C"]], np.int64),
        W0=np.asarray(w["W0"], np.float32), b0=np.asarray(w["b0"], np.float32),
        W1=np.stack([_top16(x) for x in w["W1"]]), b1=np.stack([np.asarray(x, np.float32) for x in w["b1"]]),
        W2=np.stack([_top16(x) for x in w["W2"]]), b2=np.stack([np.asarray(x, np.float32) for x in w["b2"]]),
        Wo=_top16(w["Wo"]), bo=np.asarray(w["bo"], np.float32),
        meta=np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8))


def load_model(path: str):
    """(signatures [(lsip, ldip)], fp32 weight dict, metadata dict) of a model file."""
    import json
    z = np.load(path)
    S, N, B, C = (int(x) for x in z["dims"])
    w = dict(S=S, N=N, B=B, C=C, W0=z["W0"], b0=z["b0"],
             W1=[_from_top16(x) for x in z["W1"]], b1=list(z["b1"]),
             W2=[_from_top16(x) for x in z["W2"]], b2=list(z["b2"]),
             Wo=_from_top16(z["Wo"]), bo=z["bo"])
    return [(int(a), int(b)) for a, b in z["sigs"]], w, json.loads(bytes(z["meta"]).decode())


def model_path(workload: str, model: str) -> str:
    import os
    return os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "models",
                        f"{workload}_{model}.npz")
