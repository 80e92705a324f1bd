"""TaNG's two-stage classification, step by step (test infrastructure only).

P:272-276 (§5.1.1): stage 1, the model predicts a tuple index; stage 2, the
search engine probes that tuple's hash table and compares its rules one by one.
Post-verification: a flag records whether the predicted tuple held a match; if
not, an ordered search over the remaining tuples finds the highest-priority rule.
Scenario 1 (the predicted tuple holds a *lower*-priority match) is explicitly
left uncorrected by the paper -- "paper" mode reproduces that;
"strict" mode additionally searches the tuples
whose best priority beats the in-tuple match, so its result is the brute force.

Top-k (k > 1) is SURVEY.md §8(c) reading 18: the k predicted tuples are probed
and the best of their matches is kept; k = 1 is the paper.
"""
from __future__ import annotations

import numpy as np

from .mlp import argmax, features, forward, topk
from .tss import NO_MATCH


def classify_with_pred(tss, headers: np.ndarray, pred: np.ndarray, mode: str = "paper"):
    """Stage 2 + post-verification given predicted tuples pred [n, k] (k may be 0).

    Returns (rule_id [n] u32, fellback [n] bool, accesses [n] int)."""
    pred = np.asarray(pred, dtype=np.int64).reshape(headers.size, -1)
    n = headers.size
    out = np.full(n, NO_MATCH, dtype=np.uint32)
    fell = np.zeros(n, dtype=bool)
    acc = np.zeros(n, dtype=np.int64)
    for i in range(n):
        h = headers[i]
        best, a = None, 0
        for j in pred[i]:                             # O9 over the k predicted tuples
            m, aj = tss.lookup_in_tuple(int(j), h)
            a += aj
            if m is not None and (best is None or m < best):
                best = m
        if best is None:                              # O10: post-verification
            fell[i] = True
            best, aj = tss.ordered_search(h, skip=pred[i])
            a += aj
        elif mode == "strict":                        # O11: beat-the-bound search
            best2, aj = tss.ordered_search(h, skip=pred[i], bound=best)
            a += aj
            if best2 is not None and best2 < best:
                fell[i] = True
                best = best2
        acc[i] = a
        out[i] = NO_MATCH if best is None else best[1]
    return out, fell, acc


def predict(weights: dict, headers: np.ndarray, mode: str = "fp32", k: int = 1):
    """Stage 1: logits and predicted tuple(s) [n, k]."""
    logits = forward(weights, features(headers), mode)
    pred = argmax(logits)[:, None] if k == 1 else topk(logits, k)
    return logits, pred


def classify(tss, weights: dict, headers: np.ndarray, mlp_mode: str = "bf16",
             mode: str = "paper", k: int = 1):
    """Full pipeline: returns dict(rule_id, pred, logits, fellback, accesses)."""
    logits, pred = predict(weights, headers, mlp_mode, k)
    rid, fell, acc = classify_with_pred(tss, headers, pred, mode)
    return dict(rule_id=rid, pred=pred, logits=logits, fellback=fell, accesses=acc)


def statistics(tss, pred: np.ndarray, rule_id: np.ndarray, truth: np.ndarray, accesses=None):
    """O12 / Tables 2-3: model accuracy = a predicted tuple hosts the
    brute-force winner (over matched packets); classification accuracy =
    rule_id == brute force; fallback rate; mean accesses per lookup."""
    pred = np.asarray(pred).reshape(rule_id.size, -1)
    matched = truth != NO_MATCH
    host = np.array([tss.tuple_of(int(t)) if t != NO_MATCH else -1 for t in truth])
    model_ok = np.array([host[i] in set(pred[i].tolist()) for i in range(truth.size)]) & matched
    return dict(
        model_accuracy=float(model_ok.sum() / max(1, matched.sum())),
        classification_accuracy=float((rule_id == truth).mean()) if truth.size else 1.0,
        tuples=len(tss.sigs),
        mean_accesses=float(np.mean(accesses)) if accesses is not None and len(accesses) else 0.0,
    )
