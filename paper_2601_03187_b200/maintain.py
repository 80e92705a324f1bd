"""Deferred-update policy of TaNG's maintenance workflow (§5.2.2) -- off the hot path.

Immediate updates (tang_update) keep the tuple set fixed, so accumulated inserts drift the
tuple boundaries away from what the model learned and throughput drops (more fallbacks).
The deferred update watches classification throughput per window: th_base is the first
window after the last full retrain, th_cur the current one; when 1 - th_cur/th_base > tau it
consults the counter of rules placed in a non-matching tuple since the last full retrain
(tang_stats mismatch_count): above theta -> full retraining (new TSS + model = a new
tang_build), else incremental training (warm-started fine-tune, hot-swapped with
tang_reload_model).  theta is read as a count (P:520 sets 10,000) or, when theta < 1, as the
proportion of live rules the text of P:344 describes (SURVEY.md §8(c) reading 20).
"""
from __future__ import annotations

from dataclasses import dataclass, field


@dataclass
class UpdateEngine:
    tau: float = 0.05
    theta: float = 10_000
    th_base: float | None = None
    history: list = field(default_factory=list)

    def mismatch_exceeds(self, mismatch_count: int, live_rules: int) -> bool:
        if self.theta < 1.0:                                  # proportion reading of P:344
            return mismatch_count > self.theta * max(1, live_rules)
        return mismatch_count > self.theta                    # count reading of P:520

    def observe(self, throughput: float, mismatch_count: int, live_rules: int) -> str:
        """Feed one window's throughput; returns 'none', 'incremental' or 'retrain'."""
        if self.th_base is None:
            self.th_base = throughput
            decision = "none"
        elif 1.0 - throughput / self.th_base > self.tau:
            decision = "retrain" if self.mismatch_exceeds(mismatch_count, live_rules) else "incremental"
        else:
            decision = "none"
        self.history.append((throughput, mismatch_count, decision))
        return decision

    def after_retrain(self):
        """A full retrain resets the baseline (the next window becomes th_base)."""
        self.th_base = None

    def after_incremental(self):
        """Incremental training keeps th_base: the paper compares against the last full retrain."""


def incremental_update(ctx, rules_live, sigs, weights, hdr_u8, seconds=20.0, log=None):
    """Label fresh traffic with the GPU brute force (k = 0) over the *current* tables, fine-tune
    the existing model on it (warm start) and hot-swap the weights; returns the new weights."""
    from . import tang as T, train as TR
    labels = TR.gpu_labels(ctx, hdr_u8, rules_live, sigs, placed=True)
    w, acc = TR.train(rules_live, sigs, int(weights["N"]), int(weights["B"]), hdr_u8, labels,
                      seconds=seconds, lr=3e-4, init=weights, log=log)
    ctx.reload_model(T.pack_blob(sigs, w))
    return w, acc
