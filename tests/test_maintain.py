"""Deferred-update policy and model hot-swap validation (CPU)."""
import numpy as np
import pytest

import tang_inputs as ti
from paper_2601_03187_b200 import maintain as M, tang as T, train as TR


def test_tau_theta_decisions_count_reading():
    e = M.UpdateEngine(tau=0.05, theta=10_000)
    assert e.observe(10.23, 0, 256_000) == "none"             # first window sets th_base
    assert e.observe(9.80, 2_000, 256_000) == "none"           # -4.2 % < tau
    assert e.observe(9.45, 4_000, 256_000) == "incremental"    # -7.6 % > tau, few mismatches
    e.after_incremental()
    assert e.th_base == 10.23                                   # baseline kept until a full retrain
    assert e.observe(9.11, 12_000, 256_000) == "retrain"       # many rules in non-matching tuples
    e.after_retrain()
    assert e.observe(10.1, 0, 256_000) == "none" and e.th_base == 10.1


def test_theta_proportion_reading():
    e = M.UpdateEngine(tau=0.05, theta=0.02)
    e.observe(100.0, 0, 10_000)
    assert e.observe(90.0, 150, 10_000) == "incremental"        # 1.5 % <= 2 %
    assert e.observe(90.0, 250, 10_000) == "retrain"            # 2.5 % > 2 %


def test_reload_requires_same_tuple_set():
    R = ti.classbench_ruleset("acl", 500, 1)
    sigs = TR.tuple_signatures(R)
    w = ti.random_weights(7, 64, 1, len(sigs), 0)
    ctx = T.Ctx(R, T.pack_blob(sigs, w), device=-1)
    ctx.reload_model(T.pack_blob(sigs, ti.random_weights(7, 64, 1, len(sigs), 1)))   # same set: ok
    with pytest.raises(T.TangError) as e:
        ctx.reload_model(T.pack_blob(list(reversed(sigs)), w))                         # reordered classes
    assert e.value.code == T.TANG_EMODEL
    with pytest.raises(T.TangError):
        ctx.reload_model(T.pack_blob(sigs, ti.random_weights(7, 128, 1, len(sigs), 1)))  # other N
