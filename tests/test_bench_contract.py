"""bench.py host-side pieces (no GPU): the algorithmic FLOP count behind roofline.achieved is
SURVEY.md §8(d)'s per-packet formula, the ncu traffic table scales to the bench's launch size,
and the workload table names the BASELINE.json configs."""
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_mlp_flops_matches_survey_table(bench):
    # SURVEY.md §8(d) "Algorithmic work per packet": 2(S.N + 2B.N^2 + N.C)
    assert round(bench.mlp_flops(7, 512, 6, 193) / 1e6, 2) == 6.50
    assert round(bench.mlp_flops(7, 512, 6, 400) / 1e6, 2) == 6.71
    assert round(bench.mlp_flops(7, 256, 2, 400) / 1e6, 2) == 0.73
    assert round(bench.mlp_flops(7, 256, 4, 400) / 1e6, 2) == 1.26
    # hand count of a 1-1-2 network: layer 0 7x1, two 1x1 GEMMs, output 1x2
    assert bench.mlp_flops(7, 1, 1, 2) == 2 * (7 + 2 + 2)


def test_traffic_entries_are_per_launch_with_their_launch_size(bench):
    for key in ("acl-512k/paper", "acl-512k/paper/fp8", "acl-512k/reduced/fp8"):
        workload, model = key.split("/")[0], key.split("/")[1]
        mlp = key.split("/")[2] if key.count("/") == 2 else "bf16"
        t = bench.load_traffic(workload, model, mlp)
        assert t is not None and t["dram_bytes_per_launch"] > 16 * t["packets_per_launch"]  # >= headers


def test_workloads_cover_baseline_configs(bench):
    w = bench.WORKLOADS
    assert w["acl-1k"][1] == 1000 and w["acl-10k"][1] == 10000 and w["acl-100k"][1] == 100000
    assert {w[k][0] for k in ("acl-512k", "fw-512k", "ipc-512k")} == {"acl", "fw", "ipc"}
    assert w["acl-100k-zipf"][3] == "zipf" and w["acl-1m"][1] == 1 << 20
