"""GPU parity of the tcgen05/TMEM bf16 MLP chain (P2-P5 of SURVEY.md §8(c)) against the
bf16-emulating oracle, across model shapes, ragged tails and multi-tile persistence."""
import numpy as np
import pytest

import tang_inputs as ti
from tests.test_gpu_parity import _logit_check
from tests._helpers import require_cuda

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    require_cuda()
    from paper_2601_03187_b200 import tang
    return tang


@pytest.mark.parametrize("N,B,n", [(64, 1, 1000), (128, 2, 4099), (256, 2, 3000), (512, 1, 2000),
                                   (512, 6, 19_001)])
def test_tc_logits_and_pipeline(T, N, B, n):
    """Logits within 1e-2 of the bf16-emulated oracle; flips explained; rule_id bit-exact
    with the oracle's stage 2 on the GPU's predictions; brute-force equal on G."""
    R = ti.classbench_ruleset("acl", 1000, 5)
    H = np.concatenate([ti.uniform_trace(R, n - 97, 9), ti.random_headers(97, 10)])
    err, flips = _logit_check(T, R, N, B, "bf16", H, seed=N + B, tol=1e-2)
    print(f"N={N} B={B} n={n}: max|dlogit|={err:.3g} flips={flips}")


def test_tc_wide_output_and_small_classes(T):
    """C > 256 (two N-halves in the output GEMM) and C < 16 (padding)."""
    for fam, n_rules, seed in (("acl", 3000, 1), ("fw", 40, 2)):
        R = ti.classbench_ruleset(fam, n_rules, seed)
        H = ti.uniform_trace(R, 1500, 3)
        _logit_check(T, R, 128, 1, "bf16", H, seed=3, tol=1e-2)


@pytest.mark.parametrize("k", [2, 4])
def test_tc_topk(T, k):
    torch = require_cuda()
    from oracle import mlp as omlp
    from tests._helpers import headers_dev, model, u32_dev, u32_host
    R = ti.classbench_ruleset("ipc", 1000, 3)
    H = ti.uniform_trace(R, 2000, 4)
    sigs, w, blob = model(R, 128, 1, 5)
    ctx = T.Ctx(R, blob, mlp="bf16", topk=k)
    out = u32_dev(H.size)
    pred = u32_dev(H.size * k)
    logits = torch.empty(H.size * len(sigs), dtype=torch.float32, device="cuda")
    ctx.classify_ex(headers_dev(H), out, pred, logits)
    torch.cuda.synchronize()
    L = logits.cpu().numpy().reshape(H.size, -1)
    gp = u32_host(pred).reshape(H.size, k)
    # the GPU's top-k must be the top-k of its own logits (ties to the lower index)
    assert np.array_equal(gp, omlp.topk(L.astype(np.float64), k))
